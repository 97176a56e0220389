"""Row-sharded multi-GPU Greedy (north-star item d).

One process per GPU.  Rank r owns the point rows [r0, r1) of V (aligned to
the global partial-sum split, so every per-point term is computed by exactly
one rank) plus a replica of the candidate layouts (for Greedy the candidates
are V itself).  Per step:

    K3  local partial gains G_r[c] = sum_{i in shard r} max(0, m_i - d(v_i,c))
    all-reduce(sum) of the l fp64 gains over NCCL (torch.distributed)
    K5  identical masked argmax on every rank (lowest index on ties)
    K2  local m-update with the chosen exemplar; local sum m -> msum[step]

and one all-reduce of the k trajectory sums at the end.  This is the
reference's greedy loop (pkg/src/exembatch/optimize.py:61-76) with the work
matrix W split by columns across GPUs.

The collective logic is written against a small ``ShardOps`` interface so
the multi-process CPU tests (gloo, world_size 2) can drive the same loop.

Explicit batches (``sharded_batch_sums``, BASELINE config 5) shard the same
way: each rank streams its split-aligned rows through K4 / K4-TC into its
rows of the [splits][l] partial matrix, the other rows stay zero, and one
all-reduce(sum) of that matrix reconstructs every partial exactly (x + 0 is
exact), so the fixed-order K6 reduce gives per-set sums bit-identical to a
single GPU for any number of ranks.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Protocol

import numpy as np


def shard_rows(n: int, world: int, rank: int, split_pts: int) -> tuple:
    """[r0, r1) rows of rank ``rank``: whole splits, as even as possible."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    splits = -(-n // split_pts)
    base, extra = divmod(splits, world)
    s0 = rank * base + min(rank, extra)
    s1 = s0 + base + (1 if rank < extra else 0)
    return min(n, s0 * split_pts), min(n, s1 * split_pts)


class ShardOps(Protocol):
    """What one rank must provide to run the sharded Greedy loop."""

    def start(self) -> None: ...
    def local_gains(self) -> None: ...          # fills the l-vector buffer
    def gains_buffer(self): ...                 # tensor all-reduced in place
    def select(self, step: int) -> None: ...
    def update(self, step: int) -> None: ...
    def msum_buffer(self): ...                  # [k] local sums of m
    def picks(self) -> np.ndarray: ...


def sharded_greedy_loop(ops: ShardOps, k: int, all_reduce, on_step=None):
    """Drive k Greedy steps; ``all_reduce(tensor)`` sums in place."""
    ops.start()
    for step in range(k):
        ops.local_gains()
        all_reduce(ops.gains_buffer())
        ops.select(step)
        ops.update(step)
        if on_step is not None:
            on_step(step)
    all_reduce(ops.msum_buffer())
    return ops.picks()[:k], ops.msum_buffer()


class DeviceShardOps:
    """``ShardOps`` on the B200 kernels (K3/K6, K5, K2)."""

    def __init__(self, run):
        self.run = run

    def start(self):
        self.run.start()

    def local_gains(self):
        self.run.compute_gains()

    def gains_buffer(self):
        return self.run.gains

    def select(self, step):
        self.run.select(step)

    def update(self, step):
        self.run.update(step)

    def msum_buffer(self):
        return self.run.msum

    def picks(self):
        return self.run.sel_idx.cpu().numpy()


@dataclass
class ShardedGround:
    """Local shard + candidate replica of one rank."""

    local: object        # DeviceGround of rows [r0, r1)
    cand: object         # DeviceGround of all of V (candidates)
    rows: tuple
    n: int
    aux_loss: float
    precision: object


def build_sharded_ground(V: np.ndarray, precision, rank: int, world: int,
                         device=None, aux="zero") -> ShardedGround:
    """Upload V, build the candidate replica and this rank's point shard."""
    from . import _native as N
    from .core import _aux_vector, build_ground_set
    from .device import prepare_ground

    full = build_ground_set(V, aux=aux, precision=precision, device=device)
    cand = full.on_device(device)
    sp = int(N.lib().split_points(full.n))
    r0, r1 = shard_rows(full.n, world, rank, sp)
    if world == 1:
        local = cand
    else:
        local, _, _ = prepare_ground(full.matrix[r0:r1], full.aux,
                                     precision, device)
    return ShardedGround(local=local, cand=cand, rows=(r0, r1), n=full.n,
                         aux_loss=full.aux_loss, precision=precision)


def sharded_greedy(sg: ShardedGround, k: int, group=None):
    """Row-sharded Greedy on the calling rank; returns (picks, values)."""
    import torch.distributed as dist

    from . import _native as N
    from .optimize import GreedyRun

    sp = int(N.lib().split_points(sg.n))
    run = GreedyRun(sg.local, cand=sg.cand, k_cap=k, split_pts=sp)
    ops = DeviceShardOps(run)

    def all_reduce(t):
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    picks, msum = sharded_greedy_loop(ops, k, all_reduce)
    acc = sg.precision.accumulate_dtype
    ms = msum.cpu().numpy()[:k]
    vals = acc.type(sg.aux_loss) - ms.astype(acc) / acc.type(sg.n)
    return tuple(int(i) for i in picks), tuple(float(v) for v in vals)


def combine_partials(partial, all_reduce) -> None:
    """All-reduce a [splits][l] partial matrix whose rows are owned by
    exactly one rank (zeros elsewhere): exact, order-independent."""
    all_reduce(partial)


def sharded_batch_sums(ground, batch, rank: int, world: int, group=None,
                       device=None, budget=None):
    """Per-set fp64 sums of an explicit batch over a row-sharded V.

    Rank ``rank`` evaluates every set against its rows [r0, r1) (whole
    splits, ``shard_rows``), streamed through ``budget`` bytes of device
    memory (default: the ground set's budget, else 80 % of free memory).
    Returns the device tensor of l sums, identical on every rank.
    """
    import torch
    import torch.distributed as dist

    from . import _native as N
    from .streaming import stream_packed_sums

    lib = N.lib()
    n = ground.n
    sp = int(lib.split_points(n))
    splits = -(-n // sp)
    r0, r1 = shard_rows(n, world, rank, sp)
    dev = torch.device("cuda", torch.cuda.current_device()
                       if device is None else device)
    partial = torch.zeros((splits, batch.l), dtype=torch.float64, device=dev)
    if budget is None:
        budget = ground.device_budget or int(
            0.8 * torch.cuda.mem_get_info(dev)[0])
    if r1 > r0:
        stream_packed_sums(ground, None, batch.d, batch.k_max, batch.l,
                           batch.cardinalities, dev.index, rows=(r0, r1),
                           partial=partial, budget=budget, sets=batch.sets)

    def all_reduce(t):
        if world > 1 and dist.is_available() and dist.is_initialized():
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    combine_partials(partial, all_reduce)
    sums = torch.empty(batch.l, dtype=torch.float64, device=dev)
    lib.reduce_partials(N.ptr(partial), splits, batch.l, 1.0, N.ptr(sums),
                        N.stream_handle(dev))
    return sums
