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
from typing import Protocol

import numpy as np


# NCCL settings applied before the communicator is created (SURVEY.md 8(e)
# "Determinism"): a fixed algorithm and protocol make the summation order of
# the per-step all-reduce -- and so every fp64 gain bit -- repeatable run to
# run for a given rank count (NCCL otherwise tunes per message size and
# topology).  Ring/Simple moves the 8 MB gains vector in ~10-30 us on NVLink
# 5, < 0.1 % of a step.  The INIT log (one line per rank with "nRanks") goes
# to stderr so a scaling run can verify the communicator size without
# touching the JSON line on stdout.  Every setting is a default only: an
# explicit environment value wins.
NCCL_DEFAULTS = {
    "NCCL_ALGO": "Ring",
    "NCCL_PROTO": "Simple",
    "NCCL_DEBUG": "INFO",
    "NCCL_DEBUG_SUBSYS": "INIT",
    "NCCL_DEBUG_FILE": "/dev/stderr",
}


def pin_nccl_env(environ=None) -> dict:
    """Apply ``NCCL_DEFAULTS`` (setdefault) and return the effective values;
    call before ``init_process_group("nccl")``."""
    import os

    env = os.environ if environ is None else environ
    for key, val in NCCL_DEFAULTS.items():
        env.setdefault(key, val)
    return {k: env[k] for k in ("NCCL_ALGO", "NCCL_PROTO")}


def communicator_record(group=None) -> dict:
    """What a scaling run must be able to check: ranks, backend, NCCL
    version, pinned algorithm/protocol."""
    import os

    import torch
    import torch.distributed as dist

    rec = {"backend": dist.get_backend(group),
           "nranks": dist.get_world_size(group),
           "nccl_algo": os.environ.get("NCCL_ALGO"),
           "nccl_proto": os.environ.get("NCCL_PROTO")}
    try:
        rec["nccl_version"] = ".".join(str(x) for x in torch.cuda.nccl.version())
    except Exception:  # noqa: BLE001 -- no NCCL in this torch build
        rec["nccl_version"] = None
    return rec


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


def sharded_greedy_graphed(ops: ShardOps, k: int, all_reduce):
    """``sharded_greedy_loop`` with steps 1..k-1 replayed from one CUDA graph
    (step 0 runs eagerly so every kernel and the communicator are warm)."""
    from .optimize import capture_steps

    def do_step(step):
        ops.local_gains()
        all_reduce(ops.gains_buffer())
        ops.select(step)
        ops.update(step)

    ops.start()
    do_step(0)
    capture_steps(range(1, k), do_step).replay()
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


class EmptyShardOps:
    """``ShardOps`` of a rank that owns no points (more ranks than splits):
    it contributes zero gains and zero m-sums and runs the same K5 argmax on
    the all-reduced gains, so its picks equal every other rank's."""

    def __init__(self, cand, k: int):
        from . import _native as N
        from .device import torch

        t = torch()
        self.N, self.lib, self.cand = N, N.lib(), cand
        dev = cand.dev
        self.l = cand.n
        self.gains = t.zeros(self.l, dtype=t.float64, device=dev)
        self.selected = t.zeros(self.l, dtype=t.uint8, device=dev)
        self.sel_idx = t.zeros(k, dtype=t.int64, device=dev)
        self.sel_gain = t.zeros(k, dtype=t.float64, device=dev)
        self.msum = t.zeros(k, dtype=t.float64, device=dev)
        self.scratch = t.empty(int(self.lib.reduce_scratch(self.l)),
                               dtype=t.float64, device=dev)

    def start(self):
        pass

    def local_gains(self):
        self.gains.zero_()

    def gains_buffer(self):
        return self.gains

    def select(self, step):
        N = self.N
        self.lib.argmax_select(N.ptr(self.gains), self.l, N.ptr(self.selected),
                               None, step, N.ptr(self.sel_idx),
                               N.ptr(self.sel_gain), N.ptr(self.scratch),
                               self.cand.stream)

    def update(self, step):
        pass

    def msum_buffer(self):
        return self.msum

    def picks(self):
        return self.sel_idx.cpu().numpy()


@dataclass
class ShardedGround:
    """Local shard + candidate replica of one rank."""

    local: object        # DeviceGround of rows [r0, r1) (None: no rows)
    cand: object         # DeviceGround of all of V (candidates)
    rows: tuple
    n: int
    aux_loss: float
    precision: object


def build_sharded_ground(V: np.ndarray, precision, rank: int, world: int,
                         device=None, aux="zero") -> ShardedGround:
    """Upload V, build the candidate replica and this rank's point shard."""
    from . import _native as N
    from .core import build_ground_set
    from .device import prepare_ground

    full = build_ground_set(V, aux=aux, precision=precision, device=device)
    cand = full.on_device(device)
    sp = int(N.lib().split_points(full.n))
    r0, r1 = shard_rows(full.n, world, rank, sp)
    if world == 1:
        local = cand
    elif r1 <= r0:  # more ranks than splits: this rank owns no points
        local = None
    else:
        local, _, _ = prepare_ground(full.matrix[r0:r1], full.aux,
                                     precision, device)
    return ShardedGround(local=local, cand=cand, rows=(r0, r1), n=full.n,
                         aux_loss=full.aux_loss, precision=precision)


def sharded_greedy(sg: ShardedGround, k: int, group=None, graph: bool = False):
    """Row-sharded Greedy on the calling rank; returns (picks, values).

    ``graph=True``: steps 1..k-1 (K3, K6, the NCCL all-reduce, K5, K2) are
    captured into one CUDA graph after an eager step 0 and replayed once
    (optimize.capture_steps)."""
    import torch.distributed as dist

    from . import _native as N
    from .optimize import GreedyRun

    from .device import torch
    from .optimize import checked_picks

    sp = int(N.lib().split_points(sg.n))

    def all_reduce(t):
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    with torch().cuda.device(sg.cand.device_index):
        if sg.local is None:
            ops = EmptyShardOps(sg.cand, k)
        else:
            ops = DeviceShardOps(GreedyRun(sg.local, cand=sg.cand, k_cap=k,
                                           split_pts=sp))
        if graph and k > 1:
            picks, msum = sharded_greedy_graphed(ops, k, all_reduce)
        else:
            picks, msum = sharded_greedy_loop(ops, k, all_reduce)
        picks = checked_picks(picks, k)
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


# ------------------------------------------------------- peer-memory K5
class PeerGains:
    """Per-step gains exchange over peer memory instead of an NCCL
    all-reduce (opt-in; ``peer_greedy``).

    Every rank owns an IPC-shared buffer holding its local gains for two
    step parities plus a step flag.  After its K3 + K6 a rank publishes
    ``flag = step + 1``; ``select`` then runs exem_peer_argmax_select, which
    waits for all flags, sums the W local vectors in fixed rank order
    directly from the peers' memory (NVLink P2P on a B200 node) and takes the
    argmax -- identical on every rank, and independent of any collective
    algorithm.  Step t writes parity t % 2; a rank can only reach step t+2
    after every peer published step t+1, which each peer does after its
    step-t read, so a buffer is never overwritten while being read.
    """

    def __init__(self, l: int, device, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _native as N

        self.lib = N.lib()
        self.l = l
        self.dev = device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group = group
        # the IPC allocations and the flag kernel go to the current device
        # (static cudart): make it the run's device
        with torch.cuda.device(device):
            self._open(ctypes, torch, dist, N)

    def _open(self, ctypes, torch, dist, N):
        lib, l, device, group = self.lib, self.l, self.dev, self.group
        ptr = ctypes.c_void_p()
        lib.ipc_alloc(2 * l * 8, ctypes.byref(ptr))
        self.own = ptr.value
        fptr = ctypes.c_void_p()
        lib.ipc_alloc(8, ctypes.byref(fptr))
        self.own_flag = fptr.value
        st = N.stream_handle(device)
        lib.peer_publish(N.c_void_p(self.own_flag), 0, st)
        torch.cuda.synchronize(device)
        handles = []
        for p_ in (self.own, self.own_flag):
            h = ctypes.create_string_buffer(64)
            lib.ipc_handle(N.c_void_p(p_), h)
            handles.append(h.raw)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, handles, group=group)
        self.opened = []
        gains_ptrs, flag_ptrs = [], []
        for q, (gh, fh) in enumerate(everyone):
            if q == self.rank:
                gains_ptrs.append(self.own)
                flag_ptrs.append(self.own_flag)
                continue
            for h, dst in ((gh, gains_ptrs), (fh, flag_ptrs)):
                out = ctypes.c_void_p()
                lib.ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(out))
                self.opened.append(out.value)
                dst.append(out.value)
        self.peers = torch.tensor(
            [[p_ + par * l * 8 for p_ in gains_ptrs] for par in (0, 1)],
            dtype=torch.int64, device=device)
        self.flags = torch.tensor(flag_ptrs, dtype=torch.int64, device=device)

    def local_buffer(self, step: int):
        from . import _native as N

        return N.c_void_p(self.own + (step % 2) * self.l * 8)

    def publish(self, step: int, stream) -> None:
        from . import _native as N

        self.lib.peer_publish(N.c_void_p(self.own_flag), step + 1, stream)

    def select(self, run, step: int) -> None:
        """Fixed-order sum of the peers' gains + masked argmax (K5)."""
        from . import _native as N

        self.lib.peer_argmax_select(
            N.c_void_p(self.peers[step % 2].data_ptr()),
            N.c_void_p(self.flags.data_ptr()), self.world, step + 1, self.l,
            1.0, N.ptr(run.gains), N.ptr(run.selected), step,
            N.ptr(run.sel_idx), N.ptr(run.sel_gain), N.ptr(run.scratch),
            run.stream)

    def close(self) -> None:
        import torch
        import torch.distributed as dist

        from . import _native as N

        torch.cuda.synchronize(self.dev)
        dist.barrier(group=self.group)  # no peer reads our buffers any more
        for p_ in self.opened:
            self.lib.ipc_close(N.c_void_p(p_))
        dist.barrier(group=self.group)
        self.lib.ipc_free(N.c_void_p(self.own))
        self.lib.ipc_free(N.c_void_p(self.own_flag))


def peer_greedy(sg: ShardedGround, k: int, group=None):
    """Row-sharded Greedy with the per-step exchange over peer memory
    (PeerGains) instead of NCCL; one host all-reduce of the k trajectory
    sums at the end.  Returns (picks, values) like ``sharded_greedy``."""
    import torch.distributed as dist

    from . import _native as N
    from .device import torch
    from .optimize import GreedyRun, checked_picks

    if sg.local is None:
        raise ValueError(
            "peer_greedy needs at least one split of points per rank "
            f"(n={sg.n}); use sharded_greedy or fewer ranks")
    sp = int(N.lib().split_points(sg.n))
    with torch().cuda.device(sg.local.device_index):
        return _peer_greedy(sg, k, group, sp, GreedyRun, checked_picks, dist)


def _peer_greedy(sg, k, group, sp, GreedyRun, checked_picks, dist):
    run = GreedyRun(sg.local, cand=sg.cand, k_cap=k, split_pts=sp)
    peer = PeerGains(run.l, run.dg.dev, group)
    try:
        run.start()
        for step in range(k):
            run.compute_gains(out=peer.local_buffer(step))
            peer.publish(step, run.stream)
            peer.select(run, step)
            run.update(step)
        if dist.is_initialized():
            dist.all_reduce(run.msum, op=dist.ReduceOp.SUM, group=group)
        picks = checked_picks(run.sel_idx.cpu().numpy(), k)
        msum = run.msum.cpu().numpy()[:k]
    finally:
        peer.close()
    acc = sg.precision.accumulate_dtype
    vals = acc.type(sg.aux_loss) - msum.astype(acc) / acc.type(sg.n)
    return tuple(int(i) for i in picks), tuple(float(v) for v in vals)
