"""Row-sharded Greedy over torch.distributed (gloo, world_size 2, CPU).

The product's multi-GPU driver (paper_2101_08763_b200/distributed.py) runs
the loop K3 -> all-reduce(l gains) -> K5 argmax -> K2 m-update on every rank
with V row-sharded.  Here the same ``sharded_greedy_loop`` and ``shard_rows``
run in two CPU processes over gloo, with each rank's per-shard arithmetic
supplied by the fp64 oracle (the device kernels need a B200; the GPU tests
cover them).  The sharded run must reproduce the single-process trajectory.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import exem_oracle as O
from paper_2101_08763_b200.distributed import shard_rows, sharded_greedy_loop


class OracleShardOps:
    """ShardOps over this rank's rows, fp64 numpy arithmetic."""

    def __init__(self, V, rows, k):
        self.V = np.asarray(V, np.float64)
        self.r0, self.r1 = rows
        self.loc = self.V[self.r0:self.r1]
        self.gains = torch.zeros(self.V.shape[0], dtype=torch.float64)
        self.msum = torch.zeros(k, dtype=torch.float64)
        self.sel = np.zeros(k, dtype=np.int64)
        self.mask = np.zeros(self.V.shape[0], dtype=bool)

    def start(self):
        self.m = O.aux64(self.loc)

    def local_gains(self):
        g = O.gains_m(self.loc, self.m, self.V) if len(self.loc) else np.zeros(len(self.V))
        self.gains.copy_(torch.from_numpy(g))

    def gains_buffer(self):
        return self.gains

    def select(self, step):
        g = self.gains.numpy().copy()
        g[self.mask] = -np.inf
        c = int(np.argmax(g))  # first maximum: lowest index (optimize.py:73)
        self.mask[c] = True
        self.sel[step] = c

    def update(self, step):
        c = self.sel[step]
        d = ((self.loc - self.V[c]) ** 2).sum(1)
        self.m = np.minimum(self.m, d)
        self.msum[step] = float(self.m.sum())

    def msum_buffer(self):
        return self.msum

    def picks(self):
        return self.sel


def _worker(rank, world, port, V, k, split_pts, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows = shard_rows(V.shape[0], world, rank, split_pts)
        ops = OracleShardOps(V, rows, k)

        def all_reduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

        picks, msum = sharded_greedy_loop(ops, k, all_reduce)
        out[rank] = (list(picks), msum.numpy().tolist(), rows)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,d,split_pts", [(3000, 8, 1024), (2500, 5, 1024)])
def test_row_sharded_greedy_matches_single_process(n, d, split_pts):
    rng = np.random.default_rng(n + d)
    V = rng.standard_normal((n, d))
    k = 4
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), V, k, split_pts, out),
             nprocs=world, join=True)
    picks_ref, vals_ref, _ = O.greedy_m(V, k)
    aux_loss = O.aux64(V).sum() / n
    for rank in range(world):
        picks, msum, rows = out[rank]
        assert picks == list(picks_ref)
        vals = aux_loss - np.array(msum) / n
        np.testing.assert_allclose(vals, vals_ref, rtol=0, atol=1e-9)
    # the shards tile [0, n) on split boundaries
    r0 = sorted(out[r][2] for r in range(world))
    assert r0[0][0] == 0 and r0[-1][1] == n and r0[0][1] == r0[1][0]
    assert r0[0][1] % split_pts == 0


def test_shard_rows_partition():
    for n in (1, 1000, 4097, 100_000, 1_000_000):
        for world in (1, 2, 3, 4, 8):
            sp = 1024
            ranges = [shard_rows(n, world, r, sp) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0 and a0 <= a1
                assert a1 % sp == 0 or a1 == n
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2, 1024)


# ------------------------------------------------------------ explicit batches
def _split_partials(V, sets, rows, split_pts):
    """[splits][l] fp64 partials of t_i(S_j) over this rank's rows only."""
    n = V.shape[0]
    splits = -(-n // split_pts)
    aux = O.aux64(V)
    out = np.zeros((splits, len(sets)))
    r0, r1 = rows
    for j, S in enumerate(sets):
        d = ((V[r0:r1, None, :] - V[S][None, :, :]) ** 2).sum(-1).min(1)
        t = np.minimum(aux[r0:r1], d)
        for s in range(r0 // split_pts, -(-r1 // split_pts)):
            a, b = max(r0, s * split_pts), min(r1, (s + 1) * split_pts)
            out[s, j] = t[a - r0:b - r0].sum()
    return out


def _batch_worker(rank, world, port, V, sets, split_pts, out):
    from paper_2101_08763_b200.distributed import combine_partials

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows = shard_rows(V.shape[0], world, rank, split_pts)
        part = torch.from_numpy(_split_partials(V, sets, rows, split_pts))

        def all_reduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

        combine_partials(part, all_reduce)
        out[rank] = part.numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_batch_partials_exact(world):
    """Config 5's collective: each rank fills its own split rows of the
    [splits][l] matrix, the all-reduce of the zero-padded matrices equals the
    single-process matrix BIT FOR BIT (x + 0 is exact), so the fixed-order
    per-set reduction that follows is independent of the rank count."""
    rng = np.random.default_rng(world)
    n, d, split_pts = 5000, 6, 1024
    V = rng.standard_normal((n, d))
    sets = [rng.choice(n, size=int(rng.integers(1, 6)), replace=False)
            for _ in range(7)]
    ref = _split_partials(V, sets, (0, n), split_pts)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_batch_worker, args=(world, _free_port(), V, sets, split_pts, out),
             nprocs=world, join=True)
    for rank in range(world):
        assert np.array_equal(out[rank], ref)


def test_nccl_env_is_pinned_but_overridable():
    """SURVEY 8(e) Determinism: a fixed NCCL algorithm/protocol, the INIT
    log on stderr, explicit environment values win."""
    from paper_2101_08763_b200.distributed import NCCL_DEFAULTS, pin_nccl_env

    env = {"NCCL_PROTO": "LL128"}
    eff = pin_nccl_env(env)
    assert eff == {"NCCL_ALGO": "Ring", "NCCL_PROTO": "LL128"}
    for key in NCCL_DEFAULTS:
        assert key in env
    assert env["NCCL_DEBUG_SUBSYS"] == "INIT"
    assert env["NCCL_DEBUG_FILE"] == "/dev/stderr"


def _comm_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2101_08763_b200.distributed import communicator_record

    out[rank] = communicator_record()
    dist.destroy_process_group()


def test_communicator_record_reports_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_comm_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0]["nranks"] == 2 and out[1]["nranks"] == 2
    assert out[0]["backend"] == "gloo"
