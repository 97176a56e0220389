"""Edge cases of the device path that the reference handles and a naive
kernel would get silently wrong.

* binary16 operand range: the tensor-core operands fold ||x||^2/2 into three
  f16 pieces (p0 * 2^11 + p1 + p2, exem_common.cuh fold_pieces).  Ground sets
  whose norms exceed the single-f16 range (65504) but whose distances are
  small (offset data with the auxiliary vector near it -- the reference's
  direct-form f16 arithmetic, objective.py:76-80, is fine there) must stay
  correct on the tensor cores; norms beyond the folded range route to the
  CUDA-core kernels (no NaN, no silent wrong picks).
* K5 with no valid candidate writes the sentinel -1 and the host raises
  (never a duplicate exemplar).
* GroundSet.matrix is column-major like the reference's
  (tests/test_core.py:70-73), also for large row-major inputs transposed on
  the device.
* Row-sharded Greedy with more ranks than splits (an empty shard).
"""

import os
import socket

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import Evaluator, Precision
from paper_2101_08763_b200 import _native as N
from paper_2101_08763_b200.errors import InvalidDataError
from paper_2101_08763_b200.optimize import GreedyRun, checked_picks
from spotcheck import teacher_forced_trajectory

pytestmark = pytest.mark.gpu

P16 = Precision.binary16


def _offset_case(offset, spread, n, d, seed):
    rng = np.random.default_rng(seed)
    V = (offset + spread * rng.standard_normal((n, d))).astype(np.float16)
    e0 = np.full(d, offset, dtype=np.float16)
    return V, e0


def test_f16_large_norms_stay_on_tensor_cores():
    # ||v||^2 ~ 128 * 40^2 = 2.0e5: h = ||v||^2/2 ~ 1.0e5 > 65504 (an
    # unscaled first f16 piece overflows to inf -> NaN dot products)
    V, e0 = _offset_case(40.0, 2.0, 3000, 128, 1)
    g = pb.build_ground_set(V, aux=e0, precision=P16)
    dg = g.on_device()
    assert dg.fold_ok()
    assert float(dg.norms[: g.n].max()) > 2 * 65504
    run = GreedyRun(dg, k_cap=1)
    assert run.tc  # the folded tcgen05 path
    res = pb.greedy_maximize(g, k=4)
    # fp64 truth from the stored values and stored aux distances, teacher
    # forced.  GEMM-form cancellation at ||v||^2 ~ 2e5 in fp32 (ulp 0.016)
    # against distances ~ 1e3 bounds the accuracy here, as for the
    # reference's binary32 path on such data.
    teacher_forced_trajectory(
        g, res, lambda G: 2e-3 * max(1.0, abs(G)),
        lambda f: 2e-3 * max(1.0, abs(f)), label="f16 offset 40")
    # explicit sets on K4-TC (folded operands, d = 128)
    rng = np.random.default_rng(2)
    sets = [np.sort(rng.choice(g.n, size=int(rng.integers(1, 40)),
                               replace=False)) for _ in range(40)]
    got = pb.evaluate_batch(Evaluator(), g,
                            pb.EvaluationBatch.from_sets([g.matrix[i]
                                                          for i in sets]))
    ref = _oracle_values(g, sets)
    assert np.all(np.isfinite(got))
    assert np.all(np.abs(got - ref) <= 2e-3 * np.maximum(1.0, np.abs(ref)))


def _oracle_values(g, sets):
    """fp64 oracle on the stored values, with the device's aux_loss."""
    og = O.Ground(g.matrix.astype(np.float64), np.float64,
                  aux=g.aux.astype(np.float64))
    og.aux_distances = np.asarray(g.aux_distances, np.float64)
    og.aux_loss = float(g.aux_loss)
    return O.evaluate_batch(og, [og.matrix[i] for i in sets])


def test_f16_norms_beyond_fold_range():
    # ||v||^2 ~ 64 * 3000^2 = 5.8e8 > 2 * 65504 * 2048: beyond the folded
    # range.  Explicit sets run on the CUDA cores in the reference's direct
    # form (exact here); Greedy, tensor-core only at binary16, raises.
    V, e0 = _offset_case(3000.0, 2.0, 2000, 64, 3)
    g = pb.build_ground_set(V, aux=e0, precision=P16)
    dg = g.on_device()
    assert not dg.fold_ok()
    with pytest.raises(InvalidDataError):
        pb.greedy_maximize(g, k=2)
    rng = np.random.default_rng(4)
    sets = [np.sort(rng.choice(g.n, size=int(rng.integers(1, 20)),
                               replace=False)) for _ in range(25)]
    got = pb.evaluate_batch(Evaluator(), g,
                            pb.EvaluationBatch.from_sets([g.matrix[i]
                                                          for i in sets]))
    ref = _oracle_values(g, sets)
    # f is rounded to binary32 (the accumulate dtype): ~1 ulp32(aux_loss)
    slack = 2 * float(np.spacing(np.float32(g.aux_loss)))
    assert np.all(np.abs(got - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref))
                  + slack)
    f1 = pb.evaluate_single(g, g.matrix[sets[0]])
    assert abs(f1 - ref[0]) <= 1e-5 * max(1.0, abs(ref[0])) + slack


def test_argmax_without_valid_candidate_is_an_error():
    import torch

    lib = N.lib()
    dev = torch.device("cuda", 0)
    l = 5000
    gains = torch.full((l,), float("nan"), dtype=torch.float64, device=dev)
    selected = torch.zeros(l, dtype=torch.uint8, device=dev)
    sel_idx = torch.full((2,), 7, dtype=torch.int64, device=dev)
    sel_gain = torch.zeros(2, dtype=torch.float64, device=dev)
    scratch = torch.empty(int(lib.reduce_scratch(l)), dtype=torch.float64,
                          device=dev)
    st = N.stream_handle(dev)
    lib.argmax_select(N.ptr(gains), l, N.ptr(selected), None, 0,
                      N.ptr(sel_idx), N.ptr(sel_gain), N.ptr(scratch), st)
    # all selected but one NaN-free candidate: that one is picked
    gains[3] = 1.0
    selected.fill_(1)
    selected[3] = 0
    lib.argmax_select(N.ptr(gains), l, N.ptr(selected), None, 1,
                      N.ptr(sel_idx), N.ptr(sel_gain), N.ptr(scratch), st)
    torch.cuda.synchronize()
    idx = sel_idx.cpu().numpy()
    assert idx[0] == -1 and idx[1] == 3
    assert int(selected.sum()) == l  # the sentinel marked nothing
    with pytest.raises(InvalidDataError):
        checked_picks(idx, 2)
    assert list(checked_picks(idx[1:], 1)) == [3]


@pytest.mark.parametrize("prec", [Precision.binary32, Precision.bfloat16,
                                  Precision.binary16, Precision.binary64])
def test_matrix_is_column_major(prec):
    g = pb.build_ground_set([[1.0, 2.0], [3.0, 4.0]], precision=prec)
    assert g.data.tolist() == [1.0, 3.0, 2.0, 4.0]
    assert g.matrix.flags.f_contiguous
    # a large row-major input: uploaded untransposed, transposed by K1 on
    # the device, matrix read back column-major -- same values and results
    rng = np.random.default_rng(5)
    V = rng.standard_normal((9000, 130)).astype(np.float32)
    assert V.flags.c_contiguous and V.size >= (1 << 20)
    g1 = pb.build_ground_set(V, precision=prec)
    g2 = pb.build_ground_set(np.asfortranarray(V), precision=prec)
    assert g1.matrix.flags.f_contiguous and not g1.matrix.flags.writeable
    assert g1.matrix.dtype == prec.dtype
    assert np.array_equal(g1.matrix.astype(np.float64),
                          g2.matrix.astype(np.float64))
    assert np.array_equal(g1.aux_distances, g2.aux_distances)
    assert g1.aux_loss == g2.aux_loss
    sel = g1.matrix[[3, 77, 4000]]
    assert pb.evaluate_single(g1, sel) == pb.evaluate_single(g2, sel)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _empty_shard_worker(rank, world, port, V, k, out):
    import torch
    import torch.distributed as dist

    from paper_2101_08763_b200.distributed import (build_sharded_ground,
                                                   sharded_greedy)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sg = build_sharded_ground(V, Precision.binary32, rank, world, device=0)
        picks, vals = sharded_greedy(sg, k)
        out[rank] = (sg.local is None, list(picks), list(vals))
    finally:
        dist.destroy_process_group()


def test_more_ranks_than_splits():
    import torch.multiprocessing as mp

    rng = np.random.default_rng(6)
    n, d, k, world = 2000, 16, 3, 3
    assert -(-n // int(N.lib().split_points(n))) < world
    V = rng.standard_normal((n, d)).astype(np.float32)
    g = pb.build_ground_set(V, precision=Precision.binary32)
    ref = pb.greedy_maximize(g, k=k)
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_empty_shard_worker,
                       args=(world, _free_port(), V, k, out), nprocs=world,
                       join=True, start_method="spawn")
    assert any(out[r][0] for r in range(world))  # some rank owned no rows
    for r in range(world):
        assert out[r][1] == list(ref.exemplar_indices)
        assert np.allclose(out[r][2], ref.values, rtol=1e-12, atol=1e-12)
