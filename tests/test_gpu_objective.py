"""The device ``Dissimilarity.distances`` (SQUARED_EUCLIDEAN.batch ->
exem_distance_matrix), ported from the reference's own contract tests
(/root/reference/pkg/tests/test_objective.py:40-57) plus parity with the
oracle's restatement of ``_squared_euclidean_batch`` (objective.py:75-90) at
every precision and at shapes that do not fill the 64 x 64 output tiles.
"""

import time

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import SQUARED_EUCLIDEAN, squared_euclidean
from paper_2101_08763_b200.errors import DimensionMismatchError
from spotcheck import log

pytestmark = pytest.mark.gpu


def test_batch_matches_pairwise():
    rng = np.random.default_rng(11)
    block, elems = rng.random((20, 6)), rng.random((5, 6))
    dmat = SQUARED_EUCLIDEAN.distances(block, elems)
    assert dmat.dtype == np.float64
    for a in range(20):
        for b in range(5):
            assert dmat[a, b] == pytest.approx(
                squared_euclidean(block[a], elems[b]), rel=1e-12)


def test_batch_non_negative_under_cancellation():
    base = np.full((4, 8), 1e6)
    dmat = SQUARED_EUCLIDEAN.distances(base, base[:2])
    assert np.all(dmat >= 0)
    f32 = SQUARED_EUCLIDEAN.distances(base.astype(np.float32),
                                      base[:2].astype(np.float32))
    assert np.all(f32 >= 0)


def test_batch_dim_mismatch():
    with pytest.raises(DimensionMismatchError):
        SQUARED_EUCLIDEAN.distances(np.zeros((2, 3)), np.zeros((2, 4)))


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5),
                                       (np.float16, 2e-3)])
@pytest.mark.parametrize("m,q,d", [(1, 1, 1), (63, 65, 7), (200, 130, 100),
                                   (8192, 50, 256), (70, 3, 1024)])
def test_distances_vs_oracle(dtype, tol, m, q, d):
    rng = np.random.default_rng(m * 7 + q + d)
    block = rng.standard_normal((m, d)).astype(dtype)
    elems = rng.standard_normal((q, d)).astype(dtype)
    got = SQUARED_EUCLIDEAN.distances(block, elems)
    assert got.dtype == np.dtype(dtype) and got.shape == (m, q)
    ref = O.sq_batch(block, elems).astype(np.float64)
    exact = O._d64(block, elems)
    # GEMM form (f32/f64) cancels like the reference's; the half direct form
    # accumulates wider (fp32 on exact half values) than the reference's
    # pairwise half sum, then rounds once to binary16
    scale = np.maximum(1.0, np.abs(exact))
    assert np.all(np.abs(got - ref) <= tol * scale)
    assert np.all(np.abs(got.astype(np.float64) - exact) <= tol * scale)
    assert np.all(got >= 0)


def test_distances_throughput():
    """The reference's block shape (8192 rows, objective.py:130-131) against a
    set of 64 elements at d = 100, fp32: the tiled kernel is FFMA-bound, so
    report its rate (logged; the bound is a sanity floor)."""
    import torch

    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.device import padded_rows

    m, q, d = 262_144, 256, 100
    rng = np.random.default_rng(1)
    a = rng.standard_normal((m, d), dtype=np.float32)
    b = rng.standard_normal((q, d), dtype=np.float32)
    lib = N.lib()
    prec = pb.Precision.binary32
    dev = torch.device("cuda", 0)
    d_pad = int(lib.pad_dims(d))
    A = padded_rows(a, d_pad, prec, dev)
    B = padded_rows(b, d_pad, prec, dev)
    an = torch.empty(m, dtype=torch.float64, device=dev)
    bn = torch.empty(q, dtype=torch.float64, device=dev)
    out = torch.empty((m, q), dtype=torch.float32, device=dev)
    st = N.stream_handle(dev)
    lib.row_norms(prec.tag, N.ptr(A), m, d, d_pad, N.ptr(an), st)
    lib.row_norms(prec.tag, N.ptr(B), q, d, d_pad, N.ptr(bn), st)

    def launch():
        lib.distance_matrix(prec.tag, N.ptr(A), N.ptr(an), m, N.ptr(B),
                            N.ptr(bn), q, d, d_pad, N.ptr(out), st)

    for _ in range(3):
        launch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(
        enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tflops = 2.0 * m * q * d / (ms / 1e3) / 1e12
    gbs = (m * q * 4 + m * d_pad * 4) / (ms / 1e3) / 1e9
    log({"check": "distance_matrix f32", "m": m, "q": q, "d": d, "ms": ms,
         "tflops": tflops, "out_gbs": gbs, "t": time.time()})
    # spot-check a few rows against the oracle
    rows = [0, 1, m // 2, m - 1]
    ref = O.sq_batch(a[rows], b)
    got = out[rows].cpu().numpy()
    assert np.all(np.abs(got - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref)))
    assert tflops > 5.0, tflops
