"""K2 (single explicit set) over every thread layout of the TMA kernel
(csrc/exem_setmin.cu): EG lanes x ET elements for k = 1..64 at binary32 and
k = 1..32 at binary64, several element groups carried through t_out for
larger k, and the cp.async kernel where the element group does not fit
(large d) -- against the oracle's restatement of the reference
(objective.py:113-141 min_distances, evaluate.py:105-112 _set_value,
optimize.py:115-136 assign_clusters).

Distances differ from the reference's BLAS op order only by rounding, so:
per-point minima within the precision's distance tolerance, labels equal
wherever the reference's two best elements are not a near-tie, f(S) within
the parity contract.
"""

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb

pytestmark = pytest.mark.gpu

P32, P64 = pb.Precision.binary32, pb.Precision.binary64
K32 = [1, 2, 3, 5, 8, 9, 12, 16, 17, 24, 31, 33, 40, 50, 57, 64, 65, 100, 150]
K64 = [1, 4, 8, 9, 16, 17, 25, 32, 33, 50, 70]


def _tol(prec):
    return 1e-12 if prec is P64 else 2e-5


def _case(prec, n, d, k, seed):
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((n, d))
    g = pb.build_ground_set(V, precision=prec)
    idx = np.sort(rng.choice(n, size=k, replace=False))
    og = O.Ground(np.asarray(g.matrix, np.float64), np.float64)
    return g, og, idx


def _check(g, og, idx, prec):
    elems = g.matrix[idx]
    t = pb.min_distances(g, elems)
    t_ref = O.min_distances(og, og.matrix[idx])
    # the GEMM form ||v||^2 + ||e||^2 - 2 v.e (reference objective.py:83-89)
    # cancels to ~eps * (||v||^2 + ||e||^2) at a point's own element, so the
    # scale is the norms (aux = ||v||^2 for e0 = 0), not the distance
    scale = np.maximum(1.0, np.maximum(np.abs(t_ref), og.aux_distances))
    assert np.all(np.abs(t.astype(np.float64) - t_ref) <= 4 * _tol(prec) * scale)
    # labels: equal unless the reference's two nearest elements tie closely
    lab = pb.assign_clusters(g, elems)
    D = O._d64(og.matrix, og.matrix[idx])
    ref = np.argmin(D, axis=1)
    if D.shape[1] > 1:
        part = np.partition(D, 1, axis=1)
        gap = (part[:, 1] - part[:, 0]) / np.maximum(1.0, part[:, 0])
        clear = gap > 8 * _tol(prec)
    else:
        clear = np.ones(len(ref), bool)
    assert np.array_equal(lab[clear], ref[clear])
    # f(S) through the public single-set evaluate
    f = pb.evaluate_single(g, elems)
    f_ref = O.set_value(og, og.matrix[idx])
    assert abs(f - f_ref) <= 2 * _tol(prec) * max(1.0, abs(f_ref)) + \
        2 * float(np.spacing(np.float32(g.aux_loss)))


@pytest.mark.parametrize("k", K32)
def test_set_min_layouts_f32(k):
    g, og, idx = _case(P32, 3001, 37, k, seed=k)
    _check(g, og, idx, P32)


@pytest.mark.parametrize("k", K64)
def test_set_min_layouts_f64(k):
    g, og, idx = _case(P64, 2003, 21, k, seed=100 + k)
    _check(g, og, idx, P64)


@pytest.mark.parametrize("prec,k,d", [(P32, 64, 700), (P64, 32, 600)])
def test_set_min_large_d_fallback(prec, k, d):
    """Element groups too large for shared memory take the cp.async K2."""
    g, og, idx = _case(prec, 1500, d, k, seed=d)
    _check(g, og, idx, prec)


@pytest.mark.parametrize("prec", [pb.Precision.bfloat16, pb.Precision.binary16])
@pytest.mark.parametrize("k", [1, 7, 20, 50])
def test_set_min_half_storage(prec, k):
    """Half storage: the direct-form distance in fp32 on the exact half
    values, against the fp64 oracle on the same rounded inputs."""
    import ml_dtypes

    g, og, idx = _case(prec, 2500, 48, k, seed=7 * k)
    t = pb.min_distances(g, g.matrix[idx])  # returned in the storage dtype
    t_ref = O.min_distances(og, og.matrix[idx])
    eps = float(ml_dtypes.finfo(prec.dtype).eps)  # one rounding to storage
    assert np.all(np.abs(t.astype(np.float64) - t_ref) <=
                  eps * np.maximum(1.0, np.abs(t_ref)))


def test_set_min_deterministic_and_streamed_equal():
    """Bit-identical on repeat and through the streamed (low-memory) path:
    the canonical per-256-point block partials of the TMA kernel."""
    rng = np.random.default_rng(3)
    V = rng.standard_normal((300_000, 40)).astype(np.float32)
    g = pb.build_ground_set(V, precision=P32)
    gs = pb.build_ground_set(V, precision=P32, device_budget=40 << 20)
    assert gs.streamed
    for k in (1, 10, 50):
        elems = g.matrix[rng.choice(len(V), size=k, replace=False)]
        a = pb.evaluate_single(g, elems)
        assert pb.evaluate_single(g, elems) == a
        assert pb.evaluate_single(gs, elems) == a


@pytest.mark.parametrize("n,d", [(1, 1), (2, 3), (255, 8), (256, 5), (257, 17),
                                 (513, 2)])
@pytest.mark.parametrize("k", [1, 3, 20])
def test_set_min_tiny_shapes(n, d, k):
    """Ragged last tiles, n below one 256-point tile, d = 1."""
    k = min(k, n)
    g, og, idx = _case(P32, n, d, k, seed=n * 31 + d + k)
    _check(g, og, idx, P32)
