"""Size-independent properties at BASELINE sizes (the oracle cannot run them
in seconds, so parity there is checked through the domain's invariants).

C4 (n = 1M, d = 100, bf16 tensor path and fp32 SIMT path, a few Greedy
steps): picks distinct; values non-decreasing (monotone f, SPEC); each
recorded value equals the single-set evaluation f(S_t) recomputed by a
different kernel (K2 over the explicit set) within the half / fp32 bound;
the value increments equal the picked candidates' gains divided by n
(K3 vs K2 agree); the fp64 gain of the pick -- recomputed on the host for a
sample of points -- is consistent.
C5-like (n = 4M points, d = 256, bf16, l = 256 sets of 50): streamed through
a small budget == resident, bit for bit, and invariant to set chunking.
"""

import numpy as np
import pytest

import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import EvaluationBatch, Evaluator, Precision
from paper_2101_08763_b200 import streaming as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,tol", [(Precision.bfloat16, 2e-4),
                                      (Precision.binary32, 1e-5)])
def test_c4_greedy_invariants(prec, tol):
    n, d, k = 1_000_000, 100, 4 if prec is Precision.bfloat16 else 2
    V = np.random.default_rng(0).standard_normal((n, d), dtype=np.float32)
    g = pb.build_ground_set(V, precision=prec)
    res = pb.greedy_maximize(g, k=k)
    picks, vals = list(res.exemplar_indices), np.array(res.values)
    assert len(set(picks)) == k
    assert np.all(np.diff(vals) >= -tol * max(1.0, abs(vals[-1])))
    assert res.evaluations == sum(n - t for t in range(k))
    for t in range(k):
        f = pb.evaluate_single(g, g.matrix[picks[: t + 1]])
        assert abs(f - vals[t]) <= tol * max(1.0, abs(vals[t])), (t, f, vals[t])
    # the first pick's gain, recomputed in fp64 on the host from the stored
    # values, equals n * f(S_1) (m starts at aux = ||v||^2 with e0 = 0)
    x = g.matrix.astype(np.float64)
    c = x[picks[0]]
    m0 = (x * x).sum(1)
    dist = ((x - c) ** 2).sum(1)
    gain = np.maximum(0.0, m0 - dist).sum()
    slack = 2 * float(np.spacing(np.float32(g.aux_loss)))  # aux_loss storage
    assert abs(gain / n - vals[0] + (g.aux_loss - m0.sum() / n)) <= \
        tol * max(1.0, abs(vals[0])) + slack


def test_c5_scale_streamed_bit_identical_and_chunk_invariant():
    n, d, l, card = 4_000_000, 256, 256, 50
    rng = np.random.default_rng(5)
    V = np.empty((n, d), dtype=Precision.bfloat16.dtype, order="F")
    for a in range(0, n, 1 << 20):
        b = min(n, a + (1 << 20))
        V[a:b] = rng.standard_normal((b - a, d), dtype=np.float32).astype(V.dtype)
    sets = rng.standard_normal((l, card, d), dtype=np.float32).astype(V.dtype)
    batch = EvaluationBatch.from_sets(list(sets))
    gr = pb.build_ground_set(V, precision=Precision.bfloat16)
    ref = pb.evaluate_batch(Evaluator(), gr, batch)
    del gr
    budget = S.resident_bytes(n, d, Precision.bfloat16) // 6
    gs = pb.build_ground_set(V, precision=Precision.bfloat16, device_budget=budget)
    assert gs.streamed
    assert np.array_equal(pb.evaluate_batch(Evaluator(), gs, batch), ref)
    mu = pb.estimate_set_memory(n, card, d, Precision.bfloat16)
    assert np.array_equal(
        pb.evaluate_chunked(Evaluator(), gs, batch, budget=mu * 100), ref)
    # monotone in the set: adding elements never lowers f (SPEC, submodular f)
    sub = EvaluationBatch.from_sets([s[:10] for s in sets[:8]])
    small = pb.evaluate_batch(Evaluator(), gs, sub)
    assert np.all(ref[:8] >= small - 2e-4 * np.maximum(1.0, np.abs(ref[:8])))
