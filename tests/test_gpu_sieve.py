"""SieveStreaming over the device evaluator (paper_2101_08763_b200/sieve.py).

The reference has no streaming optimizer, so the checker is
the fp64 host restatement oracle/exem_oracle.py:sieve_streaming of the same
algorithm, plus the algorithm's own guarantee: f(S) >= (1/2 - eps) OPT >=
(1/2 - eps) f(Greedy)."""

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import Precision

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,k,eps", [(400, 3, 4, 0.2), (1500, 8, 6, 0.1),
                                       (3000, 20, 10, 0.1)])
def test_sieve_fp64_matches_oracle(n, d, k, eps):
    rng = np.random.default_rng(n + d)
    V = rng.random((n, d))
    g = pb.build_ground_set(V, precision=Precision.binary64)
    res = pb.sieve_streaming_maximize(g, k, eps=eps)
    picks, vals, evals = O.sieve_streaming(V, k, eps)
    assert res.exemplar_indices == picks
    assert np.allclose(res.values, vals, rtol=1e-12, atol=1e-12)
    assert res.evaluations == evals


@pytest.mark.parametrize("prec", [Precision.binary32, Precision.bfloat16])
def test_sieve_guarantee_vs_greedy(prec):
    rng = np.random.default_rng(9)
    V = rng.standard_normal((5000, 16))
    g = pb.build_ground_set(V, precision=prec)
    k, eps = 8, 0.1
    res = pb.sieve_streaming_maximize(g, k, eps=eps)
    greedy = pb.greedy_maximize(g, k=k)
    assert 1 <= len(res.exemplar_indices) <= k
    assert len(set(res.exemplar_indices)) == len(res.exemplar_indices)
    assert res.values[-1] >= (0.5 - eps) * greedy.values[-1]
    # the recorded value is f of the returned set
    f = pb.evaluate_single(g, g.matrix[list(res.exemplar_indices)])
    tol = 2e-4 if prec.is_half else 1e-5
    assert abs(f - res.values[-1]) <= tol * max(1.0, abs(f))


def test_sieve_argument_errors():
    g = pb.build_ground_set(np.random.default_rng(0).random((10, 2)))
    with pytest.raises(pb.BudgetExceedsGroundSetError):
        pb.sieve_streaming_maximize(g, 11)
    with pytest.raises(ValueError):
        pb.sieve_streaming_maximize(g, 2, eps=0.0)
    assert pb.sieve_streaming_maximize(g, 0).exemplar_indices == ()


@pytest.mark.parametrize("prec", [Precision.binary64, Precision.binary32])
def test_sieve_block_size_invariant(prec):
    """Block processing (one distance pass + one scoring launch per block,
    rescoring only a sieve that just grew) makes the element-at-a-time
    decisions: same picks and values for every block size, including a
    stream order that revisits nothing and ends mid-block."""
    rng = np.random.default_rng(4)
    V = rng.standard_normal((2500, 12))
    g = pb.build_ground_set(V, precision=prec)
    order = rng.permutation(2500)[:2333]
    ref = pb.sieve_streaming_maximize(g, 7, eps=0.15, order=order, block=1)
    for block in (5, 64, 300):
        res = pb.sieve_streaming_maximize(g, 7, eps=0.15, order=order,
                                          block=block)
        assert res.exemplar_indices == ref.exemplar_indices, block
        assert res.values == ref.values
        assert res.evaluations == ref.evaluations
