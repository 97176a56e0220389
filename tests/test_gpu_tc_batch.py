"""K4-TC (tcgen05 explicit-set batch kernel, exem_tc_batch.cu) parity.

Half-precision batches (binary16 / bfloat16, k_max <= 256) are evaluated on
tensor cores.  Compared with the fp64 oracle on the identical half-rounded
inputs (the parity contract of SURVEY.md 8(c) for the half paths, stated in
tests/contract.py):

    |f_dev - f_ref| <= HALF_F_REL * max(1, |f_ref|) + 2 ulp32(aux_loss)

and the reference's own half bound (5e-2 vs binary32) through
test_gpu_parity.py.  Geometry cases cover: one set per tile (k_max = 256),
many sets per tile (k_max = 1 -> 32 sets; k_max <= 10 runs the 17-32
set-per-tile kernel), ragged
cardinalities (blank slots), l not a multiple of the sets per tile, n not a
multiple of the 128-point tile with several partial-sum splits, the
stationary set tile with whole / per-chunk point stages (d <= 256) and the
streamed set tile (d = 700).
"""

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import EvaluationBatch, Evaluator, Precision
from paper_2101_08763_b200 import evaluate as E
from contract import check_half_values, oracle_on_device_inputs

pytestmark = pytest.mark.gpu

P16, BF16 = Precision.binary16, Precision.bfloat16


def _case(prec, n, d, l, kmin, kmax, seed):
    rng = np.random.default_rng(seed)
    scale = 0.5 if prec is P16 else 1.0
    data = rng.standard_normal((n, d)) * scale
    g = pb.build_ground_set(data, precision=prec)
    sets = [np.sort(rng.choice(n, size=int(rng.integers(kmin, kmax + 1)),
                               replace=False)) for _ in range(l)]
    return g, sets


def _check(g, sets, vals, nref=None, label="K4-TC"):
    og = oracle_on_device_inputs(g)
    sub = sets if nref is None else sets[:nref]
    ref = O.evaluate_batch(og, [og.matrix[i] for i in sub])
    check_half_values(g, vals[:len(sub)], ref,
                      label=f"{label} {g.precision.name} n={g.n} d={g.d}")


@pytest.mark.parametrize("prec", [BF16, P16])
@pytest.mark.parametrize("n,d,l,kmin,kmax", [
    (3000, 100, 150, 1, 50),      # ragged, 5 interleaved sets in N = 256
    (1000, 2, 70, 1, 1),          # k_max = 1: 32 sets in N = 32
    (2500, 16, 45, 8, 8),         # 32 sets of 8 in N = 256 (wide kernel)
    (4000, 100, 120, 10, 10),     # 25 sets of 10 in N = 256 (wide kernel)
    (3000, 64, 61, 2, 9),         # 28 sets of 9 (wide kernel, ragged)
    (3000, 64, 61, 2, 15),        # 16 sets of 15 (main kernel, ragged)
    (2000, 100, 40, 1, 16),       # 16 sets of 16: the main kernel
    (1300, 256, 20, 1, 256),      # one set per tile, per-chunk point stages
    (777, 700, 9, 3, 40),         # streamed set tile (d > stationary budget)
    (20_000, 37, 33, 1, 12),      # several splits, n % 128 != 0
])
def test_tc_batch_vs_fp64(prec, n, d, l, kmin, kmax):
    g, sets = _case(prec, n, d, l, kmin, kmax, seed=n + d + l)
    batch = EvaluationBatch.from_sets([g.matrix[i] for i in sets])
    assert E.tc_batch_supported(prec, batch.k_max)
    vals = pb.evaluate_batch(Evaluator(), g, batch)
    _check(g, sets, vals, nref=min(l, 40))


@pytest.mark.parametrize("prec", [BF16, P16])
def test_tc_batch_deterministic_and_chunk_invariant(prec):
    g, sets = _case(prec, 5000, 64, 200, 1, 30, seed=11)
    batch = EvaluationBatch.from_sets([g.matrix[i] for i in sets])
    ev = Evaluator()
    first = pb.evaluate_batch(ev, g, batch)
    assert np.array_equal(first, pb.evaluate_batch(ev, g, batch))
    mu = pb.estimate_set_memory(g.n, batch.k_max, batch.d, g.precision)
    for size in (200, 77, 8, 1):
        assert np.array_equal(
            pb.evaluate_chunked(ev, g, batch, budget=mu * size), first)
    # a set's value does not depend on its neighbours in the set tile
    same = pb.evaluate_batch(ev, g, EvaluationBatch.from_sets(
        [batch.sets[5]] * 11))
    assert np.all(same == first[5])


def test_tc_batch_blank_slots_and_duplicates():
    """Blank slots are copies of element 0 (never change a minimum); sets
    with repeated vectors equal the deduplicated set."""
    rng = np.random.default_rng(3)
    g = pb.build_ground_set(rng.standard_normal((900, 20)), precision=BF16)
    a = g.matrix[[4, 17, 300]]
    b = g.matrix[[4, 4, 17, 300, 300, 17]]
    c = g.matrix[[4]]
    li = rng.choice(900, 60, replace=False)
    vals = pb.evaluate_batch(Evaluator(), g,
                             EvaluationBatch.from_sets([a, b, c, g.matrix[li]]))
    assert vals[0] == vals[1]
    _check(g, [[4, 17, 300], [4, 17, 300], [4], li], vals)


def test_tc_batch_large_sets_use_simt_path():
    """k_max > 256 does not fit one TMEM tile: the SIMT K4 evaluates it."""
    rng = np.random.default_rng(5)
    g = pb.build_ground_set(rng.standard_normal((1200, 12)), precision=BF16)
    sets = [rng.choice(1200, 300, replace=False), rng.choice(1200, 5, replace=False)]
    batch = EvaluationBatch.from_sets([g.matrix[i] for i in sets])
    assert not E.tc_batch_supported(BF16, batch.k_max)
    vals = pb.evaluate_batch(Evaluator(), g, batch)
    _check(g, sets, vals)


@pytest.mark.parametrize("l", [1, 7, 23])
def test_tc_batch_multicast_clusters_identical(monkeypatch, l):
    """Point tiles shared by TMA multicast across clusters of 1, 2 or 4 CTAs
    (EXEM_TCB_MC; default 2) give bit-identical sums -- every (split, set)
    partial is still computed by one CTA in a fixed order -- including an odd
    number of set tiles (a cluster's spare tile is computed and dropped)."""
    g, sets = _case(BF16, 9000, 100, 50, 1, 50, seed=17)
    sets = (sets * 3)[:l * 5]
    batch = EvaluationBatch.from_sets([g.matrix[i] for i in sets])
    out = {}
    for mc in ("1", "2", "4"):
        monkeypatch.setenv("EXEM_TCB_MC", mc)
        out[mc] = pb.evaluate_batch(Evaluator(), g, batch)
    _check(g, sets, out["2"], nref=20)
    assert np.array_equal(out["1"], out["2"])
    assert np.array_equal(out["1"], out["4"])
