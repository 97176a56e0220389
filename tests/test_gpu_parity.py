"""Parity of the device path (through the C-ABI) with the reference.

Checked against (a) the golden vectors recorded from the reference itself
(tests/golden/) and (b) the pinned CPU oracle (oracle/exem_oracle.py) on the
same seeded inputs.  Tolerances are the parity contract of SURVEY.md 8(c):

  fp64   |f - ref| <= 1e-12 * max(1, |ref|)
  fp32   |f - ref| <= 1e-5 * max(1, |ref|) (+ 2 ulp32(aux_loss) vs the
         reference's own fp32 values, which carry that rounding)
  f16/bf16  vs the fp64 oracle on the identical stored inputs: the bounds of
         tests/contract.py (relative to max(1,|f|) and max(1,|G|)), and the
         reference's half bound 5e-2 vs binary32 (tests/test_evaluate.py:230-243).
"""

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import EvaluationBatch, Evaluator, Precision
from contract import (HALF_F_REL, HALF_G_REL, check_half_gains,
                      check_half_values, oracle_on_device_inputs, ulp32)
from spotcheck import teacher_forced_trajectory

pytestmark = pytest.mark.gpu

P16, BF16, P32, P64 = (Precision.binary16, Precision.bfloat16,
                       Precision.binary32, Precision.binary64)


def _sets(golden, key):
    card, idx = golden[key + "_card"], golden[key + "_idx"]
    out, pos = [], 0
    for c in card:
        out.append(idx[pos:pos + c])
        pos += c
    return out


def _close(vals, ref, tol, ulp_of=None):
    vals = np.asarray(vals, np.float64)
    ref = np.asarray(ref, np.float64)
    slack = 0.0 if ulp_of is None else 2 * float(np.spacing(np.float32(abs(ulp_of))))
    err = np.abs(vals - ref) - slack
    bound = tol * np.maximum(np.abs(ref), 1.0)
    assert np.all(err <= bound), (np.max(np.abs(vals - ref)), vals, ref)


# ------------------------------------------------------------------ hand cases
def test_hand_values(hand):
    g = pb.build_ground_set([[1.0], [3.0]], precision=P64)
    assert g.aux_loss == hand["line_aux_loss"]
    assert pb.evaluate_single(g, [[3.0]]) == hand["line_f3"]
    assert pb.evaluate_single(g, [[1.0]]) == hand["line_f1"]
    assert pb.evaluate_single(g, [[1.0], [3.0]]) == hand["line_f13"]
    assert pb.evaluate_single(g, []) == 0.0
    batch = EvaluationBatch.from_sets([[[3.0]], [[1.0]], [[1.0], [3.0]]])
    for name in pb.BACKENDS:
        assert pb.evaluate_batch(Evaluator(name), g, batch).tolist() == hand["line_batch"]
    r1, r2 = pb.greedy_maximize(g, k=1), pb.greedy_maximize(g, k=2)
    assert [list(r1.exemplar_indices), list(r1.values), r1.evaluations] == hand["line_greedy1"]
    assert [list(r2.exemplar_indices), list(r2.values), r2.evaluations] == hand["line_greedy2"]
    tie = pb.build_ground_set([[2.0], [2.0], [1.0]], precision=P64)
    assert list(pb.greedy_maximize(tie, k=1).exemplar_indices) == hand["tie_greedy1"]
    z = pb.build_ground_set([[0.0], [2.0]], precision=P64)
    assert pb.evaluate_single(z, [[2.0]]) == hand["zero2_f2"]
    a = pb.build_ground_set([[1.0]], aux=[2.0], precision=P64)
    assert a.aux_loss == hand["custom_aux_loss"]
    assert pb.kmedoids_loss(g, [[0.0]]) == hand["kmedoids_line_0"]
    assert [pb.point_loss(g, 0, [[3.0]]), pb.point_loss(g, 1, [[3.0]])] == hand["point_loss_line"]
    assert [pb.marginal_gain(g, [], [[3.0]]),
            pb.marginal_gain(g, [[3.0]], [[1.0]])] == hand["marginal_line"]
    assert pb.marginal_gain(g, [[3.0]], [[3.0]]) == 0.0
    g4 = pb.build_ground_set([[0.0], [1.0], [9.0], [10.0]], precision=P64)
    assert pb.assign_clusters(g4, [[0.5], [9.5]]).tolist() == hand["assign_hand"]
    g5 = pb.build_ground_set([[5.0]], precision=P64)
    assert pb.assign_clusters(g5, [[4.0], [6.0]]).tolist() == [0]


def test_errors_on_device_path():
    g = pb.build_ground_set([[1.0]])
    with pytest.raises(pb.DimensionMismatchError):
        pb.evaluate_single(g, [[1.0, 2.0]])
    with pytest.raises(ValueError):
        pb.evaluate_batch(Evaluator(precision=P64), g,
                          EvaluationBatch.from_sets([[[1.0]]]))
    with pytest.raises(pb.BudgetExceedsGroundSetError):
        pb.greedy_maximize(g, k=2)
    assert pb.greedy_maximize(g, k=0).exemplar_indices == ()
    with pytest.raises(pb.EmptyEvaluationSetError):
        pb.kmedoids_loss(g, [])
    with pytest.raises(pb.EmptyEvaluationSetError):
        pb.assign_clusters(g, [])
    with pytest.raises(IndexError):
        pb.point_loss(g, 1, [[1.0]])
    with pytest.raises(pb.OutOfMemoryError):
        pb.evaluate_chunked(Evaluator(), g, EvaluationBatch.from_sets([[[1.0]]]), budget=1)


# ------------------------------------------------------------------ golden
@pytest.mark.parametrize("tag,prec,tol", [("f64", P64, 1e-12), ("f32", P32, 1e-5)])
def test_random_instances_vs_reference(golden, tag, prec, tol):
    for it in range(12):
        key = f"rand_{tag}_{it}"
        g = pb.build_ground_set(golden[key + "_data"], precision=prec)
        ref_aux = golden[key + "_auxd"]
        _close(g.aux_distances, ref_aux, tol)
        _close([g.aux_loss], golden[key + "_auxloss"], tol)
        idx = _sets(golden, key)
        batch = EvaluationBatch.from_sets([g.matrix[i] for i in idx])
        vals = pb.evaluate_batch(Evaluator(), g, batch)
        assert vals.dtype == prec.accumulate_dtype
        ref = golden[key + "_vals"]
        _close(vals, ref, tol, None if tag == "f64" else g.aux_loss)
        for j, i in enumerate(idx):
            _close([pb.evaluate_single(g, g.matrix[i])], [ref[j]], tol,
                   None if tag == "f64" else g.aux_loss)
        _close(pb.min_distances(g, g.matrix[idx[0]]), golden[key + "_mind0"], tol)
        assert np.array_equal(pb.assign_clusters(g, g.matrix[idx[0]]),
                              golden[key + "_labels0"])


@pytest.mark.parametrize("key,k,prec", [
    ("g_u64", 5, P64), ("g_u32", 6, P32), ("g_n32", 6, P32), ("g_n64", 6, P64),
    ("g_n32d100", 4, P32),
])
def test_greedy_vs_reference(golden, key, k, prec):
    g = pb.build_ground_set(golden[key + "_data"], precision=prec)
    res = pb.greedy_maximize(g, k=k)
    assert list(res.exemplar_indices) == golden[key + "_picks"].tolist()
    assert res.evaluations == int(golden[key + "_evals"][0])
    tol = 1e-12 if prec is P64 else 1e-5
    _close(res.values, golden[key + "_values"], tol,
           None if prec is P64 else g.aux_loss)


def test_c1_greedy_and_single_set(golden):
    if "c1_f32_picks" not in golden:
        pytest.skip("C1 fixture not generated")
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_golden import c1_data, sha

    V, S = c1_data()
    assert sha(V) == str(golden["c1_sha"][0])
    for tag, prec, tol in (("f32", P32, 1e-5), ("f64", P64, 1e-12)):
        g = pb.build_ground_set(V, precision=prec)
        _close([g.aux_loss], golden[f"c1_{tag}_auxloss"], tol)
        _close([pb.evaluate_single(g, g.matrix[S])], golden[f"c1_{tag}_fS"], tol,
               None if tag == "f64" else g.aux_loss)
        res = pb.greedy_maximize(g, k=10)
        assert list(res.exemplar_indices) == golden[f"c1_{tag}_picks"].tolist()
        _close(res.values, golden[f"c1_{tag}_values"], tol,
               None if tag == "f64" else g.aux_loss)


# ------------------------------------------------------------------ properties
def test_determinism_and_chunking_bit_identical():
    rng = np.random.default_rng(53)
    data = rng.standard_normal((3000, 24))
    g = pb.build_ground_set(data, precision=P32)
    sets = [g.matrix[np.sort(rng.choice(3000, size=int(rng.integers(1, 9)),
                                        replace=False))] for _ in range(300)]
    batch = EvaluationBatch.from_sets(sets)
    ev = Evaluator()
    first = pb.evaluate_batch(ev, g, batch)
    for _ in range(2):
        assert np.array_equal(first, pb.evaluate_batch(ev, g, batch))
    mu = pb.estimate_set_memory(g.n, batch.k_max, batch.d, g.precision)
    for size in (300, 129, 128, 7, 1):
        assert np.array_equal(pb.evaluate_chunked(ev, g, batch, budget=mu * size), first)
    same = pb.evaluate_batch(ev, g, EvaluationBatch.from_sets([sets[0]] * 9))
    assert np.all(same == same[0])


def test_blank_slots_never_read():
    rng = np.random.default_rng(71)
    g = pb.build_ground_set(rng.random((250, 3)), precision=P32)
    sets = [g.matrix[:1]] + [g.matrix[rng.choice(250, 5, replace=False)] for _ in range(4)]
    batch = EvaluationBatch.from_sets(sets)
    packed = pb.pack_batch(batch, g.precision)
    assert packed.blank_slots > 0
    base = pb.tiled_evaluate(g, packed)
    poisoned = packed.values.copy()
    cube = poisoned.reshape(packed.d, packed.k_max, packed.l)
    for j, c in enumerate(packed.cardinalities):
        cube[:, c:, j] = 1e9
    import dataclasses

    assert np.array_equal(pb.tiled_evaluate(g, dataclasses.replace(packed, values=poisoned)), base)
    out, loads = pb.tiled_evaluate(g, packed, instrument=True)
    assert np.array_equal(out, base) and loads.shape == (g.n,)


@pytest.mark.parametrize("prec", [P32, P64])
def test_random_vs_oracle_large_sets(prec):
    """K4 at sizes with several splits and set tiles vs the pinned oracle."""
    rng = np.random.default_rng(7)
    n, d = 20_000, 37
    data = rng.standard_normal((n, d))
    g = pb.build_ground_set(data, precision=prec)
    og = O.Ground(data, prec.dtype)
    sets = [g.matrix[np.sort(rng.choice(n, size=int(rng.integers(1, 12)), replace=False))]
            for _ in range(260)]
    vals = pb.evaluate_batch(Evaluator(), g, EvaluationBatch.from_sets(sets))
    ref = O.evaluate_batch(og, sets[:40])
    tol = 1e-12 if prec is P64 else 1e-5
    _close(vals[:40], ref, tol, None if prec is P64 else g.aux_loss)


def test_submodular_and_monotone_on_device():
    rng = np.random.default_rng(77)
    data = rng.random((40, 5))
    g = pb.build_ground_set(data, precision=P64)
    for _ in range(100):
        a = int(rng.integers(0, 8))
        b = int(rng.integers(0, 8))
        perm = rng.permutation(40)
        A, B, e = data[perm[:a]], data[perm[:a + b]], data[perm[a + b]]
        fa, fb = pb.exemplar_value(g, A), pb.exemplar_value(g, B)
        scale = max(1.0, abs(fb))
        assert fa <= fb + 1e-12 * scale
        assert pb.marginal_gain(g, A, e) >= pb.marginal_gain(g, B, e) - 1e-12 * scale


def test_greedy_guarantee_vs_brute_force():
    rng = np.random.default_rng(113)
    factor = 1.0 - np.exp(-1.0)
    for _ in range(10):
        n = int(rng.integers(4, 13))
        k = int(rng.integers(1, 4))
        g = pb.build_ground_set(rng.random((n, 2)), precision=P64)
        greedy = pb.greedy_maximize(g, k=k)
        best, opt = pb.brute_force_optimum(g, k)
        assert len(best) == k
        assert greedy.values[-1] >= factor * opt - 1e-12
    with pytest.raises(pb.InstanceTooLargeError):
        pb.brute_force_optimum(pb.build_ground_set(rng.random((64, 1))), 32)


def test_greedy_memory_budget_identical():
    rng = np.random.default_rng(109)
    g = pb.build_ground_set(rng.standard_normal((2000, 8)), precision=P64)
    base = pb.greedy_maximize(g, k=4)
    budget = 600 * pb.estimate_set_memory(2000, 4, 8, P64)
    chunked = pb.greedy_maximize(g, k=4, memory_budget=budget)
    assert chunked.exemplar_indices == base.exemplar_indices
    assert chunked.values == base.values
    with pytest.raises(pb.OutOfMemoryError):
        pb.greedy_maximize(g, k=2, memory_budget=10)


def test_greedy_select_all_and_tiny_shapes():
    g = pb.build_ground_set([[0.5]], precision=P32)
    r = pb.greedy_maximize(g, k=1)
    assert r.exemplar_indices == (0,) and r.values == (g.aux_loss,)
    rng = np.random.default_rng(3)
    g = pb.build_ground_set(rng.random((7, 1)), precision=P64)
    r = pb.greedy_maximize(g, k=7)
    assert sorted(r.exemplar_indices) == list(range(7))
    assert abs(r.values[-1] - g.aux_loss) <= 1e-12 * max(1, g.aux_loss)


# ------------------------------------------------------------------ SIMT gains
@pytest.mark.parametrize("prec,n,d", [(P32, 20_000, 100), (P64, 6000, 16), (P32, 5000, 2),
                                      (P64, 2500, 48)])
def test_greedy_simt_matches_fp64_truth(prec, n, d):
    """K3-SIMT gains and the whole Greedy trajectory vs the fp64 oracle in
    the incremental form on the same (storage-rounded) inputs."""
    rng = np.random.default_rng(n + d)
    data = rng.standard_normal((n, d)).astype(prec.dtype)
    g = pb.build_ground_set(data, precision=prec)
    k = 3
    res = pb.greedy_maximize(g, k=k)
    picks, vals, gains = O.greedy_m(data.astype(np.float64), k)
    tol = 1e-12 if prec is P64 else 1e-5
    for t in range(k):
        top2 = np.sort(gains[t])[-2:]
        if res.exemplar_indices[t] != picks[t]:
            # a documented near-tie: both gains equal within fp32 tolerance
            assert abs(gains[t][res.exemplar_indices[t]] - top2[1]) <= tol * n
            break
    else:
        _close(res.values, vals, tol, None if prec is P64 else g.aux_loss)


# ------------------------------------------------------------------ half / TC
def _half_round(data, prec):
    return np.asarray(data, np.float32).astype(prec.dtype).astype(np.float64)


@pytest.mark.parametrize("prec", [P16, BF16])
def test_half_batch_vs_binary32_and_oracle(golden, prec):
    data = golden["half_data"]
    gh = pb.build_ground_set(data, precision=prec)
    sets = list(golden["half_idx"])
    vh = pb.evaluate_batch(Evaluator(), gh, EvaluationBatch.from_sets([gh.matrix[i] for i in sets]))
    # the reference's own half bound vs binary32 (test_evaluate.py:230-243)
    np.testing.assert_allclose(vh, golden["half_vals32"], rtol=5e-2, atol=5e-2)
    # tight: vs fp64 on the identical inputs (tests/contract.py)
    x = _half_round(data, prec)
    assert np.array_equal(gh.matrix.astype(np.float64), x)
    og = oracle_on_device_inputs(gh)
    ref = O.evaluate_batch(og, [og.matrix[i] for i in sets])
    check_half_values(gh, vh, ref, label=f"golden half batch {prec.name}")
    # f16 rounds aux_loss to binary16 like the reference (core.py:307-309)
    og = O.Ground(x, np.float64)
    assert abs(gh.aux_loss - og.aux_loss) <= 2 * np.spacing(
        np.asarray(og.aux_loss, prec.dtype if prec is P16 else np.float32))


@pytest.mark.parametrize("prec", [BF16, P16])
@pytest.mark.parametrize("n,d", [(3000, 100), (1000, 2), (2000, 16), (600, 512), (300, 1024), (700, 250)])
def test_tc_greedy_gains_vs_fp64(prec, n, d):
    """K3-TC (tcgen05) gains vs fp64 truth on the same half-rounded inputs,
    covering A-stationary (d <= 250) and A-streaming (d >= 512) modes."""
    from paper_2101_08763_b200.optimize import GreedyRun

    rng = np.random.default_rng(d * 7 + n)
    data = rng.standard_normal((n, d)) * (0.5 if prec is P16 else 1.0)
    g = pb.build_ground_set(data, precision=prec)
    x = g.matrix.astype(np.float64)
    dg = g.on_device()
    run = GreedyRun(dg, k_cap=2)
    run.start()
    run.compute_gains()
    G = run.gains.cpu().numpy()
    m = g.aux_distances.astype(np.float64)
    ref = O.gains_m(x, m, x)
    check_half_gains(G, ref, label=f"K3-TC {prec.name} n={n} d={d} step 1")
    # one step later (m updated through K2 + the folded -h refresh)
    run.select(0)
    run.update(0)
    c = int(run.sel_idx[0].item())
    assert c == int(np.argmax(G))
    run.compute_gains()
    G2 = run.gains.cpu().numpy()
    m2 = np.minimum(m, ((x - x[c]) ** 2).sum(1))
    ref2 = O.gains_m(x, m2, x)
    G2[c] = ref2[c]  # the selected candidate's gain is not used
    check_half_gains(G2, ref2, label=f"K3-TC {prec.name} n={n} d={d} step 2")


@pytest.mark.parametrize("prec", [BF16, P16])
def test_tc_greedy_trajectory(prec):
    rng = np.random.default_rng(5)
    n, d, k = 4000, 100, 5
    data = rng.standard_normal((n, d)) * (0.5 if prec is P16 else 1.0)
    g = pb.build_ground_set(data, precision=prec)
    res = pb.greedy_maximize(g, k=k)
    # every step teacher-forced against fp64 truth on the stored inputs: a
    # near-tie (pick within the gain tolerance of the maximum) does not end
    # the comparison
    slack = 2 * ulp32(g.aux_loss)
    teacher_forced_trajectory(
        g, res, lambda G: HALF_G_REL * max(1.0, abs(G)),
        lambda f: HALF_F_REL * max(1.0, abs(f)) + slack,
        label=f"K3-TC trajectory {prec.name}")


@pytest.mark.parametrize("prec", [P32, P64, P16, BF16])
def test_tiled_evaluate_matches_evaluate_batch(prec):
    """PackedBatch.values uploaded raw and widened/padded on the device
    (exem_widen_packed) vs the sets interleaved on the device
    (exem_pack_elements): the same packed layout, so tiled_evaluate and
    evaluate_batch agree bit for bit (the reference's backend equivalence,
    tests/test_acceptance.py:46-71)."""
    rng = np.random.default_rng(13)
    g = pb.build_ground_set(rng.standard_normal((3000, 29)) *
                            (0.5 if prec is P16 else 1.0), precision=prec)
    sets = [g.matrix[rng.choice(3000, int(rng.integers(1, 40)), replace=False)]
            for _ in range(77)]
    batch = EvaluationBatch.from_sets(sets)
    a = pb.evaluate_batch(Evaluator(), g, batch)
    b = pb.tiled_evaluate(g, pb.pack_batch(batch, g.precision))
    assert np.array_equal(a, b)


def test_aux_loss_within_one_step_all_members():
    """Reference test_core.py:95-102 for every member including the added
    bfloat16 (its epsilon from ml_dtypes.finfo: np.finfo rejects it)."""
    import ml_dtypes

    rng = np.random.default_rng(3)
    data = rng.random((100, 5))
    for precision in pb.Precision:
        g = pb.build_ground_set(data, precision=precision)
        exact = float(np.mean(np.asarray(g.aux_distances, dtype=np.float64)))
        eps = float(ml_dtypes.finfo(precision.dtype).eps)
        assert g.aux_loss == pytest.approx(exact, rel=4 * eps), precision


def test_point_loss_decomposition_within_fp64_bound():
    """Reference test_objective.py:155-164 at the fp64 parity bound: the
    per-point losses recompose the whole loss (the device sums in its own
    fixed order, so equality is to rounding, not bitwise)."""
    rng = np.random.default_rng(23)
    data = rng.random((50, 4))
    g = pb.build_ground_set(data, precision=pb.Precision.binary64)
    for _ in range(10):
        idx = rng.choice(50, size=4, replace=False)
        elems = g.matrix[idx]
        parts = np.array([pb.point_loss(g, i, elems) for i in range(50)])
        whole = pb.kmedoids_loss(g, np.vstack([elems, np.zeros((1, 4))]))
        assert abs(float(np.sum(parts)) - whole) <= 1e-12 * max(1.0, abs(whole))


@pytest.mark.parametrize("prec", [BF16, P16])
@pytest.mark.parametrize("d", [2, 8, 16, 26, 27])
@pytest.mark.parametrize("bn", ["256", "128"])
def test_tc_greedy_small_d(prec, d, bn, monkeypatch):
    """Small d: one or two K = 16 MMAs per tile (d <= 26; d = 27 is the
    first three-step shape), with the shipped 256-point tiles and the
    128-point / four-TMEM-buffer experiment layout (EXEM_TC_BN = 128), both
    teacher-forced against fp64 truth, with the epilogue width chosen per
    run (clustered data makes the screens fire)."""
    if bn != "256":
        monkeypatch.setenv("EXEM_TC_BN", bn)
    rng = np.random.default_rng(d)
    n, k = 5000, 6
    centres = rng.standard_normal((8, d)) * 3.0
    data = centres[rng.integers(0, 8, n)] + rng.standard_normal((n, d))
    data *= 0.5 if prec is P16 else 1.0
    g = pb.build_ground_set(data, precision=prec)
    res = pb.greedy_maximize(g, k=k)
    slack = 2 * ulp32(g.aux_loss)
    teacher_forced_trajectory(
        g, res, lambda G: HALF_G_REL * max(1.0, abs(G)),
        lambda f: HALF_F_REL * max(1.0, abs(f)) + slack,
        label=f"K3-TC small d={d} {prec.name} bn={bn}")
