"""Pin the CPU oracle (oracle/exem_oracle.py) to the reference's own outputs.

The golden vectors were produced by running the unmodified reference
(tests/golden/make_golden.py).  If these pass, the oracle is a faithful
restatement and may be used as the checker for the device path.
"""

import numpy as np
import pytest

import exem_oracle as O


def _sets(golden, key):
    card = golden[key + "_card"]
    idx = golden[key + "_idx"]
    out, pos = [], 0
    for c in card:
        out.append(idx[pos:pos + c])
        pos += c
    return out


def test_hand_cases(hand):
    g = O.Ground([[1.0], [3.0]], np.float64)
    assert g.aux_loss == hand["line_aux_loss"] == 5.0
    assert O.set_value(g, [[3.0]]) == hand["line_f3"] == 4.5
    assert O.set_value(g, [[1.0]]) == hand["line_f1"]
    assert O.set_value(g, [[1.0], [3.0]]) == hand["line_f13"]
    assert O.evaluate_batch(g, [[[3.0]], [[1.0]], [[1.0], [3.0]]]).tolist() == hand["line_batch"]
    picks, vals = O.greedy(g, 2)
    assert [list(picks), list(vals)] == hand["line_greedy2"][:2]
    tie = O.Ground([[2.0], [2.0], [1.0]], np.float64)
    assert list(O.greedy(tie, 1)[0]) == hand["tie_greedy1"]
    assert O.Ground([[1.0]], np.float64, aux=[2.0]).aux_loss == hand["custom_aux_loss"]
    g4 = O.Ground([[0.0], [1.0], [9.0], [10.0]], np.float64)
    assert O.assign_clusters(g4, [[0.5], [9.5]]).tolist() == hand["assign_hand"]


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_random_instances_bitwise(golden, tag):
    dtype = np.float64 if tag == "f64" else np.float32
    for it in range(12):
        key = f"rand_{tag}_{it}"
        g = O.Ground(golden[key + "_data"], dtype)
        assert np.array_equal(g.aux_distances, golden[key + "_auxd"])
        assert g.aux_loss == golden[key + "_auxloss"][0]
        sets = [g.matrix[i] for i in _sets(golden, key)]
        vals = O.evaluate_batch(g, sets)
        # same numpy/BLAS in this image -> the restatement is bit-exact
        assert np.array_equal(vals, golden[key + "_vals"]), key
        assert np.array_equal(O.min_distances(g, sets[0]), golden[key + "_mind0"])
        assert np.array_equal(O.assign_clusters(g, sets[0]), golden[key + "_labels0"])


@pytest.mark.parametrize("key,k,dtype", [
    ("g_u64", 5, np.float64), ("g_u32", 6, np.float32),
    ("g_n32", 6, np.float32), ("g_n64", 6, np.float64),
])
def test_greedy_trajectories(golden, key, k, dtype):
    g = O.Ground(golden[key + "_data"], dtype)
    picks, vals = O.greedy(g, k)
    assert list(picks) == golden[key + "_picks"].tolist()
    assert np.array_equal(np.array(vals), golden[key + "_values"])


@pytest.mark.parametrize("key,k,dtype", [
    ("g_u64", 5, np.float64), ("g_n64", 6, np.float64), ("g_n32", 6, np.float32),
    ("g_n32d100", 4, np.float32),
])
def test_incremental_form_matches_reference_greedy(golden, key, k, dtype):
    """The device's optimizer-aware form (fp64 truth) picks what the
    reference picks; values agree to the parity contract."""
    data = np.asarray(golden[key + "_data"], dtype=dtype).astype(np.float64)
    picks, vals, _ = O.greedy_m(data, k)
    assert list(picks) == golden[key + "_picks"].tolist()
    ref = golden[key + "_values"]
    tol = 1e-12 if dtype == np.float64 else 1e-5
    ulp = 0.0 if dtype == np.float64 else 2 * np.spacing(np.float32(np.abs(ref).max() + 1))
    scale = np.maximum(np.abs(ref), 1.0)
    # reference fp32 f carries its own ~ulp(aux_loss) rounding
    assert np.all(np.abs(np.array(vals) - ref) <= tol * scale + ulp * 50)


def test_half_reference_fixture(golden):
    data = golden["half_data"]
    g16 = O.Ground(data, np.float16)
    g32 = O.Ground(data, np.float32)
    sets = list(golden["half_idx"])
    v16 = O.evaluate_batch(g16, [g16.matrix[i] for i in sets])
    v32 = O.evaluate_batch(g32, [g32.matrix[i] for i in sets])
    assert np.array_equal(v16, golden["half_vals16"])
    assert np.array_equal(v32, golden["half_vals32"])


@pytest.fixture(autouse=True, scope="module")
def _golden_path():
    import sys
    from pathlib import Path

    p = str(Path(__file__).resolve().parent / "golden")
    if p not in sys.path:
        sys.path.insert(0, p)
    yield


def test_c1_single_set_value(golden):
    if "c1_f32_fS" not in golden:
        pytest.skip("C1 fixture not generated")
    from make_golden import c1_data, sha

    V, S = c1_data()
    assert sha(V) == str(golden["c1_sha"][0]), "numpy RNG stream changed"
    for tag, dt in (("f32", np.float32), ("f64", np.float64)):
        g = O.Ground(V, dt)
        assert O.set_value(g, g.matrix[S]) == golden[f"c1_{tag}_fS"][0]
        assert g.aux_loss == golden[f"c1_{tag}_auxloss"][0]
