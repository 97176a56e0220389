"""Benchmark records in the reference's CSV schema (paper_2101_08763_b200/
bench.py), mirroring pkg/tests/test_bench.py: schema and round trip,
speedup pairing rules, the R^2 helper, generation outside the timed region
(noop backend) -- and that ``generate_problem`` draws exactly the
reference's problem (golden: the reference's own generator, run here)."""

import math

import numpy as np
import pytest

import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import bench as B


def _rec(**kw):
    base = dict(vary="n", n=100, l=5, k=2, d=3, precision="binary32",
                backend="b200", workers=1, seed=0, repetitions=3,
                runtime_seconds=0.5)
    base.update(kw)
    return B.BenchRecord(**base)


def test_csv_schema_and_round_trip(tmp_path):
    assert B.CSV_FIELDS == ("vary", "n", "l", "k", "d", "precision", "backend",
                            "workers", "seed", "repetitions", "runtime_seconds")
    recs = [_rec(), _rec(n=200, runtime_seconds=float("nan"))]
    p = tmp_path / "r.csv"
    B.write_csv(recs, p)
    back = B.read_csv(p)
    assert back[0] == recs[0] and back[1].failed and not back[0].failed
    assert p.read_text().splitlines()[0] == ",".join(B.CSV_FIELDS)


def test_speedup_rules():
    assert B.compute_speedup(_rec(runtime_seconds=2.0), _rec(runtime_seconds=0.5)) == 4.0
    with pytest.raises(pb.IncomparableRecordsError):
        B.compute_speedup(_rec(), _rec(n=7))


def test_linear_fit_r2():
    assert B.linear_fit_r2([1, 2, 3], [2, 4, 6]) == pytest.approx(1.0)
    assert B.linear_fit_r2([1, 2, 3], [5, 5, 5]) == 1.0
    assert B.linear_fit_r2([1, 2, 3, 4], [1, 3, 2, 4]) < 1.0


def test_argument_validation():
    with pytest.raises(ValueError):
        B.run_benchmark("x", [1])
    with pytest.raises(ValueError):
        B.run_benchmark("n", [])
    with pytest.raises(ValueError):
        B.run_benchmark("n", [10], repetitions=0)
    with pytest.raises(ValueError):
        B.generate_problem(0, 1, 1, 1, 0)
    with pytest.raises(pb.BudgetExceedsGroundSetError):
        B.generate_problem(3, 1, 4, 1, 0)


@pytest.mark.parametrize("tag,prec", [("32", pb.Precision.binary32),
                                      ("64", pb.Precision.binary64),
                                      ("16", pb.Precision.binary16)])
def test_generator_draws_the_reference_problem(golden, tag, prec):
    """Same seed -> the reference's generate_problem values and sets
    (recorded from the reference itself in tests/golden/make_golden.py)."""
    values, idx = B.draw_problem(50, 4, 3, 5, 11, prec)
    stored = np.asarray(values).astype(prec.dtype)
    assert np.array_equal(stored, golden[f"gen{tag}_values"])
    assert np.array_equal(stored[idx], golden[f"gen{tag}_sets"])


@pytest.mark.gpu
def test_run_benchmark_on_device(tmp_path):
    recs = B.run_benchmark("n", [2000, 4000], fixed={"l": 40, "k": 5, "d": 16},
                           backends=("b200", "noop"), repetitions=2)
    assert [r.backend for r in recs] == ["b200", "noop"] * 2
    assert all(r.runtime_seconds > 0 and not math.isnan(r.runtime_seconds)
               for r in recs)
    ground, batch = B.generate_problem(2000, 40, 5, 16, 0)
    assert ground.n == 2000 and batch.l == 40 and batch.k_max == 5
    B.write_csv(recs, tmp_path / "gpu.csv")
