"""Benchmark records in the reference's CSV schema (mirror of
``pkg/src/exembatch/bench.py``), timing the B200 device path.

The schema, problem generator and speedup rule are the reference's
(bench.py:22-39 fields/presets, :66-93 generator, :172-179 speedup), so a CSV
written here and one written by the reference's ``run_benchmark`` on the
same (n, l, k, d, seed) describe the *same* problems and
``compute_speedup`` / ``figures/plot_bench.py --baseline reference`` can pair
them row by row.  The device path records ``backend="b200"`` (the
reference's backend names are accepted as aliases of that one path).
Timing is the wall clock of the public ``evaluate_batch`` call -- host
batch in, host values out, device synchronised -- median of the
repetitions, generation outside the timed region (bench.py:96-99,150-151).
"""

from __future__ import annotations

import csv
import statistics
import time
from dataclasses import asdict, dataclass
from typing import Optional, Sequence

import numpy as np

from .core import DeviceLimits, EvaluationBatch, Precision, build_ground_set
from .errors import (
    BudgetExceedsGroundSetError,
    IncomparableRecordsError,
    OutOfMemoryError,
)
from .evaluate import Evaluator, evaluate_batch

CSV_FIELDS = ("vary", "n", "l", "k", "d", "precision", "backend", "workers",
              "seed", "repetitions", "runtime_seconds")
DESK_DEFAULTS = {"n": 20000, "l": 500, "k": 10, "d": 100}
LARGE_DEFAULTS = {"n": 50000, "l": 5000, "k": 10, "d": 100}


@dataclass(frozen=True)
class BenchRecord:
    """One timed configuration (bench.py:42-63)."""

    vary: str
    n: int
    l: int
    k: int
    d: int
    precision: str
    backend: str
    workers: int
    seed: int
    repetitions: int
    runtime_seconds: float

    @property
    def failed(self) -> bool:
        return self.runtime_seconds != self.runtime_seconds  # NaN

    def shape_key(self):
        return (self.n, self.l, self.k, self.d, self.seed)


def generate_problem(n: int, l: int, k: int, d: int, seed: int,
                     precision: Precision = Precision.binary32):
    """The reference's seeded problem (bench.py:66-93): uniform [0, 1)
    ground data (kept below 1 after half rounding), l sets of k vectors
    sampled without replacement -- the same draws, so the same problem."""
    values, idx = draw_problem(n, l, k, d, seed, precision)
    ground = build_ground_set(values, aux="zero", precision=precision)
    sets = [ground.matrix[i] for i in idx]
    return ground, EvaluationBatch.from_sets(sets)


def draw_problem(n: int, l: int, k: int, d: int, seed: int,
                 precision: Precision = Precision.binary32):
    """Host part of ``generate_problem``: (values (n, d), set indices (l, k))
    in the reference's draw order."""
    if min(n, l, k, d) < 1:
        raise ValueError("n, l, k and d must all be >= 1")
    if k > n:
        raise BudgetExceedsGroundSetError(f"k={k} exceeds n={n}")
    rng = np.random.default_rng(seed)
    wide = precision is Precision.binary64
    values = rng.random((n, d), dtype=np.float64 if wide else np.float32)
    if precision is Precision.binary16:  # keep half-rounded values below 1
        values = np.minimum(values.astype(np.float16), np.float16(
            np.nextafter(np.float16(1), np.float16(0))))
    elif precision is Precision.bfloat16:  # (bf16 is this package's)
        values = np.minimum(values.astype(precision.dtype),
                            precision.dtype.type(1.0 - 2.0 ** -8))
    idx = np.stack([np.sort(rng.choice(n, size=k, replace=False))
                    for _ in range(l)])
    return values, idx


def _time_once(fn) -> float:
    start = time.perf_counter()
    fn()
    return time.perf_counter() - start


def run_benchmark(vary: str, values: Sequence[int],
                  fixed: Optional[dict] = None,
                  backends: Sequence[str] = ("b200",),
                  precisions: Sequence[Precision] = (Precision.binary32,),
                  repetitions: int = 5, seed: int = 0, workers: int = 1,
                  limits: Optional[DeviceLimits] = None) -> list:
    """Time every (value, backend, precision) combination (bench.py:102-169);
    an out-of-memory failure becomes a NaN record."""
    if vary not in ("n", "l", "k"):
        raise ValueError("vary must be one of 'n', 'l', 'k'")
    if not values:
        raise ValueError("values must be non-empty")
    if repetitions < 1:
        raise ValueError("repetitions must be >= 1")
    shape = dict(DESK_DEFAULTS)
    shape.update(fixed or {})
    limits = limits or DeviceLimits()
    records = []
    for value in values:
        cfg = dict(shape)
        cfg[vary] = int(value)
        for precision in precisions:
            ground, batch = generate_problem(cfg["n"], cfg["l"], cfg["k"],
                                             cfg["d"], seed, precision)
            for backend in backends:
                if backend == "noop":
                    run = lambda: np.zeros(batch.l)  # noqa: E731
                else:
                    ev = Evaluator(backend=backend, limits=limits,
                                   worker_count=workers)
                    run = lambda: evaluate_batch(ev, ground, batch)  # noqa: E731
                try:
                    run()  # warm-up: library load, tensor maps, allocator
                    runtime = statistics.median(
                        _time_once(run) for _ in range(repetitions))
                except OutOfMemoryError:
                    runtime = float("nan")
                records.append(BenchRecord(
                    vary=vary, n=cfg["n"], l=cfg["l"], k=cfg["k"], d=cfg["d"],
                    precision=precision.value, backend=backend,
                    workers=workers, seed=seed, repetitions=repetitions,
                    runtime_seconds=runtime))
    return records


def compute_speedup(baseline: BenchRecord, candidate: BenchRecord) -> float:
    """baseline / candidate runtime for the same problem (bench.py:172-179)."""
    if baseline.shape_key() != candidate.shape_key():
        raise IncomparableRecordsError(
            f"records describe different problems: {baseline.shape_key()} "
            f"vs {candidate.shape_key()}")
    return baseline.runtime_seconds / candidate.runtime_seconds


def write_csv(records: Sequence[BenchRecord], path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=CSV_FIELDS)
        w.writeheader()
        for rec in records:
            row = asdict(rec)
            row["runtime_seconds"] = repr(rec.runtime_seconds)
            w.writerow(row)


def read_csv(path) -> list:
    ints = ("n", "l", "k", "d", "workers", "seed", "repetitions")
    out = []
    with open(path, newline="") as fh:
        for row in csv.DictReader(fh):
            kw = {f: row[f] for f in CSV_FIELDS}
            for f in ints:
                kw[f] = int(kw[f])
            kw["runtime_seconds"] = float(kw["runtime_seconds"])
            out.append(BenchRecord(**kw))
    return out


def linear_fit_r2(xs: Sequence[float], ys: Sequence[float]) -> float:
    """R^2 of a least-squares line through (xs, ys) (bench.py:214-224)."""
    x = np.asarray(xs, dtype=np.float64)
    y = np.asarray(ys, dtype=np.float64)
    slope, intercept = np.polyfit(x, y, 1)
    ss_res = float(np.sum((y - (slope * x + intercept)) ** 2))
    ss_tot = float(np.sum((y - y.mean()) ** 2))
    return 1.0 if ss_tot == 0 else 1.0 - ss_res / ss_tot
