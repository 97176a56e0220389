"""The other BASELINE configs as sub-records of bench.py's JSON line.

bench.py's headline is config 4 (full Greedy, n = 1M, d = 100).  Every other
configuration of BASELINE.json is timed here in a few steps so that one
driver run observes all of them (each record: value, roofline of its
dominant kernel, a CPU baseline on a bounded sample):

  C4 variants   other precisions of the headline Greedy step: fp16 / bf16
                (K3-TC), binary32 on the CUDA cores (K3-SIMT), binary32 on the
                tensor cores (split-bf16), bf16 on clustered data (a Gaussian
                mixture: many positive gains, the epilogue's worst case)
  C2            one Greedy step, n = 100k, d = 100, binary32, |S u c| = 20
  C3            n = 100k, |S u c| = 50, d in {2, 100, 1024} x {bf16, fp32}
                (+ fp64 at d = 100)
  C5            the rank-0 shard of the 8-GPU job (50M / 8 rows, d = 256,
                l = 4096 sets of 50) streamed through an 8 GiB device budget
                (public evaluate_batch, V in host memory), and the resident
                K4-TC kernel time the roofline refers to

A Greedy step at |S| = t is reached by teacher forcing t seeded exemplars
(GreedyRun.force: K2 m-updates only) -- the per-step work of K3 does not
depend on S, only on l = n - t.  Timing: CUDA events on the launching
stream, synchronize on both sides; the dominant kernel's launches are
bracketed individually.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
UNIT = "candidate-set evals/s"


def load_peaks():
    out = {"bf16": 1400.0, "fp32": 74.4, "fp64": 37.2, "relu_gpairs": None,
           "src": "fallback"}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        j = json.loads(mp.read_text())
        out["bf16"] = float(j.get("bf16_tflops_sustained",
                                  j.get("bf16_tflops", out["bf16"])))
        out["hbm"] = float(j.get("hbm_gbs", 6540.0))
        out["src"] = "MEASURED_PEAKS.json"
    sp = ROOT / "profiles" / "simt_peak.json"
    if sp.exists():
        j = json.loads(sp.read_text())
        out["fp32"] = float(j["fp32_ffma_tflops"])
        out["fp64"] = float(j["fp64_dfma_tflops"])
        # the relu-sum as K3-TC computes it (FADD2 pairs) when measured,
        # else the FMNMX + FADD form
        out["relu_gpairs"] = j.get("relu_sum_fadd2_gpairs",
                                   j.get("relu_sum_gpairs"))
    return out


def gaussian(n, d, seed):
    return np.random.default_rng(seed).standard_normal((n, d),
                                                       dtype=np.float32)


def blobs(n, d, seed, k=16, spread=3.0):
    """Gaussian mixture in the shape of the reference's clustering demo
    (pkg/demos/03_greedy_clustering.py:20-23): k blob centres N(0, spread^2)
    away from the origin (e0 = 0), unit-variance points, random order."""
    rng = np.random.default_rng(seed)
    centres = rng.standard_normal((k, d), dtype=np.float32) * spread
    lab = rng.integers(0, k, size=n)
    return centres[lab] + rng.standard_normal((n, d), dtype=np.float32)


def cpu_rate(V, set_size, seconds, threads, dtype=np.float32, seed=0,
             rows=None):
    """The oracle port of the reference's evaluate path (numpy/OpenBLAS, one
    BLAS thread per worker, the row split of evaluate.py:162-170) on random
    sets of ``set_size`` at full n (or on the first ``rows`` rows, the rate
    then scaled by rows/n: per-set cost is linear in n)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import exem_oracle as O  # CPU baseline leg only

    n = V.shape[0]
    sub = V if rows is None or rows >= n else V[:rows]
    g = O.Ground(sub, dtype)
    rng = np.random.default_rng(seed + 1)
    done, t_total = 0, 0.0
    while True:
        sets = [g.matrix[rng.choice(sub.shape[0], size=set_size,
                                    replace=False)] for _ in range(threads)]
        t0 = time.perf_counter()
        O.evaluate_batch(g, sets, workers=threads)
        t_total += time.perf_counter() - t0
        done += len(sets)
        if t_total >= seconds:
            break
    rate = done / t_total * (sub.shape[0] / n)
    return rate, done, t_total, sub.shape[0]


def _events(torch):
    return (torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True))


def greedy_record(name, V, prec_name, *, t0=0, warm=1, steps=2,
                  split32=False, cpu_seconds=2.0, seed=0, workload=""):
    """Time ``steps`` Greedy steps at |S| = t0 + warm .. (K3 + K6 + K5 +
    K2), after t0 forced exemplars and ``warm`` untimed real steps."""
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.optimize import GreedyRun

    pk = load_peaks()
    prec = pb.Precision.from_name(prec_name)
    n, d = V.shape
    g = pb.build_ground_set(V, precision=prec)
    dg = g.on_device()
    lib = N.lib()
    with torch.cuda.device(dg.device_index):
        stream = torch.cuda.current_stream()
        run = GreedyRun(dg, k_cap=t0 + warm + steps, split32=split32)
        run.start()
        forced = np.random.default_rng(seed + 17).choice(n, size=t0,
                                                         replace=False)
        for s in range(t0):
            run.force(s, int(forced[s]))
        for s in range(t0, t0 + warm):
            run.step(s)
        ev = []
        orig = run.compute_gains

        def timed(chunk=None, out=None):
            a, b = _events(torch)
            a.record(stream)
            orig(chunk, out=out)
            b.record(stream)
            ev.append((a, b))

        run.compute_gains = timed
        launches0 = lib.launch_count()
        torch.cuda.synchronize()
        e0, e1 = _events(torch)
        e0.record(stream)
        for s in range(t0 + warm, t0 + warm + steps):
            run.step(s)
        e1.record(stream)
        torch.cuda.synchronize()
        launches = lib.launch_count() - launches0
        ms = e0.elapsed_time(e1)
        kms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        run.compute_gains = orig
    timed_t = list(range(t0 + warm, t0 + warm + steps))
    l_mean = float(np.mean([n - t for t in timed_t]))
    value = sum(n - t for t in timed_t) / (ms / 1e3)
    flop = 2.0 * n * l_mean * d
    if split32:
        kp = int(lib.tc_kp(int(lib.tc_split_dim(d))))
        executed = 2.0 * n * l_mean * kp
        roof = {"bound": "tensor", "kernel": "gains_tc_kernel (split-bf16 "
                "operands)", "achieved": executed / (kms / 1e3) / 1e12,
                "peak": pk["bf16"], "unit": "TFLOP/s",
                "algorithmic_fp32_tflops": flop / (kms / 1e3) / 1e12,
                "note": "binary32 gains from bf16 pieces: the executed "
                        f"K' = {kp} (6d + 6 rounded) is the tensor-pipe work; "
                        "algorithmic fp32 flops vs the FFMA peak "
                        f"{pk['fp32']:.1f} TF/s in algorithmic_fp32_tflops"}
    elif prec.is_half:
        roof = {"bound": "tensor", "kernel": "gains_tc_kernel",
                "achieved": flop / (kms / 1e3) / 1e12, "peak": pk["bf16"],
                "unit": "TFLOP/s"}
    else:
        f64 = prec is pb.Precision.binary64
        roof = {"bound": "fp64-pipe" if f64 else "fp32-pipe",
                "kernel": "gains_simt_kernel",
                "achieved": flop / (kms / 1e3) / 1e12,
                "peak": pk["fp64" if f64 else "fp32"], "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel_ms_avg"] = kms
    roof["kernel_share_of_step"] = kms * steps / ms
    roof["algorithmic_flop_per_launch"] = flop
    roof["traffic"] = None
    roof["peak_source"] = pk["src"] + " / profiles/simt_peak.json"
    if d <= 16 and pk.get("relu_gpairs"):
        # epilogue-bound shape: one FMNMX + one FADD per (candidate, point)
        # pair at least; denominator measured by
        # tools/simt_peak.cu (relu_sum_gpairs)
        pairs = n * l_mean / (kms / 1e3) / 1e9
        roof["epilogue"] = {"bound": "relu-sum issue rate (FADD2 pairs: "
                            "1 instruction per (candidate, point) value)",
                            "achieved_gpairs": pairs,
                            "peak_gpairs": float(pk["relu_gpairs"]),
                            "frac": pairs / float(pk["relu_gpairs"])}
    set_size = int(round(np.mean(timed_t))) + 1
    threads = os.cpu_count() or 1
    cdt = np.float64 if prec is pb.Precision.binary64 else np.float32
    rate, cnt, secs, rows = cpu_rate(V, set_size, cpu_seconds, threads,
                                     dtype=cdt, seed=seed)
    return {
        "name": name, "metric": "candidate-set evals/s", "value": value,
        "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
        "warmup": warm, "dtype": prec_name + (" (split-bf16 tensor)" if
                                              split32 else ""),
        "config": {"workload": workload, "n": n, "d": d,
                   "set_size": set_size, "timed_steps": timed_t,
                   "forced_exemplars": t0},
        "dist_evals_per_s": {"executed": n * value,
                             "reference_equivalent": n * value * set_size},
        "roofline": roof,
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads,
                         "kind": "port", "sample":
                         f"{cnt} sets of size {set_size} at n={rows}, d={d}, "
                         f"{np.dtype(cdt).name}, {secs:.1f}s; "
                         "oracle/exem_oracle.py restatement of "
                         "evaluate.py:142-170"},
        "gpu_launches": int(launches),
        "k3_epilogue": ({"groups": run.epi,
                         "screen_hit_fraction": run.hit_fraction}
                        if run.tc else None),
    }


def c5_record(cpu_seconds=2.0, n_total=50_000_000, shards=8, d=256, l=4096,
              card=50, budget_gb=8.0, seed=1000):
    """Rank 0's shard of config 5 on one GPU: V generated on the device
    (seeded), brought to host memory (bf16, column-major), then the public
    evaluate_batch streams it through ``budget_gb`` of device memory; and
    the resident K4-TC kernel over the same rows (the roofline's kernel)."""
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.distributed import shard_rows
    from paper_2101_08763_b200.evaluate import DeviceBatch, batch_partials

    pk = load_peaks()
    prec = pb.Precision.bfloat16
    lib = N.lib()
    r0, r1 = shard_rows(n_total, shards, 0, int(lib.split_points(n_total)))
    rows = r1 - r0
    gen = torch.Generator(device="cuda").manual_seed(seed)
    vt = torch.randn((d, rows), generator=gen, device="cuda",
                     dtype=torch.float32).to(torch.bfloat16)
    V = vt.view(torch.int16).cpu().numpy().view(prec.dtype).T  # F-order
    V.flags.writeable = False  # frozen: build_ground_set uses it in place
    del vt
    sets = np.random.default_rng(7).standard_normal(
        (l, card, d), dtype=np.float32).astype(prec.dtype)
    batch = pb.EvaluationBatch.from_sets(list(sets))
    budget = int(budget_gb * 2**30)
    g = pb.build_ground_set(V, precision=prec, device_budget=budget)
    assert g.streamed
    ev = pb.Evaluator()
    pb.evaluate_batch(ev, g, batch)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vals = pb.evaluate_batch(ev, g, batch)
    torch.cuda.synchronize()
    t_stream = time.perf_counter() - t0
    del g
    # resident kernel (the roofline's K4-TC launch)
    gr = pb.build_ground_set(V, precision=prec)
    dg = gr.on_device()
    with torch.cuda.device(dg.device_index):
        st = N.stream_handle(dg.dev)
        db = DeviceBatch(None, d, card, l, batch.cardinalities, prec,
                         dg.d_pad, dg.dev, st, sets=batch.sets)
        part = torch.empty((dg.splits, l), dtype=torch.float64, device=dg.dev)
        batch_partials(dg, db, part, dg.split_pts, dg.splits)
        torch.cuda.synchronize()
        e0, e1 = _events(torch)
        reps = 2
        e0.record()
        for _ in range(reps):
            batch_partials(dg, db, part, dg.split_pts, dg.splits)
        e1.record()
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1) / reps
        sums = torch.empty(l, dtype=torch.float64, device=dg.dev)
        lib.reduce_partials(N.ptr(part), dg.splits, l, 1.0, N.ptr(sums), st)
        acc = prec.accumulate_dtype
        vr = acc.type(gr.aux_loss) - sums.cpu().numpy().astype(acc) / \
            acc.type(rows)
    same = bool(np.array_equal(vr, vals))
    flop = 2.0 * rows * l * card * d
    threads = os.cpu_count() or 1
    sub_rows = 200_000
    rate, cnt, secs, used = cpu_rate(np.asarray(V[:sub_rows], np.float32),
                                     card, cpu_seconds, threads, seed=seed)
    rate *= sub_rows / rows  # linear in n (tests/test_acceptance.py:178-208)
    achieved = flop / (kms / 1e3) / 1e12
    return {
        "name": "C5 rank-0 shard, streamed", "metric": "set evals/s",
        "value": l / t_stream, "unit": "set evals/s (l=4096 sets of 50)",
        "seconds_per_pass": t_stream, "dtype": "bf16",
        "config": {"workload": "C5 low-memory: evaluate_batch of l=4096 "
                   "explicit sets |S|=50 over rank 0's shard of the 8-GPU "
                   f"n=50M job ({rows} rows), d={d}, V in host memory "
                   f"streamed through a {budget_gb:.0f} GiB device budget",
                   "n_total": n_total, "shards": shards, "rows": rows, "d": d,
                   "l": l, "set_size": card},
        "dist_evals_per_s": {"reference_equivalent":
                             rows * l * card / t_stream},
        "streamed_equals_resident": same,
        "resident_kernel_ms": kms,
        "roofline": {"bound": "tensor", "kernel": "batch_tc_kernel",
                     "achieved": achieved, "peak": pk["bf16"],
                     "unit": "TFLOP/s", "frac": achieved / pk["bf16"],
                     "algorithmic_flop_per_launch": flop,
                     "kernel_ms_avg": kms, "traffic": None,
                     "stream_over_kernel": t_stream / (kms / 1e3)},
        "cpu_baseline": {"value": rate, "unit": "set evals/s",
                         "cores": threads, "kind": "port",
                         "sample": f"{cnt} sets of {card} at n={sub_rows} "
                         f"(first rows of the shard), fp32, {secs:.1f}s, "
                         f"scaled by {sub_rows}/{rows} (per-set cost is "
                         "linear in n)"},
    }


def c1_record(cpu_seconds=2.0, reps=50):
    """BASELINE config 1 through the public API with host arrays: single-set
    f(S) (|S| = 10, evaluate_single) and Greedy k = 10 (build_ground_set +
    greedy_maximize), binary32, on the seeded C1 draw (tests/golden/
    make_golden.py:c1_data); picks checked against the reference's golden
    picks (tests/golden/golden.npz, generated by the reference itself)."""
    import torch

    import paper_2101_08763_b200 as pb

    rng = np.random.default_rng(1234)
    V = rng.standard_normal((10000, 100), dtype=np.float32)
    S = np.sort(rng.choice(10000, size=10, replace=False))
    prec = pb.Precision.binary32
    gz = ROOT / "tests" / "golden" / "golden.npz"
    golden = np.load(gz) if gz.exists() else None
    g = pb.build_ground_set(V, precision=prec)
    elems = np.asarray(g.matrix[S])
    pb.evaluate_single(g, elems)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f = pb.evaluate_single(g, elems)
        ts.append(time.perf_counter() - t0)
    single_ms = float(np.median(ts)) * 1e3
    pb.greedy_maximize(pb.build_ground_set(V, precision=prec), k=10)  # warm
    torch.cuda.synchronize()
    gts = []
    for _ in range(5):
        t0 = time.perf_counter()
        res = pb.greedy_maximize(pb.build_ground_set(V, precision=prec), k=10)
        gts.append(time.perf_counter() - t0)
    greedy_s = float(np.median(gts))
    evals = res.evaluations
    match = None
    if golden is not None and "c1_f32_picks" in golden.files:
        match = list(res.exemplar_indices) == golden["c1_f32_picks"].tolist()
    # CPU: the oracle port on the same draw; single set 1 thread, Greedy
    # extrapolated from a sample of its candidate sets (mean |S u c| = 6)
    sys.path.insert(0, str(ROOT / "oracle"))
    import exem_oracle as O  # CPU baseline leg only

    og = O.Ground(V, np.float32)
    cts = []
    for _ in range(5):
        t0 = time.perf_counter()
        O.evaluate_batch(og, [og.matrix[S]], workers=1)
        cts.append(time.perf_counter() - t0)
    threads = os.cpu_count() or 1
    rate, cnt, secs, _ = cpu_rate(V, 6, cpu_seconds, threads, seed=1234)
    return {
        "name": "C1 public API", "metric": "candidate-set evals/s",
        "value": evals / greedy_s, "unit": UNIT, "dtype": "fp32",
        "config": {"workload": "C1: single-set f(S) |S|=10 + Greedy k=10, "
                   "n=10k, d=100, seed 1234, host numpy arrays in and out "
                   "(build_ground_set + evaluate_single / greedy_maximize)",
                   "n": 10000, "d": 100, "k": 10},
        "single_set_ms": single_ms, "single_set_f": float(f),
        "greedy_seconds": greedy_s, "greedy_evaluations": evals,
        "picks_match_reference_golden": match,
        "roofline": {"bound": "latency", "note": "n=10k: every kernel is a "
                     "few microseconds; the public call is bound by launch "
                     "and host<->device latency, not by a pipe"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads,
                         "kind": "port", "single_set_ms_1thread":
                         float(np.median(cts)) * 1e3,
                         "greedy_seconds_extrapolated": evals / rate,
                         "sample": f"{cnt} sets of size 6 (mean |S u c| of "
                         f"the k=10 Greedy) at n=10000, fp32, {secs:.1f}s; "
                         "single set: 5 reps on 1 thread; oracle/"
                         "exem_oracle.py restatement of evaluate.py:142-170"},
    }


def all_records(cpu_seconds=2.0, headline_precision="bf16", log=None):
    """Every sub-record; a failing one is reported, not fatal."""
    out = []
    n4, d4 = 1_000_000, 100
    other_half = "fp16" if headline_precision == "bf16" else "bf16"
    V4 = gaussian(n4, d4, 0)
    plan = [
        ("C4 " + other_half, lambda: greedy_record(
            "C4 " + other_half, V4, other_half, warm=3, steps=3,
            cpu_seconds=cpu_seconds, workload="C4 Greedy step, n=1M, d=100")),
        ("C4 fp32 K3-SIMT", lambda: greedy_record(
            "C4 fp32 K3-SIMT", V4, "fp32", warm=1, steps=2,
            cpu_seconds=cpu_seconds,
            workload="C4 Greedy step, n=1M, d=100, binary32 CUDA cores")),
        ("C4 fp32 split-bf16", lambda: greedy_record(
            "C4 fp32 split-bf16", V4, "fp32", split32=True, warm=2, steps=3,
            cpu_seconds=cpu_seconds,
            workload="C4 Greedy step, n=1M, d=100, binary32 on tensor cores")),
        ("C4 bf16 clustered", lambda: greedy_record(
            "C4 bf16 clustered", blobs(n4, d4, 3), "bf16", warm=3, steps=3,
            cpu_seconds=cpu_seconds, workload="C4 Greedy step on a 16-blob "
            "Gaussian mixture (demos/03 shape): many positive gains")),
    ]
    plan.append(("C1", lambda: c1_record(cpu_seconds=cpu_seconds)))
    V2 = gaussian(100_000, 100, 0)
    plan.append(("C2 fp32", lambda: greedy_record(
        "C2 fp32", V2, "fp32", t0=17, warm=1, steps=2,
        cpu_seconds=cpu_seconds, workload="C2 batched step, n=100k, d=100, "
        "|S u c|=20")))
    for d in (2, 16, 100, 512, 1024):
        for p in ("bf16", "fp32") + (("fp64",) if d == 100 else ()):
            nm = f"C3 d={d} {p}"
            plan.append((nm, (lambda d=d, p=p, nm=nm: greedy_record(
                nm, gaussian(100_000, d, 0), p, t0=47, warm=1, steps=2,
                cpu_seconds=cpu_seconds,
                workload=f"C3 sweep, n=100k, d={d}, |S u c|=50"))))
    plan.append(("C5", lambda: c5_record(cpu_seconds=cpu_seconds)))
    for nm, fn in plan:
        t0 = time.perf_counter()
        try:
            rec = fn()
        except Exception as e:  # report, keep going
            rec = {"name": nm, "error": f"{type(e).__name__}: {e}"}
        rec["wall_s"] = time.perf_counter() - t0
        out.append(rec)
        if log is not None:
            print(json.dumps(rec), file=log, flush=True)
        import torch

        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    sys.path.insert(0, str(ROOT))
    recs = all_records(log=sys.stderr)
    print(json.dumps(recs))
