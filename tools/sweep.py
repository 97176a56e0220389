"""Precision / dimensionality sweep of the batched Greedy gains (K3) and the
explicit-set batch kernel (K4) -- BASELINE configs 2 and 3, plus a 1-GPU
slice of config 5.  Run on the GPU box:

    python tools/sweep.py [--only c2,c3,k4] [--out gpurun_out/sweep]

C2: n=100k, d=100, fp32, |S u c| = 20 (19 real Greedy steps, then step 20's
    l = 99,981 candidate sets timed).
C3: n=100k, |S u c| = 50 (49 real Greedy steps, then step 50 timed),
    d in {2,16,100,512,1024} x {fp64, fp32, fp16, bf16}.
K4: explicit packed sets (evaluate_batch's kernel): n points x l sets of
    |S_j| elements, d=256 (a 1/50 row slice of C5 by default).

Each timed launch is bracketed by CUDA events on the launching stream
(median of 3 after 1 warm-up).  Roofline denominators: measured FFMA/DFMA
peaks from tools/simt_peak.cu (gpurun_out/simt_peak.json when present),
cuBLAS bf16 sustained from MEASURED_PEAKS.json for the tensor path.
Algorithmic flop = 2*n*l*d (candidate-set pairs x the d-dim dot); the
executed figure uses the kernel's padded K.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def peaks():
    out = {"bf16": 1400.0, "fp32": 74.4, "fp64": 37.2, "src": "spec"}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        j = json.loads(mp.read_text())
        out["bf16"] = float(j.get("bf16_tflops_sustained", out["bf16"]))
    for p in (ROOT / "gpurun_out" / "simt_peak.json",
              ROOT / "profiles" / "simt_peak.json"):
        if p.exists():
            j = json.loads(p.read_text())
            out["fp32"] = float(j["fp32_ffma_tflops"])
            out["fp64"] = float(j["fp64_dfma_tflops"])
            out["src"] = f"measured ({p.relative_to(ROOT)})"
            break
    return out


def timed(fn, stream, reps=3):
    import torch

    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def greedy_case(n, d, prec_name, picks, seed, pk, split32=False):
    """Run `picks` real Greedy steps, then time the next step's K3 launch."""
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.optimize import GreedyRun

    prec = pb.Precision.from_name(prec_name)
    V = np.random.default_rng(seed).standard_normal((n, d), dtype=np.float32)
    g = pb.build_ground_set(V, precision=prec)
    dg = g.on_device(0)
    run = GreedyRun(dg, k_cap=picks + 1, split32=split32)
    run.start()
    for s in range(picks):
        run.step(s)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    # K3 alone (the launch that dominates a step) and the whole step
    t_gain = timed(lambda: run.compute_gains(), st)
    t0 = time.perf_counter()
    run.step(picks)
    torch.cuda.synchronize()
    t_step_wall = time.perf_counter() - t0
    l = n - picks
    flop = 2.0 * n * l * d
    lib = N.lib()
    if prec.is_half or run.split32:
        kexec = int(-(-(d + 6) // 16) * 16)
        if run.split32:
            kexec = int(-(-(6 * d + 6) // 16) * 16)
        pipe, peak = "tensor", pk["bf16"]
        kern = "gains_tc_kernel" + (" (split-bf16 fp32)" if run.split32 else "")
    else:
        kexec = int(lib.pad_dims(d))
        pipe = "fp64-pipe" if prec_name == "fp64" else "fp32-pipe"
        peak = pk["fp64"] if prec_name == "fp64" else pk["fp32"]
        kern = "gains_simt_kernel"
    achieved = flop / t_gain / 1e12
    rec = {
        "n": n, "d": d, "precision": prec_name, "set_size": picks + 1, "l": l,
        "kernel": kern, "kernel_s": t_gain, "step_wall_s": t_step_wall,
        "cand_sets_per_s": l / t_gain, "pairs_per_s": n * l / t_gain,
        "ref_equiv_dist_evals_per_s": n * l * (picks + 1) / t_gain,
        "alg_tflops": achieved,
        "exec_tflops": 2.0 * n * l * kexec / t_gain / 1e12,
        "bound": pipe, "peak_tflops": peak, "frac": achieved / peak,
        "exec_frac": 2.0 * n * l * kexec / t_gain / 1e12 / peak,
        "epilogue_pairs_per_clk_per_sm": None,
    }
    del run, dg, g
    torch.cuda.empty_cache()
    return rec


def c1_case():
    """BASELINE config 1 on the device: single-set f(S) with |S| = 10 and the
    whole Greedy k = 10, n = 10,000, d = 100, fp32, Gaussian seed 1234
    (the reference's CPU path: 4.1-4.6 ms per f(S), 294 s for the Greedy
    on 1 thread, 63 s on 8).  Wall clock of the public
    calls, host arrays in and out."""
    import torch

    import paper_2101_08763_b200 as pb

    rng = np.random.default_rng(1234)
    V = rng.standard_normal((10000, 100), dtype=np.float32)
    S = np.sort(rng.choice(10000, size=10, replace=False))
    g = pb.build_ground_set(V, precision=pb.Precision.binary32)
    pb.evaluate_single(g, g.matrix[S])
    torch.cuda.synchronize()
    reps = 50
    t0 = time.perf_counter()
    for _ in range(reps):
        pb.evaluate_single(g, g.matrix[S])
    t_single = (time.perf_counter() - t0) / reps
    pb.greedy_maximize(g, k=10)
    t0 = time.perf_counter()
    res = pb.greedy_maximize(g, k=10)
    t_greedy = time.perf_counter() - t0
    return {"n": 10000, "d": 100, "precision": "fp32", "set_size": 10,
            "l": 1, "kernel": "evaluate_single / greedy_maximize (public API)",
            "kernel_s": t_single, "greedy_k10_s": t_greedy,
            "greedy_picks": list(res.exemplar_indices),
            "cand_sets_per_s": sum(10000 - t for t in range(10)) / t_greedy,
            "alg_tflops": 0.0, "bound": "latency", "frac": float("nan")}


def k4_case(n, d, prec_name, l, card, seed, pk):
    """Time K4 (explicit packed sets) through the evaluate_batch kernels."""
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import evaluate as E

    prec = pb.Precision.from_name(prec_name)
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((n, d), dtype=np.float32)
    g = pb.build_ground_set(V, precision=prec)
    idx = np.stack([rng.choice(n, size=card, replace=False) for _ in range(l)])
    vals = g.matrix[idx.reshape(-1)].reshape(l, card, d)
    packed = np.ascontiguousarray(vals.transpose(2, 1, 0))  # [d][k][l]
    st = torch.cuda.current_stream()
    t = timed(lambda: E.device_packed_sums(g, packed, d, card, l,
                                           [card] * l), st, reps=2)
    flop = 2.0 * n * l * card * d
    peak = pk["fp64"] if prec_name == "fp64" else (
        pk["bf16"] if prec.is_half and getattr(E, "tc_batch_supported",
                                              lambda *a: False)(prec, card)
        else pk["fp32"])
    rec = {"n": n, "d": d, "precision": prec_name, "l": l, "set_size": card,
           "kernel": "batch_eval", "kernel_s": t,
           "sets_per_s": l / t, "ref_equiv_dist_evals_per_s": n * l * card / t,
           "alg_tflops": flop / t / 1e12, "peak_tflops": peak,
           "frac": flop / t / 1e12 / peak,
           "note": "includes host pack+H2D of the set buffer"}
    del g
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c3,k4")
    ap.add_argument("--out", default="gpurun_out/sweep")
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--dims", default="2,16,100,512,1024")
    ap.add_argument("--precs", default="fp64,fp32,fp16,bf16")
    ap.add_argument("--k4-n", type=int, default=1_000_000)
    args = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    pk = peaks()
    only = set(args.only.split(","))
    recs = []

    def emit(tag, r):
        r["case"] = tag
        recs.append(r)
        print(json.dumps(r), flush=True)

    if "c1" in only:
        emit("C1", c1_case())
    if "c2" in only:
        emit("C2", greedy_case(args.n, 100, "fp32", 19, 0, pk))
        emit("C2", greedy_case(args.n, 100, "fp32", 19, 0, pk, split32=True))
    if "c3" in only:
        for d in [int(x) for x in args.dims.split(",")]:
            for p in args.precs.split(","):
                emit("C3", greedy_case(args.n, d, p, 49, 0, pk))
    if "k4" in only:
        for p in ("fp32", "bf16"):
            emit("K4", k4_case(args.k4_n, 256, p, 4096, 50, 0, pk))
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.with_suffix(".jsonl").write_text(
        "".join(json.dumps(r) + "\n" for r in recs))
    lines = [f"peaks: {pk}", "",
             "| case | d | prec | set | l | kernel | ms | cand-sets/s | alg TF/s "
             "| bound | frac |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in recs:
        lines.append(
            f"| {r['case']} | {r['d']} | {r['precision']} | {r['set_size']} | "
            f"{r['l']} | {r['kernel']} | {1e3 * r['kernel_s']:.2f} | "
            f"{r.get('cand_sets_per_s', r.get('sets_per_s')):.4g} | "
            f"{r['alg_tflops']:.1f} | {r.get('bound', '')} | {r['frac']:.3f} |")
    out.with_suffix(".md").write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
