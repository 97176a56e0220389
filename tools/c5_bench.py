"""BASELINE config 5 -- low-memory streaming regime on one B200.

    python tools/c5_bench.py [--n 50000000] [--shards 8] [--d 256] [--l 4096]
                             [--k 50] [--precision bf16] [--budget-gb 8]

Config 5 is n = 50M points, d = 256, l = 4096 explicit sets of |S_j| = 50,
sharded by rows across 8 GPUs.  One GPU here runs rank 0's share (n/shards
rows, the per-GPU work of the 8-GPU job; `--shards 1` runs all 50M rows on
one GPU).  V is generated per shard (N(0,1) float32, seed = 1000 + rank,
rounded to the storage precision) and kept in host memory; the ground set is
built with ``device_budget`` so it STREAMS through the device in
split-aligned slices (streaming.py) unless it fits.  The sets' vectors are
N(0,1) draws (seed 7) -- in an 8-GPU run they are broadcast once.

Measured (CUDA events on the compute stream):
  kernel   K4 / K4-TC over every slice with V already resident in HBM
           (value the roofline refers to: 2*n*l*|S|*d flop per pass)
  stream   the public evaluate_batch on the streamed ground set: H2D of
           every slice + K1 prepare + operand pack + K4, overlapped
Prints one JSON line.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50_000_000)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--l", type=int, default=4096)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--budget-gb", type=float, default=8.0)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()

    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.distributed import shard_rows
    from paper_2101_08763_b200.evaluate import DeviceBatch, batch_partials
    from paper_2101_08763_b200 import streaming as S

    torch.cuda.set_device(0)
    lib = N.lib()
    prec = pb.Precision.from_name(args.precision)
    sp_global = int(lib.split_points(args.n))
    r0, r1 = shard_rows(args.n, args.shards, 0, sp_global)
    rows = r1 - r0
    d, l, k = args.d, args.l, args.k
    t0 = time.perf_counter()
    V = np.empty((rows, d), dtype=prec.dtype, order="F")
    rng = np.random.default_rng(1000)
    step = 1 << 20
    for a in range(0, rows, step):
        b = min(rows, a + step)
        V[a:b] = rng.standard_normal((b - a, d), dtype=np.float32).astype(prec.dtype)
    sets = np.random.default_rng(7).standard_normal((l, k, d), dtype=np.float32)
    t_gen = time.perf_counter() - t0

    budget = int(args.budget_gb * 2**30)
    t0 = time.perf_counter()
    g = pb.build_ground_set(V, precision=prec, device_budget=budget)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    batch = pb.EvaluationBatch.from_sets(list(sets.astype(prec.dtype)))

    # ---- streamed end to end through the public API (V from host memory)
    ev = pb.Evaluator()
    stream_s = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        vals = pb.evaluate_batch(ev, g, batch)
        torch.cuda.synchronize()
        stream_s.append(time.perf_counter() - a)

    # ---- where the streamed time goes (host pack, batch upload, per-slice
    # DMA / prepare / K4), events on the copy and compute streams
    torch.cuda.synchronize()
    a = time.perf_counter()
    db0 = DeviceBatch(None, d, k, l, batch.cardinalities, prec,
                      int(lib.pad_dims(d)), torch.device("cuda", 0),
                      N.stream_handle(), sets=batch.sets)
    torch.cuda.synchronize()
    t_upload = time.perf_counter() - a
    del db0
    budget_rows = budget - S.batch_device_bytes(d, k, l, prec,
                                                -(-rows // sp_global)) - \
        S._margin(rows)
    gsm = S.GroundStream(g, budget_rows)
    db1 = DeviceBatch(None, d, k, l, batch.cardinalities, prec,
                      int(lib.pad_dims(d)), gsm.dev, N.stream_handle(),
                      sets=batch.sets)
    part = torch.zeros((-(-rows // sp_global), l), dtype=torch.float64,
                       device=gsm.dev)
    torch.cuda.synchronize()
    evs = []
    a = time.perf_counter()
    for slot, q0, q1 in gsm.slices(pack_points=db1.xs is not None):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        from ctypes import c_void_p
        batch_partials(slot, db1, c_void_p(part.data_ptr() +
                                           (q0 // sp_global) * l * 8),
                       sp_global, -(-(q1 - q0) // sp_global))
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    t_loop = time.perf_counter() - a
    k4_slices = [x.elapsed_time(y) / 1e3 for x, y in evs]
    gsm.close()
    del db1, part, gsm
    breakdown = {"batch_upload_s": t_upload,
                 "slice_loop_s": t_loop, "k4_per_slice_s": k4_slices,
                 "k4_sum_s": float(sum(k4_slices))}

    # ---- kernel only: the same K4 launches with each slice resident
    sp = int(lib.split_points(rows))
    dg_budget = S.resident_bytes(rows, d, prec)
    kernel_s = None
    if dg_budget < 0.7 * torch.cuda.mem_get_info()[0]:
        gr = pb.build_ground_set(V, precision=prec)
        dg = gr.on_device()
        st = N.stream_handle()
        db = DeviceBatch(None, d, k, l, batch.cardinalities, prec, dg.d_pad,
                         dg.dev, st, sets=batch.sets)
        partial = torch.empty((dg.splits, l), dtype=torch.float64,
                              device=dg.dev)
        batch_partials(dg, db, partial, dg.split_pts, dg.splits)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            batch_partials(dg, db, partial, dg.split_pts, dg.splits)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        kernel_s = float(np.median(ts))
        sums = torch.empty(l, dtype=torch.float64, device=dg.dev)
        lib.reduce_partials(N.ptr(partial), dg.splits, l, 1.0, N.ptr(sums), st)
        acc = prec.accumulate_dtype
        vr = acc.type(gr.aux_loss) - sums.cpu().numpy().astype(acc) / acc.type(rows)
        same = bool(np.array_equal(vr, vals))
        del gr, dg, db, partial
    else:
        same = None
    flop = 2.0 * rows * l * k * d
    mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    simt = json.loads((ROOT / "profiles" / "simt_peak.json").read_text())
    if prec.is_half:
        peak = float(mp.get("bf16_tflops_sustained", 1400.0))
        bound = "tensor"
    else:
        peak = float(simt["fp64_dfma_tflops" if prec is pb.Precision.binary64
                          else "fp32_ffma_tflops"])
        bound = "fp32-pipe" if prec is pb.Precision.binary32 else "fp64-pipe"
    t_stream = float(np.median(stream_s))
    plan = S.plan_slices(rows, d, prec, budget - S.batch_device_bytes(
        d, k, l, prec, -(-rows // sp)) - S._margin(rows), sp)
    out = {
        "config": "C5 low-memory streaming: n=%d d=%d l=%d |S|=%d, rank-0 "
                  "shard of %d (%d rows)" % (args.n, d, l, k, args.shards, rows),
        "precision": args.precision, "rows": rows, "streamed": g.streamed,
        "device_budget_bytes": budget, "slices": len(plan.slices),
        "rows_per_slice": plan.rows_per_slice,
        "host_V_bytes": int(V.nbytes),
        "stream_s": t_stream, "stream_sets_per_s": l / t_stream,
        "stream_h2d_gbs": V.nbytes / t_stream / 1e9,
        "kernel_s": kernel_s,
        "kernel_sets_per_s": (l / kernel_s) if kernel_s else None,
        "ref_equiv_dist_evals_per_s": rows * l * k / (kernel_s or t_stream),
        "roofline": {"bound": bound, "achieved": flop / (kernel_s or t_stream) / 1e12,
                     "peak": peak, "unit": "TFLOP/s",
                     "frac": flop / (kernel_s or t_stream) / 1e12 / peak},
        "stream_over_kernel": (t_stream / kernel_s) if kernel_s else None,
        "streamed_equals_resident": same,
        "gen_s": t_gen, "build_s": t_build,
        "projected_8gpu_job_s": t_stream if args.shards == 8 else None,
        "breakdown": breakdown,
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
