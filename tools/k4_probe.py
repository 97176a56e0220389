"""K4-TC timing experiments: time the batch kernel alone (resident V, CUDA
events) for a few shapes and EXEM_TCB_DEBUG masks (1: no epilogue math,
2: no MMA, 4: no point TMA, 8: no aux load; the masks exist only in a probe
build: EXEM_NVCC_FLAGS=-DEXEM_TCB_PROBE_BUILD python -m
paper_2101_08763_b200.build, and rebuild normally afterwards).  Run on the
GPU box:

    python tools/k4_probe.py [--n 1000000] [--dims 100,256] [--ks 50]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def one(n, d, l, k, reps):
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.evaluate import DeviceBatch, batch_partials

    torch.cuda.set_device(0)
    prec = pb.Precision.bfloat16
    rng = np.random.default_rng(0)
    V = rng.standard_normal((n, d), dtype=np.float32)
    g = pb.build_ground_set(V, precision=prec)
    dg = g.on_device()
    sets = rng.standard_normal((l, k, d), dtype=np.float32)
    batch = pb.EvaluationBatch.from_sets(list(sets.astype(prec.dtype)))
    st = N.stream_handle()
    db = DeviceBatch(None, d, k, l, batch.cardinalities, prec, dg.d_pad,
                     dg.dev, st, sets=batch.sets)
    partial = torch.empty((dg.splits, l), dtype=torch.float64, device=dg.dev)
    batch_partials(dg, db, partial, dg.split_pts, dg.splits)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        batch_partials(dg, db, partial, dg.split_pts, dg.splits)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = float(np.median(ts))
    lib = N.lib()
    import ctypes

    spt, w, nc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    lib.raw("exem_tc_set_geometry")(k, ctypes.byref(spt), ctypes.byref(w),
                                    ctypes.byref(nc))
    tiles = -(-n // 128) * -(-l // spt.value)
    return {"n": n, "d": d, "l": l, "k": k, "s": t,
            "tflops": 2.0 * n * l * k * d / t / 1e12,
            "ns_per_tile_per_sm": t * 1e9 * 148 / tiles,
            "ncols": nc.value, "spt": spt.value,
            "dbg": int(os.environ.get("EXEM_TCB_DEBUG", "0"))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dims", default="100,256")
    ap.add_argument("--ks", default="50")
    ap.add_argument("--l", type=int, default=4096)
    ap.add_argument("--dbgs", default="0,1,2,4,8,5")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    if a.child:
        d, k = int(a.dims), int(a.ks)
        print(json.dumps(one(a.n, d, a.l, k, a.reps)), flush=True)
        return
    for d in a.dims.split(","):
        for k in a.ks.split(","):
            for dbg in a.dbgs.split(","):
                env = dict(os.environ, EXEM_TCB_DEBUG=dbg)
                r = subprocess.run([sys.executable, __file__, "--child",
                                    "--n", str(a.n), "--dims", d, "--ks", k,
                                    "--l", str(a.l), "--reps", str(a.reps)],
                                   env=env, capture_output=True, text=True,
                                   timeout=600)
                print(r.stdout.strip() or r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
