"""HBM-roofline evidence for the memory-bound kernels:
K1 ground_prepare, K2 set_min (single-set evaluate, k = 1/10/50) and the
Greedy m-update (greedy_update), timed with CUDA events at n = 1M, d = 100,
fp32 and bf16 (bf16 ground sets keep vt at the 2-byte storage type,
EXEM_VT_STORAGE: vb = 2).  Algorithmic bytes per launch:

  K1            read n*d*b (storage) + write n*d_pad*vb (vt) + 12n (norms, aux)
  set_min       SURVEY 8(d): n*d*vb (V once) + 8n (norms) + k*d*4 (elements)
                + 4n aux (+ 8n labels when requested); also 2*n*k*d flop on
                the FMA pipe (f32: one FFMA per point-element-dimension; the
                half storage's direct form (v-e)^2: FADD + FFMA, two), so the
                bound is max(HBM time, FMA-pipe time)
  greedy_update read vt (n*d*vb) + 8n norms + 4n m, write 4n m (+ the three
                folded h columns of the TC point operand for half storage,
                6n, when the xp refresh is on)

achieved = bytes / median launch time; peak = MEASURED_PEAKS.json hbm_gbs.

    python tools/hbm_kernels.py [--n 1000000] [--d 100]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timed(fn, reps=5):
    import torch

    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--d", type=int, default=100)
    args = ap.parse_args()
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.device import padded_rows, to_device_bytes

    torch.cuda.set_device(0)
    lib = N.lib()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    n, d = args.n, args.d
    V = np.random.default_rng(0).standard_normal((n, d), dtype=np.float32)
    out = []

    simt = ROOT / "profiles" / "simt_peak.json"
    ffma = json.loads(simt.read_text())["fp32_ffma_tflops"] \
        if simt.exists() else 72.5

    def rec(name, bytes_, t, flop=0.0, instr=1):
        r = {"kernel": name, "n": n, "d": d, "bytes": bytes_, "ms": t * 1e3,
             "achieved_gbs": bytes_ / t / 1e9, "peak_gbs": peak,
             "frac_hbm": bytes_ / t / 1e9 / peak}
        floor = bytes_ / (peak * 1e9)
        fma_t = instr * flop / (ffma * 1e12)  # FMA-pipe time
        if flop:
            r.update(flop=flop, achieved_tflops=flop / t / 1e12,
                     peak_ffma_tflops=ffma, fma_pipe_instr_per_flop2=instr)
            floor = max(floor, fma_t)
        r["bound"] = "ffma" if flop and fma_t > bytes_ / (peak * 1e9) \
            else "hbm"
        r["frac"] = floor / t  # of max(HBM time, FFMA time)
        out.append(r)
        print(json.dumps(r), flush=True)

    for prec in (pb.Precision.binary32, pb.Precision.bfloat16):
        g = pb.build_ground_set(V, precision=prec)
        dg = g.on_device()
        st = N.stream_handle()
        tag = dg.vt_tag  # | EXEM_VT_STORAGE for bf16: 2-byte vt
        vb = dg.vt.element_size()
        half = vb == 2
        instr = 2 if half else 1
        src = to_device_bytes(g.matrix.ravel(order="F"), dg.dev)
        e0 = to_device_bytes(g.aux, dg.dev)
        t = timed(lambda: lib.ground_prepare(
            tag, N.ptr(src), n, d, N.ptr(e0), N.ptr(dg.vt), dg.ld,
            N.ptr(dg.norms), N.ptr(dg.aux), N.ptr(dg.aux_sum),
            N.ptr(dg.scratch), 1, st))
        rec(f"K1 ground_prepare ({prec.value}, vt {vb}-byte)",
            n * d * prec.bytes_per_value + n * dg.d_pad * vb + 12 * n, t)
        src_r = to_device_bytes(np.ascontiguousarray(g.matrix), dg.dev)
        t = timed(lambda: lib.ground_prepare_rows(
            tag, N.ptr(src_r), n, d, N.ptr(e0), N.ptr(dg.vt), dg.ld,
            N.ptr(dg.norms), N.ptr(dg.aux), N.ptr(dg.aux_sum),
            N.ptr(dg.scratch), 1, st))
        rec(f"K1 ground_prepare_rows ({prec.value}, row-major source, vt "
            f"{vb}-byte)",
            n * d * prec.bytes_per_value + n * dg.d_pad * vb + 12 * n, t)
        for k in (1, 10, 16, 50, 64, 100, 128):
            elems = padded_rows(g.matrix[:k], dg.d_pad, prec, dg.dev)
            en = torch.empty(k, dtype=torch.float64, device=dg.dev)
            lib.row_norms(prec.tag, N.ptr(elems), k, d, dg.d_pad, N.ptr(en), st)
            s = torch.empty(1, dtype=torch.float64, device=dg.dev)
            # k > 64: several element groups, the running minimum carried in
            # t_out (as objective.device_set_min does)
            tb = (torch.empty(n, dtype=torch.float32, device=dg.dev)
                  if k > 64 else None)
            t = timed(lambda: lib.set_min(
                tag, N.ptr(dg.vt), dg.ld, n, d, N.ptr(dg.norms),
                N.ptr(dg.aux), N.ptr(elems), N.ptr(en), k, 1, N.ptr(tb), None,
                N.ptr(s), N.ptr(dg.scratch), st))
            groups = -(-k // 64)  # V passes (element groups of 64)
            rec(f"K2 set_min k={k} ({prec.value}, vt {vb}-byte)",
                groups * n * d * vb + 12 * n + k * d * 4 +
                (8 * n * (2 * groups - 1) if k > 64 else 0), t,
                2.0 * n * k * d, instr)
        # assign_clusters: K2 with the argmin-label epilogue, k = 50 exemplars
        elems = padded_rows(g.matrix[:50], dg.d_pad, prec, dg.dev)
        en = torch.empty(50, dtype=torch.float64, device=dg.dev)
        lib.row_norms(prec.tag, N.ptr(elems), 50, d, dg.d_pad, N.ptr(en), st)
        lab = torch.empty(n, dtype=torch.int64, device=dg.dev)
        s = torch.empty(1, dtype=torch.float64, device=dg.dev)
        t = timed(lambda: lib.set_min(
            tag, N.ptr(dg.vt), dg.ld, n, d, N.ptr(dg.norms),
            N.ptr(dg.aux), N.ptr(elems), N.ptr(en), 50, 0, None, N.ptr(lab),
            N.ptr(s), N.ptr(dg.scratch), st))
        rec(f"K2 set_min k=50 + labels (assign_clusters, {prec.value})",
            n * d * vb + 8 * n + 8 * n + 50 * d * 4, t, 2.0 * n * 50 * d,
            instr)
        m = torch.empty(dg.ld, dtype=torch.float32, device=dg.dev)
        m.copy_(dg.aux)
        sel = torch.zeros(1, dtype=torch.int64, device=dg.dev)
        msum = torch.empty(1, dtype=torch.float64, device=dg.dev)
        variants = [(None, "m only")]
        if half:  # the Greedy's TC point operand (its h columns refreshed)
            variants.append((torch.zeros((int(lib.tc_rows(n)), dg.kp),
                                         dtype=dg.vt.dtype, device=dg.dev),
                             "with the TC h refresh"))
        for xp, what in variants:
            t = timed(lambda: lib.greedy_update(
                tag, N.ptr(dg.vt), dg.ld, n, d, N.ptr(dg.norms),
                N.ptr(dg.vt), dg.ld, N.ptr(dg.norms), N.ptr(sel), 0, N.ptr(m),
                N.ptr(xp), dg.kp if xp is not None else 0, N.ptr(msum),
                N.ptr(dg.scratch), st))
            rec(f"K2 greedy_update (m-update, {prec.value}, vt {vb}-byte, "
                f"{what})",
                n * d * vb + 20 * n + (6 * n if xp is not None else 0), t,
                2.0 * n * d, instr)
    # .exem loader straight to the device (io.py: mapped payload -> one DMA
    # -> K1), wall clock of the public load_ground_set, file bytes / time
    import tempfile
    import time

    with tempfile.TemporaryDirectory() as tmp:
        path = Path(tmp) / "v.exem"
        pb.write_ground_file(path, V, pb.Precision.binary32)
        for rep in range(3):
            t0 = time.perf_counter()
            g = pb.load_ground_set(path)
            g.on_device()
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
        size = path.stat().st_size
        r = {"kernel": "load_ground_set(.exem, binary32) -> device (wall)",
             "n": n, "d": d, "bytes": size, "ms": t * 1e3,
             "achieved_gbs": size / t / 1e9, "peak_gbs": None, "frac": None}
        out.append(r)
        print(json.dumps(r), flush=True)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "hbm_kernels.jsonl").write_text(
        "".join(json.dumps(r) + "\n" for r in out))


if __name__ == "__main__":
    main()
