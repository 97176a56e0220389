"""gpurun_out/hbm_kernels.jsonl (tools/hbm_kernels.py) -> a markdown table.

    python tools/hbm_md.py gpurun_out/hbm_kernels.jsonl > profiles/<tag>_hbm_kernels.md
"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
peak = next((r["peak_gbs"] for r in rows if r.get("peak_gbs")), None)
print("# HBM / FFMA-bound kernels (tools/hbm_kernels.py), n = 1M, d = 100, "
      "CUDA events, median of 5\n")
print(f"Bytes = SURVEY 8(d) algorithmic bytes per launch (V read once: n*d*vb "
      f"+ 8n norms + 4n aux + k*d*4 elements, + outputs; vb = 2 for bf16 "
      f"ground sets, which keep vt at the storage type); flop = 2*n*k*d. "
      f"Roofline = max(bytes / HBM peak {peak} GB/s, FMA-pipe time = flop x "
      "instr / FFMA peak (profiles/simt_peak.json); instr = 1 for the f32 "
      "GEMM form, 2 for the half direct form (v-e)^2 = FADD + FFMA); "
      "frac = that time / measured time.\n")
print("| kernel | bytes | flop | ms | GB/s | TF/s | bound | fraction of roofline |")
print("|---|---|---|---|---|---|---|---|")
for r in rows:
    fl = r.get("flop") or 0
    tf = f"{r['achieved_tflops']:.1f}" if r.get("achieved_tflops") else ""
    frac = f"{r['frac']:.2f}" if r.get("frac") is not None else "(wall)"
    print(f"| {r['kernel']} | {r['bytes'] / 1e6:.0f} MB | "
          f"{fl / 1e9:.1f} G | {r['ms']:.3f} | {r['achieved_gbs']:.0f} | {tf} | "
          f"{r.get('bound') or ''} | {frac} |")
