"""Same-box A/B of the paired FFMA2 outer product (K3-SIMT binary32, C2 /
C3 fp32 shapes): the shipped library vs an experiment build without it.

    tools/build_ab.sh nof2="-DEXEM_SIMT_NO_FFMA2 -DEXEM_K2_NO_FFMA2"
    python tools/ffma2_ab.py        # on the GPU box (gpurun)
"""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path("/root/repo")
CHILD = r'''
import sys, json
sys.path.insert(0, %r); sys.path.insert(0, %r)
import bench_configs as B
V = B.gaussian(100_000, %d, 0)
r = B.greedy_record("ab", V, %r, t0=17, warm=1, steps=2, cpu_seconds=0.0)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"]}))
'''
for rep in range(1):
    for d, prec in ((100, "fp32"), (1024, "fp32"), (16, "fp32"), (512, "fp32")):
        for name, env_add in (("ffma2", {}), ("base_nof2", {"EXEM_LIB_PATH": str(ROOT / "paper_2101_08763_b200/_ab/libnof2.so")})):
            env = dict(os.environ, **env_add)
            p = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), str(ROOT / "tools"), d, prec)],
                               env=env, capture_output=True, text=True, cwd=ROOT)
            out = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-300:]
            print(rep, d, prec, name, out, flush=True)
