"""Same-box A/B of the K3-SIMT operand path: TMA-fed (default) vs the
cp.async kernel (EXEM_SIMT_CPASYNC=1), at the C2 / C3 fp32 / fp64 shapes."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import sys, json
sys.path.insert(0, %r); sys.path.insert(0, %r)
import bench_configs as B
V = B.gaussian(100_000, %d, 0)
r = B.greedy_record("ab", V, %r, t0=17, warm=1, steps=2, cpu_seconds=0.0)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"]}))
'''

for rep in range(2):
    for d, prec in ((100, "fp32"), (1024, "fp32"), (100, "fp64"), (16, "fp32")):
        for name, env_add in (("tma", {}), ("cpasync", {"EXEM_SIMT_CPASYNC": "1"})):
            env = dict(os.environ, **env_add)
            p = subprocess.run([sys.executable, "-c",
                                CHILD % (str(ROOT), str(ROOT / "tools"), d, prec)],
                               env=env, capture_output=True, text=True, cwd=ROOT)
            out = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-300:]
            print(rep, d, prec, name, out, flush=True)
