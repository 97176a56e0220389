import json, sys
from pathlib import Path
ROOT = Path("/root/repo"); sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import bench_configs as B
for d in (16, 512, 1024):
    V = B.gaussian(100_000, d, 0)
    r = B.greedy_record("bk", V, "fp32", t0=17, warm=1, steps=2, cpu_seconds=0.0)
    print(json.dumps({"d": d, "ms": r["ms_per_step"], "frac": r["roofline"]["frac"]}), flush=True)
