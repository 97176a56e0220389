"""K3-SIMT Greedy step timings at the C2 / C3 fp32 / fp64 shapes (n = 100k,
|S u c| = 19) with the shipped library -- the numbers DESIGN.md quotes for
the last-chunk skip of zero padding dimensions."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import bench_configs as B  # noqa: E402

for d, prec in ((2, "fp32"), (16, "fp32"), (100, "fp32"), (37, "fp32"),
                (100, "fp64")):
    V = B.gaussian(100_000, d, 0)
    r = B.greedy_record("tail", V, prec, t0=17, warm=1, steps=2,
                        cpu_seconds=0.0)
    print(json.dumps({"d": d, "prec": prec, "ms": r["ms_per_step"],
                      "frac": r["roofline"]["frac"]}), flush=True)
