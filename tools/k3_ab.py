"""Same-box A/B of K3-TC builds: time warm Greedy steps at C4 size on
Gaussian and blob data for each library given (EXEM_LIB_PATH per run, one
subprocess each, alternating A B A B).

    python tools/k3_ab.py A=path/to/libA.so B=paper_2101_08763_b200/libexem_b200.so
"""
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
kind = %r
if kind in ("gauss", "blobs"):
    V = B.blobs(1_000_000, 100, 3) if kind == "blobs" else B.gaussian(1_000_000, 100, 0)
    r = B.greedy_record("ab", V, "bf16", warm=3, steps=5, cpu_seconds=0.0)
else:  # c3d<d>: the C3 sweep shape (n = 100k, |S u c| = 50)
    r = B.greedy_record("ab", B.gaussian(100_000, int(kind[3:]), 0), "bf16",
                        t0=47, warm=1, steps=2, cpu_seconds=0.0)
print(json.dumps({"ms": r["ms_per_step"], "kms": r["roofline"]["kernel_ms_avg"],
                  "epi": r["k3_epilogue"]}))
'''


def main():
    # NAME=lib.so[:EPI]  (EPI forces the epilogue width via EXEM_K3_EPI)
    libs = dict(a.split("=", 1) for a in sys.argv[1:])
    out = {}
    for rep in range(2):
        for data in os.environ.get("K3AB_DATA", "gauss,blobs").split(","):
            for name, path in libs.items():
                lib, _, epi = path.partition(":")
                env = dict(os.environ, EXEM_LIB_PATH=str(Path(lib).resolve()))
                if epi:
                    env["EXEM_K3_EPI"] = epi
                code = CHILD % (str(ROOT), str(ROOT / "tools"), data)
                p = subprocess.run([sys.executable, "-c", code], env=env,
                                   capture_output=True, text=True, cwd=ROOT)
                line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-500:]
                print(rep, data, name, line, flush=True)
                try:
                    out.setdefault(f"{data} {name}", []).append(json.loads(line)["ms"])
                except Exception:
                    pass
    print(json.dumps(out))


if __name__ == "__main__":
    main()
