"""A few K3-TC Greedy steps at C4 size on a chosen data shape, for ncu:
    ncu --set full -k regex:gains_tc -s 2 -c 1 python tools/k3_probe_data.py blobs
(data: gauss | blobs -- the 16-blob mixture of tools/bench_configs.blobs)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))


def main():
    import torch

    import paper_2101_08763_b200 as pb
    from bench_configs import blobs, gaussian

    kind = sys.argv[1] if len(sys.argv) > 1 else "blobs"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    n, d = 1_000_000, 100
    V = blobs(n, d, 3) if kind == "blobs" else gaussian(n, d, 0)
    g = pb.build_ground_set(V, precision=pb.Precision.bfloat16)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    res = pb.greedy_maximize(g, k=steps)
    t1.record()
    torch.cuda.synchronize()
    print(kind, res.exemplar_indices, f"{t0.elapsed_time(t1) / steps:.1f} ms/step")


if __name__ == "__main__":
    main()
