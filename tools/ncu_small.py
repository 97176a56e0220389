"""Driver for ncu captures of the CUDA-core kernels (run under ncu):
K3-SIMT fp32 gains (C2 shape: n = 100k, d = 100), K2 set_min (k = 10) and
the Greedy m-update at n = 1M, d = 100.

    ncu --set full -k regex:"gains_simt|set_min|greedy_update" -c 3 \
        -o gpurun_out/prof_simt python tools/ncu_small.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200.optimize import GreedyRun

    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    V = rng.standard_normal((100_000, 100), dtype=np.float32)
    g = pb.build_ground_set(V, precision=pb.Precision.binary32)
    run = GreedyRun(g.on_device(), k_cap=2)
    run.start()
    run.compute_gains()  # gains_simt_kernel (C2 shape)
    W = rng.standard_normal((1_000_000, 100), dtype=np.float32)
    g2 = pb.build_ground_set(W, precision=pb.Precision.binary32)
    pb.evaluate_single(g2, g2.matrix[:10])  # set_min_kernel, k = 10
    r2 = GreedyRun(g2.on_device(), k_cap=1)
    r2.start()
    r2.sel_idx.zero_()
    r2.update(0)  # greedy_update_kernel
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
