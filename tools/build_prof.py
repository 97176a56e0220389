"""Host-side cost of build_ground_set at BASELINE config 4 (n = 1M, d = 100):
validation, the storage-dtype cast, and the whole build (upload + K1), for a
row-major (C-order) and a column-major input.

    python tools/build_prof.py
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2101_08763_b200 as pb  # noqa: E402
from paper_2101_08763_b200.core import _as_observation_matrix  # noqa: E402


def main():
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
    V = np.random.default_rng(0).standard_normal((1_000_000, 100),
                                                 dtype=np.float32)
    prec = pb.Precision.bfloat16
    pb.build_ground_set(V[:1000], precision=prec)
    t0 = time.perf_counter()
    arr = _as_observation_matrix(V)
    t1 = time.perf_counter()
    arr.astype(prec.dtype, copy=False)
    t2 = time.perf_counter()
    print(f"validate {t1 - t0:.3f} s  cast {t2 - t1:.3f} s")
    for name, src in (("C-order", V), ("F-order", np.asfortranarray(V))):
        for _ in range(2):
            t = time.perf_counter()
            g = pb.build_ground_set(src, precision=prec)
            torch.cuda.synchronize()
            print(f"{name} build total {time.perf_counter() - t:.3f} s")
        t = time.perf_counter()
        pb.greedy_maximize(g, k=1)
        torch.cuda.synchronize()
        print(f"{name} greedy k=1 (incl packs) {time.perf_counter() - t:.3f} s")


if __name__ == "__main__":
    main()
