"""SieveStreaming throughput (elements/s) by block size, one B200.

    python tools/sieve_bench.py [--n 100000] [--d 100] [--k 50] [--eps 0.1]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--d", type=int, default=100)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--eps", type=float, default=0.1)
    ap.add_argument("--stream", type=int, default=20_000)
    ap.add_argument("--blocks", default="1,64")
    a = ap.parse_args()
    import torch

    import paper_2101_08763_b200 as pb

    V = np.random.default_rng(0).standard_normal((a.n, a.d), dtype=np.float32)
    g = pb.build_ground_set(V, precision=pb.Precision.binary32)
    order = np.arange(a.stream)
    out = {}
    for blk in (int(x) for x in a.blocks.split(",")):
        pb.sieve_streaming_maximize(g, a.k, a.eps, order=order[:blk], block=blk)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pb.sieve_streaming_maximize(g, a.k, a.eps, order=order,
                                          block=blk)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[blk] = res
        print(json.dumps({"n": a.n, "d": a.d, "k": a.k, "eps": a.eps,
                          "stream": a.stream, "block": blk, "s": dt,
                          "elements_per_s": a.stream / dt,
                          "picked": len(res.exemplar_indices),
                          "f": res.values[-1] if res.values else 0.0}),
              flush=True)
    ref = next(iter(out.values()))
    print("same picks across blocks:",
          all(r.exemplar_indices == ref.exemplar_indices for r in out.values()))


if __name__ == "__main__":
    main()
