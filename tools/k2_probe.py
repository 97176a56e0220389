"""Launch K2 set_min once per k (n = 1M, d = 100, binary32) for an ncu
capture:  ncu --set full -k regex:set_min -c <len(ks)> python tools/k2_probe.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.device import padded_rows

    ks = [int(x) for x in (sys.argv[1:] or ["1", "50"])]
    n, d = 1_000_000, 100
    V = np.random.default_rng(0).standard_normal((n, d), dtype=np.float32)
    prec = pb.Precision.binary32
    g = pb.build_ground_set(V, precision=prec)
    dg = g.on_device()
    lib = N.lib()
    st = N.stream_handle()
    for k in ks:
        elems = padded_rows(g.matrix[:k], dg.d_pad, prec, dg.dev)
        en = torch.empty(k, dtype=torch.float64, device=dg.dev)
        lib.row_norms(prec.tag, N.ptr(elems), k, d, dg.d_pad, N.ptr(en), st)
        s = torch.empty(1, dtype=torch.float64, device=dg.dev)
        lib.set_min(dg.vt_tag, N.ptr(dg.vt), dg.ld, n, d, N.ptr(dg.norms),
                    N.ptr(dg.aux), N.ptr(elems), N.ptr(en), k, 1, None, None,
                    N.ptr(s), N.ptr(dg.scratch), st)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
