"""Time K2 set_min (n = 1M, d = 100, binary32) for k in KS under the current
environment (EXEM_K2_* experiment knobs); one JSON line."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))


def main():
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.device import padded_rows
    from hbm_kernels import timed

    n, d = 1_000_000, 100
    V = np.random.default_rng(0).standard_normal((n, d), dtype=np.float32)
    prec = pb.Precision.binary32
    g = pb.build_ground_set(V, precision=prec)
    dg = g.on_device()
    lib = N.lib()
    st = N.stream_handle()
    out = {}
    for k in (1, 10, 50):
        elems = padded_rows(g.matrix[:k], dg.d_pad, prec, dg.dev)
        en = torch.empty(k, dtype=torch.float64, device=dg.dev)
        lib.row_norms(prec.tag, N.ptr(elems), k, d, dg.d_pad, N.ptr(en), st)
        s = torch.empty(1, dtype=torch.float64, device=dg.dev)
        out[k] = round(timed(lambda: lib.set_min(
            dg.vt_tag, N.ptr(dg.vt), dg.ld, n, d, N.ptr(dg.norms),
            N.ptr(dg.aux), N.ptr(elems), N.ptr(en), k, 1, None, None,
            N.ptr(s), N.ptr(dg.scratch), st), reps=10) * 1e3, 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
