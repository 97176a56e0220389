"""Driver for ncu captures of the 2-byte vt kernels (EXEM_VT_STORAGE), bf16
ground set n = 1M, d = 100: K1 pair kernel (column-major source), K1 slab
kernel (row-major source), K2 set_min_tma at k = 1 and k = 50, and the
m-update pair kernel with the TC h refresh.

    ncu --set full -k regex:"ground_prepare|set_min_tma|greedy_update_pair" \
        -c 5 -o gpurun_out/prof_vt16 python tools/ncu_vt16.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.device import padded_rows, to_device_bytes

    torch.cuda.set_device(0)
    n, d = 1_000_000, 100
    prec = pb.Precision.bfloat16
    V = np.random.default_rng(0).standard_normal((n, d), dtype=np.float32)
    g = pb.build_ground_set(np.asfortranarray(V), precision=prec)
    dg = g.on_device()  # K1 pair kernel (column-major source)
    lib = N.lib()
    st = dg.stream
    src_r = to_device_bytes(np.ascontiguousarray(g.matrix), dg.dev)
    e0 = to_device_bytes(g.aux, dg.dev)
    lib.ground_prepare_rows(dg.vt_tag, N.ptr(src_r), n, d, N.ptr(e0),
                            N.ptr(dg.vt), dg.ld, N.ptr(dg.norms),
                            N.ptr(dg.aux), N.ptr(dg.aux_sum),
                            N.ptr(dg.scratch), 1, st)  # K1 slab kernel
    for k in (1, 50):
        elems = padded_rows(g.matrix[:k], dg.d_pad, prec, dg.dev)
        en = torch.empty(k, dtype=torch.float64, device=dg.dev)
        lib.row_norms(prec.tag, N.ptr(elems), k, d, dg.d_pad, N.ptr(en), st)
        s = torch.empty(1, dtype=torch.float64, device=dg.dev)
        lib.set_min(dg.vt_tag, N.ptr(dg.vt), dg.ld, n, d, N.ptr(dg.norms),
                    N.ptr(dg.aux), N.ptr(elems), N.ptr(en), k, 1, None, None,
                    N.ptr(s), N.ptr(dg.scratch), st)
    m = dg.aux.clone()
    xp = torch.zeros((int(lib.tc_rows(n)), dg.kp), dtype=dg.vt.dtype,
                     device=dg.dev)
    sel = torch.zeros(1, dtype=torch.int64, device=dg.dev)
    msum = torch.empty(1, dtype=torch.float64, device=dg.dev)
    lib.greedy_update(dg.vt_tag, N.ptr(dg.vt), dg.ld, n, d, N.ptr(dg.norms),
                      N.ptr(dg.vt), dg.ld, N.ptr(dg.norms), N.ptr(sel), 0,
                      N.ptr(m), N.ptr(xp), dg.kp, N.ptr(msum),
                      N.ptr(dg.scratch), st)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
