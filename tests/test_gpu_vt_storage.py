"""2-byte V for half ground sets (EXEM_VT_STORAGE, include/exem_b200.h).

bf16/f16 ground sets keep the column-major ``vt`` at the storage type; K1
writes it, and K2 set_min (TMA kernel), the Greedy m-update and the TC
operand packers read it, widening in registers.  The arithmetic is that of
the binary32-widened layout (the values are the same), so every output is
compared BIT FOR BIT against the same entry point run on the widening
(``DeviceGround.vt_c()``, unflagged tag) -- and the widened layout itself is
pinned to the oracle by the rest of the suite.  Reference paths:
objective.py:113-141 (min_distances), evaluate.py:105-112 (_set_value),
optimize.py:74-76 (m-update), optimize.py:115-136 (assign_clusters).
"""

import numpy as np
import pytest

import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import _native as N
from paper_2101_08763_b200.device import padded_rows
from paper_2101_08763_b200.errors import DimensionMismatchError

pytestmark = pytest.mark.gpu

HALVES = [pb.Precision.bfloat16, pb.Precision.binary16]


def _ground(prec, n, d, seed=0):
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((n, d)).astype(np.float32)
    return pb.build_ground_set(V, precision=prec), rng


@pytest.mark.parametrize("prec", HALVES, ids=lambda p: p.value)
def test_vt_is_two_byte_and_widening_exact(prec):
    import torch

    g, _ = _ground(prec, 3000, 37)
    dg = g.on_device()
    assert dg.vt.element_size() == 2 and dg.vt_flag == N.VT_STORAGE
    assert dg.vt.shape == (dg.d_pad, dg.ld)
    wide = dg.vt_c()
    assert wide.dtype == torch.float32
    assert torch.equal(wide, dg.vt.float())
    # padding dimensions and points are zero
    assert not dg.vt[g.d:].any() and not dg.vt[:, g.n:].any()
    # the stored values are the reference's storage values
    assert np.array_equal(dg.column_major_storage(), g.matrix)


@pytest.mark.parametrize("prec", HALVES + [pb.Precision.binary32],
                         ids=lambda p: p.value)
@pytest.mark.parametrize("n,d", [(3000, 37), (3001, 37), (256, 100), (1, 5),
                                 (2999, 100), (1000, 220), (700, 400)])
@pytest.mark.parametrize("misalign", [False, True], ids=["aligned", "offset"])
def test_k1_layouts_bit_equal(prec, n, d, misalign):
    """K1 over every source layout and vt element type gives the same
    norms, aux, fixed-order aux sum and vt: column-major source (the pair
    kernel for even n with 2-byte vt, the one-point kernel otherwise) and
    row-major source (the shared-memory slab kernel, or the 32-dimension
    tile kernel when the slab does not fit), each writing 2-byte or
    binary32 vt.  ``offset``: the source starts one value past a 16-byte
    boundary (the pair / slab kernels step aside for the scalar ones)."""
    import torch

    from paper_2101_08763_b200.device import to_device_bytes

    g, _ = _ground(prec, n, d, seed=n + d)
    dg = g.on_device()
    lib = N.lib()
    st = dg.stream
    e0 = to_device_bytes(g.aux, dg.dev)
    tags = [(prec.tag, torch.float32)]
    if dg.vt_flag:
        tags.append((dg.vt_tag, dg.vt.dtype))
    out = []
    for rows in (False, True):
        host = np.ascontiguousarray(g.matrix) if rows else \
            np.asfortranarray(g.matrix)
        raw = to_device_bytes(host.ravel(order="C" if rows else "F"), dg.dev)
        off = prec.bytes_per_value if misalign else 0
        buf = torch.zeros(raw.numel() + 16, dtype=torch.uint8, device=dg.dev)
        buf[off:off + raw.numel()].copy_(raw)
        src = N.c_void_p(buf.data_ptr() + off)
        prep = lib.ground_prepare_rows if rows else lib.ground_prepare
        for tag, vdt in tags:
            vt = torch.full((dg.d_pad, dg.ld), 7, dtype=vdt, device=dg.dev)
            norms = torch.empty(dg.ld, dtype=torch.float64, device=dg.dev)
            aux = torch.empty(dg.ld, dtype=torch.float32, device=dg.dev)
            s = torch.empty(1, dtype=torch.float64, device=dg.dev)
            prep(tag, src, n, d, N.ptr(e0), N.ptr(vt), dg.ld,
                 N.ptr(norms), N.ptr(aux), N.ptr(s), N.ptr(dg.scratch), 1, st)
            out.append((vt.float().cpu(), norms.cpu(), aux.cpu(), s.item()))
    v0, n0, a0, s0 = out[0]
    for v1, n1, a1, s1 in out[1:]:
        assert torch.equal(v0, v1)
        assert torch.equal(n0, n1) and torch.equal(a0, a1)
        assert s0 == s1


@pytest.mark.parametrize("prec", HALVES, ids=lambda p: p.value)
@pytest.mark.parametrize("n,d,k", [(5000, 100, 1), (5000, 100, 10),
                                   (4099, 37, 50), (4099, 100, 64),
                                   (3000, 16, 100), (2000, 300, 20)])
def test_set_min_storage_bit_equal(prec, n, d, k):
    import torch

    g, rng = _ground(prec, n, d, seed=k)
    dg = g.on_device()
    lib = N.lib()
    idx = np.sort(rng.choice(n, size=k, replace=False))
    st = dg.stream
    e = padded_rows(g.matrix[idx], dg.d_pad, prec, dg.dev)
    en = torch.empty(k, dtype=torch.float64, device=dg.dev)
    lib.row_norms(prec.tag, N.ptr(e), k, d, dg.d_pad, N.ptr(en), st)
    assert lib.set_min_storage_ok(dg.vt_tag, d, k, 1) == 1
    outs = []
    for tag, vt in ((dg.vt_tag, dg.vt), (prec.tag, dg.vt_c())):
        t_out = torch.empty(n, dtype=torch.float32, device=dg.dev)
        lab = torch.empty(n, dtype=torch.int64, device=dg.dev)
        s = torch.empty(1, dtype=torch.float64, device=dg.dev)
        lib.set_min(tag, N.ptr(vt), dg.ld, n, d, N.ptr(dg.norms),
                    N.ptr(dg.aux), N.ptr(e), N.ptr(en), k, 1, N.ptr(t_out),
                    N.ptr(lab), N.ptr(s), N.ptr(dg.scratch), st)
        outs.append((t_out.cpu().numpy(), lab.cpu().numpy(), s.item()))
    (t0, l0, s0), (t1, l1, s1) = outs
    assert np.array_equal(t0.view(np.uint32), t1.view(np.uint32))
    assert np.array_equal(l0, l1)
    assert s0 == s1


@pytest.mark.parametrize("prec", HALVES, ids=lambda p: p.value)
def test_public_api_storage_equals_widened(prec, monkeypatch):
    """evaluate_single / min_distances / assign_clusters through the public
    API (storage path) equal the same calls forced onto the widening."""
    g, rng = _ground(prec, 6000, 64, seed=3)
    idx = np.sort(rng.choice(6000, size=40, replace=False))
    elems = g.matrix[idx]
    f_s = pb.evaluate_single(g, elems)
    t_s = pb.min_distances(g, elems)
    lab_s = pb.assign_clusters(g, elems)
    # the predicate patched to 0 sends every K2 call to vt_c()
    monkeypatch.setattr(type(N.lib()), "set_min_storage_ok",
                        lambda self, *a: 0, raising=False)
    g2 = pb.build_ground_set(np.asarray(g.matrix, np.float32), precision=prec)
    f_w = pb.evaluate_single(g2, elems)
    t_w = pb.min_distances(g2, elems)
    lab_w = pb.assign_clusters(g2, elems)
    assert f_s == f_w
    assert np.array_equal(np.asarray(t_s), np.asarray(t_w))
    assert np.array_equal(lab_s, lab_w)


@pytest.mark.parametrize("prec", HALVES, ids=lambda p: p.value)
def test_greedy_update_and_pack_storage_bit_equal(prec):
    import torch

    n, d = 4099, 100
    g, _ = _ground(prec, n, d, seed=7)
    dg = g.on_device()
    lib = N.lib()
    st = dg.stream
    res = []
    for tag, vt in ((dg.vt_tag, dg.vt), (prec.tag, dg.vt_c())):
        m = dg.aux.clone()
        xp = torch.zeros((int(lib.tc_rows(n)), dg.kp), dtype=dg.vt.dtype,
                         device=dg.dev)
        lib.tc_pack_points(tag, N.ptr(vt), dg.ld, n, d, N.ptr(dg.norms),
                           N.ptr(m), N.ptr(xp), st)
        xc = torch.zeros_like(xp)
        lib.tc_pack_candidates(tag, N.ptr(vt), dg.ld, n, d, N.ptr(dg.norms),
                               N.ptr(xc), st)
        sel = torch.tensor([17, 4000], dtype=torch.int64, device=dg.dev)
        msum = torch.zeros(2, dtype=torch.float64, device=dg.dev)
        for step in range(2):
            lib.greedy_update(tag, N.ptr(vt), dg.ld, n, d, N.ptr(dg.norms),
                              N.ptr(vt), dg.ld, N.ptr(dg.norms), N.ptr(sel),
                              step, N.ptr(m), N.ptr(xp), dg.kp, N.ptr(msum),
                              N.ptr(dg.scratch), st)
        plain = torch.zeros((int(lib.tc_rows(n)), int(lib.tc_batch_kp(d))),
                            dtype=dg.vt.dtype, device=dg.dev)
        lib.tc_pack_points_plain(tag, N.ptr(vt), dg.ld, n, d, N.ptr(plain), st)
        res.append([x.cpu() for x in (m, xp, xc, msum, plain)])
    for a, b in zip(*res):
        assert torch.equal(a.contiguous().view(torch.uint8),
                           b.contiguous().view(torch.uint8))


def test_storage_flag_rejected_for_wide_tags():
    import torch

    g, _ = _ground(pb.Precision.binary32, 600, 8)
    dg = g.on_device()
    lib = N.lib()
    m = dg.aux.clone()
    sel = torch.zeros(1, dtype=torch.int64, device=dg.dev)
    s = torch.zeros(1, dtype=torch.float64, device=dg.dev)
    with pytest.raises(DimensionMismatchError, match="EXEM_VT_STORAGE"):
        lib.greedy_update(N.F32 | N.VT_STORAGE, N.ptr(dg.vt), dg.ld, g.n, g.d,
                          N.ptr(dg.norms), N.ptr(dg.vt), dg.ld,
                          N.ptr(dg.norms), N.ptr(sel), 0, N.ptr(m), None, 0,
                          N.ptr(s), N.ptr(dg.scratch), dg.stream)
    assert lib.set_min_storage_ok(N.F32 | N.VT_STORAGE, 8, 4, 1) == 0
    # entry points that do not take the flag reject it loudly
    out = torch.zeros((dg.d_pad, dg.ld), dtype=torch.float32, device=dg.dev)
    with pytest.raises(DimensionMismatchError, match="unknown dtype"):
        lib.widen_packed(N.BF16 | N.VT_STORAGE, N.ptr(dg.vt), dg.ld, dg.ld, 1,
                         dg.d_pad, N.ptr(out), dg.stream)
