"""Low-memory regime: ground sets larger than the device budget.

North-star item (c) / BASELINE config 5.  The paper's low-memory scheme
chunks the evaluation sets under a memory budget with V preloaded
(reference ``evaluate_chunked`` evaluate.py:296-319); here
V itself is tiled as well, so a ground set far larger than one GPU's budget
streams through it:

* V stays in host memory (the F-order ``GroundSet.matrix``, page-locked
  once with ``exem_host_register``).
* The device holds a two-slot ring of **row slices**.  A slice is a run of
  whole partial-sum splits (``exem_split_points`` of the global n), so every
  per-point term lands in the same split -- and the same fixed-order sum --
  as in a resident run: streamed results are bit-identical to resident ones.
* Slice s+1 is uploaded (``exem_h2d_rows``: one 2-D DMA of the column-major
  slice) on a copy stream while slice s is prepared (K1 into the SIMT layout
  and, for half storage, the tensor-core point operand) and evaluated on the
  compute stream; two events per slot order the reuse.
* Sums whose reference order is the per-256-point block partials (K1's
  aux sum, K2's per-set sum) are written at their global block offsets and
  reduced once at the end (``exem_sum_fixed``), again bit-identical.

Sharding (``distributed.py``) composes with this: a rank streams its own
row range.
"""

from __future__ import annotations

import weakref
from ctypes import c_void_p
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import OutOfMemoryError


def _csize(precision) -> int:
    return 8 if precision.compute_dtype == np.float64 else 4


def layout_bytes(rows: int, d: int, precision, with_src: bool = False,
                 tc_operands: int = 1, vt_storage: bool = False) -> int:
    """Device bytes of the layouts of ``rows`` points:
    SIMT vt + norms + aux, plus ``tc_operands`` half operands for the
    half precisions, plus the raw upload buffer when ``with_src``.
    ``vt_storage``: vt at the 2-byte storage type of a half ground set (the
    resident layout, EXEM_VT_STORAGE); streamed slots keep it widened."""
    lib = N.lib()
    ld = int(lib.pad_points(rows))
    d_pad = int(lib.pad_dims(d))
    cs = _csize(precision)
    vs = precision.bytes_per_value if (vt_storage and precision.is_half) \
        else cs
    b = d_pad * ld * vs + ld * 8 + ld * cs
    if precision.is_half:
        kp = max(int(lib.tc_kp(d)), int(lib.tc_batch_kp(d)))
        b += tc_operands * int(lib.tc_rows(rows)) * kp * 2
    if with_src:
        b += rows * d * precision.bytes_per_value
    return b


def resident_bytes(n: int, d: int, precision) -> int:
    """Bytes of a fully resident ground set (incl. the reduction scratch)."""
    lib = N.lib()
    return (layout_bytes(n, d, precision, tc_operands=2, vt_storage=True) +
            int(lib.reduce_scratch(int(lib.pad_points(n)))) * 8)


@dataclass(frozen=True)
class StreamPlan:
    """Row slices of a streamed ground set."""

    rows_per_slice: int
    slices: tuple          # ((r0, r1), ...), split-aligned
    slot_bytes: int


def plan_slices(n: int, d: int, precision, free_bytes: int,
                split_pts: int = None) -> StreamPlan:
    """Largest split-aligned slice such that two ring slots fit the budget;
    ``OutOfMemoryError`` when not even one split per slot fits (the same
    error the reference raises for a budget below one set,
    evaluate.py:91-95)."""
    lib = N.lib()
    sp = int(split_pts or lib.split_points(n))
    per_slot = lambda r: layout_bytes(r, d, precision, with_src=True)  # noqa: E731
    if 2 * per_slot(min(sp, n)) > free_bytes:
        raise OutOfMemoryError(
            f"a streamed slice of {sp} points needs {2 * per_slot(sp)} bytes "
            f"of ring buffers but only {free_bytes} are free")
    splits = -(-n // sp)
    lo, hi = 1, splits
    while lo < hi:  # most splits per slice that still fit
        mid = (lo + hi + 1) // 2
        if 2 * per_slot(min(mid * sp, n)) <= free_bytes:
            lo = mid
        else:
            hi = mid - 1
    rows = min(lo * sp, n)
    slices = tuple((r0, min(n, r0 + rows)) for r0 in range(0, n, rows))
    return StreamPlan(rows_per_slice=rows, slices=slices,
                      slot_bytes=per_slot(rows))


def _unpin(matrix, ptr):
    try:
        N.lib().host_unregister(c_void_p(ptr))
    except Exception:
        pass
    del matrix


def pin_host(ground) -> None:
    """Page-lock the host matrix once per ground set (async DMA source);
    unlocked when the ground set is collected."""
    pinned = getattr(ground, "_pinned", None)
    if pinned is None or pinned.get("done"):
        return
    m = ground.matrix
    pinned["done"] = True
    try:
        N.lib().host_register(c_void_p(m.ctypes.data), m.nbytes)
    except Exception:
        # e.g. a read-only file mapping the driver refuses to lock: the 2-D
        # DMA then stages through pageable memory (slower, still correct)
        return
    weakref.finalize(ground, _unpin, m, m.ctypes.data)


class _Slot:
    """One ring slot: device layouts of up to ``cap`` points.  Exposes the
    attributes the batch kernels read from a ``DeviceGround``."""

    def __init__(self, cap, d, precision, dev, device_index):
        from .device import compute_torch_dtype, torch

        t = torch()
        lib = N.lib()
        self.d, self.precision, self.dev = d, precision, dev
        self.device_index = device_index
        self.d_pad = int(lib.pad_dims(d))
        ldc = int(lib.pad_points(cap))
        cdt = compute_torch_dtype(precision)
        self.src = t.empty(cap * d * precision.bytes_per_value,
                           dtype=t.uint8, device=dev)
        self._vt = t.empty(self.d_pad * ldc, dtype=cdt, device=dev)
        self.norms = t.empty(ldc, dtype=t.float64, device=dev)
        self.aux = t.empty(ldc, dtype=cdt, device=dev)
        self.kp = int(lib.tc_kp(d)) if precision.is_half else 0
        self.plain = bool(precision.is_half and lib.tc_batch_plain(d))
        self._xp = None
        if precision.is_half:
            tdt = t.bfloat16 if precision.tag == N.BF16 else t.float16
            kp = max(self.kp, int(lib.tc_batch_kp(d)))
            self._xp = t.empty((int(lib.tc_rows(cap)), kp), dtype=tdt,
                               device=dev)
        self.uploaded = t.cuda.Event()
        self.consumed = t.cuda.Event()
        self.n = 0
        self.ld = 0

    @property
    def vt(self):
        return self._vt[: self.d_pad * self.ld].view(self.d_pad, self.ld)

    # a slot's vt is always at the compute type (the streamed path keeps
    # the widened layout; DeviceGround keeps half storage at 2 bytes)
    vt_flag = 0

    def vt_c(self):
        return self.vt

    @property
    def vt_tag(self) -> int:
        return self.precision.tag

    @property
    def stream(self):
        return N.stream_handle(self.dev)

    def xp0(self):
        return self._xp

    def xp_batch(self):
        """K4-TC point operand of the slice (packed by ``slices``)."""
        return self._xp


class GroundStream:
    """Streams the rows [row0, row1) of a host ground set through a
    two-slot device ring (see module docstring)."""

    def __init__(self, ground, free_bytes: int, device=None, rows=None):
        from .device import require_cuda, to_device_bytes, torch

        t = torch()
        self.t = t
        self.lib = N.lib()
        self.ground = ground
        self.idx = require_cuda(device)
        self.dev = t.device("cuda", self.idx)
        self.prec = ground.precision
        self.n, self.d = ground.n, ground.d
        self.split_pts = int(self.lib.split_points(self.n))
        self.row0, self.row1 = rows if rows is not None else (0, self.n)
        if self.row0 % self.split_pts:
            raise ValueError("a streamed row range must start on a split")
        self.plan = plan_slices(self.row1 - self.row0, self.d, self.prec,
                                free_bytes, self.split_pts)
        from .device import row_major

        host = ground.matrix
        self.row_major = row_major(host)
        self.check_finite = False  # set by stream_build (K1 NaN marker)
        assert self.row_major or host.flags.f_contiguous
        self._host_ptr = c_void_p(host.ctypes.data)
        with t.cuda.device(self.idx):
            pin_host(ground)
            self.e0 = to_device_bytes(ground.aux, self.dev)
            blocks = int(self.lib.pad_points(self.n)) // 256 + 8
            self.block_partials = t.zeros(blocks, dtype=t.float64,
                                          device=self.dev)
            cap = self.plan.rows_per_slice
            self.slots = [_Slot(cap, self.d, self.prec, self.dev, self.idx)
                          for _ in range(2)]
            self.copy_stream = t.cuda.Stream(self.dev)

    def close(self):
        """Release the ring (the host pages stay locked for reuse)."""
        self.slots = []

    def upload(self, dst, r0: int, rows: int, stream) -> None:
        """Rows [r0, r0+rows) of the host matrix -> the device staging
        buffer, in the host's own layout (2-D DMA of a column-major slice,
        or one contiguous copy of a row-major slice)."""
        bpv = self.prec.bytes_per_value
        if self.row_major:
            self.lib.h2d_bytes(N.ptr(dst), c_void_p(self._host_ptr.value +
                                                    r0 * self.d * bpv),
                               rows * self.d * bpv, stream)
        else:
            self.lib.h2d_rows(N.ptr(dst), self._host_ptr, self.n, r0, rows,
                              self.d, bpv, stream)

    def prepare(self, src, rows, vt, ld, norms, aux, partials, stream):
        """K1 on an uploaded slice (row- or column-major source)."""
        fn = (self.lib.ground_prepare_rows if self.row_major
              else self.lib.ground_prepare)
        fn(self.prec.tag, src, rows, self.d, N.ptr(self.e0), vt, ld, norms,
           aux, None, partials, int(self.check_finite), stream)

    def block_ptr(self, r0: int) -> c_void_p:
        return c_void_p(self.block_partials.data_ptr() + (r0 // 256) * 8)

    def slices(self, pack_points: bool = True):
        """Yield (slot, r0, r1) with the slot's layouts ready on the current
        stream; r0/r1 are global row indices.  K1's aux block partials land
        in ``block_partials`` at the slice's global block offset."""
        t, lib, prec = self.t, self.lib, self.prec
        with t.cuda.device(self.idx):
            compute = t.cuda.current_stream(self.dev)
            st = N.stream_handle(self.dev)
            for s, (a, b) in enumerate(self.plan.slices):
                r0, r1 = self.row0 + a, self.row0 + b
                rows = r1 - r0
                slot = self.slots[s % 2]
                cs = self.copy_stream
                cs.wait_event(slot.consumed)  # K1 of the slot's last use done
                with t.cuda.stream(cs):
                    self.upload(slot.src, r0, rows, c_void_p(cs.cuda_stream))
                    slot.uploaded.record(cs)
                compute.wait_event(slot.uploaded)
                slot.n = rows
                slot.ld = int(lib.pad_points(rows))
                self.prepare(N.ptr(slot.src), rows, N.ptr(slot.vt), slot.ld,
                             N.ptr(slot.norms), N.ptr(slot.aux),
                             self.block_ptr(r0), st)
                slot.consumed.record(compute)
                if prec.is_half and pack_points:
                    if slot.plain:
                        lib.tc_pack_points_plain(prec.tag, N.ptr(slot.vt),
                                                 slot.ld, rows, self.d,
                                                 N.ptr(slot.xp_batch()), st)
                    else:
                        lib.tc_pack_points(prec.tag, N.ptr(slot.vt), slot.ld,
                                           rows, self.d, N.ptr(slot.norms),
                                           None, N.ptr(slot.xp0()), st)
                yield slot, r0, r1


# ---------------------------------------------------------------- consumers
def stream_build(ground, free_bytes: int, device=None,
                 check_finite: bool = False):
    """Streamed K1: (aux_distances host array, fixed-order aux sum; NaN iff
    ``check_finite`` and V holds a non-finite stored value)."""
    from .device import aux_dtype, torch

    t = torch()
    gs = GroundStream(ground, free_bytes - _margin(ground.n), device)
    gs.check_finite = check_finite
    try:
        with t.cuda.device(gs.idx):
            cdt = t.float64 if ground.precision.compute_dtype == np.float64 \
                else t.float32
            host_aux = t.empty(ground.n, dtype=cdt, pin_memory=True)
            f16 = ground.precision.tag == N.F16
            max_norm = t.zeros((), dtype=t.float64, device=gs.dev)
            for slot, r0, r1 in gs.slices(pack_points=False):
                host_aux[r0:r1].copy_(slot.aux[: r1 - r0], non_blocking=True)
                if f16:  # range of the folded tensor-core operands
                    t.maximum(max_norm, slot.norms[: r1 - r0].max(),
                              out=max_norm)
            total = t.empty(1, dtype=t.float64, device=gs.dev)
            count = -(-int(gs.lib.pad_points(ground.n)) // 256)
            gs.lib.sum_fixed(N.ptr(gs.block_partials), count, N.ptr(total), 0,
                             N.stream_handle(gs.dev))
            t.cuda.synchronize(gs.dev)
            aux = host_aux.numpy().astype(aux_dtype(ground.precision))
            ground._ext()["max_norm"] = float(max_norm.item())
            return aux, float(total.item())
    finally:
        gs.close()


def stream_set_min(ground, elems: np.ndarray, include_aux: bool,
                   want_t: bool, want_labels: bool, device=None):
    """Streamed K2 over one explicit set: (sum_t, t, labels) exactly as the
    resident ``device_set_min``."""
    from .device import padded_rows, torch

    t = torch()
    lib = N.lib()
    prec = ground.precision
    n, k = ground.n, int(elems.shape[0])
    fixed = n * (8 if want_labels else 0) + n * _csize(prec) * int(want_t) + \
        k * 8 * int(lib.pad_dims(ground.d)) + _margin(n)
    gs = GroundStream(ground, ground.device_budget - fixed, device)
    try:
        with t.cuda.device(gs.idx):
            st = N.stream_handle(gs.dev)
            e = padded_rows(elems, int(lib.pad_dims(ground.d)), prec, gs.dev)
            en = t.empty(max(k, 1), dtype=t.float64, device=gs.dev)
            if k:
                lib.row_norms(prec.tag, N.ptr(e), k, ground.d,
                              int(lib.pad_dims(ground.d)), N.ptr(en), st)
            cdt = gs.slots[0].aux.dtype
            t_out = t.empty(n, dtype=cdt, device=gs.dev) if want_t else None
            lab = t.empty(n, dtype=t.int64, device=gs.dev) if want_labels else None
            for slot, r0, r1 in gs.slices(pack_points=False):
                tp = c_void_p(t_out.data_ptr() + r0 * t_out.element_size()) \
                    if want_t else None
                lp = c_void_p(lab.data_ptr() + r0 * 8) if want_labels else None
                lib.set_min(prec.tag, N.ptr(slot.vt), slot.ld, r1 - r0,
                            ground.d, N.ptr(slot.norms), N.ptr(slot.aux),
                            N.ptr(e), N.ptr(en), k, int(include_aux), tp, lp,
                            None, gs.block_ptr(r0), st)
            s = t.empty(1, dtype=t.float64, device=gs.dev)
            lib.sum_fixed(N.ptr(gs.block_partials), -(-n // 256), N.ptr(s), 0,
                          st)
            total = float(s.item())
            return (total, t_out.cpu().numpy() if want_t else None,
                    lab.cpu().numpy() if want_labels else None)
    finally:
        gs.close()


def batch_device_bytes(d: int, k_max: int, l: int, precision,
                       splits: int) -> int:
    """Device bytes of an uploaded batch + its partial sums."""
    lib = N.lib()
    l_pad = -(-l // 128) * 128
    b = int(lib.pad_dims(d)) * k_max * l_pad * _csize(precision)
    b += k_max * l_pad * 8 + 4 * l + splits * l * 8 + 8 * l
    if precision.is_half and k_max <= 256:
        b += int(lib.tc_set_rows(l, k_max)) * (int(lib.tc_batch_kp(d)) * 2 + 4)
    return b


def stream_packed_sums(ground, values, d, k_max, l, cardinalities,
                       device=None, rows=None, partial=None, budget=None,
                       sets=None):
    """Streamed K4 / K4-TC: per-set fp64 sums over the rows [row0, row1)
    (all rows by default).  With ``partial`` given (a [splits][l] fp64
    device tensor), the per-split partials are written there at their
    global split rows and no reduction is done (the sharded caller reduces
    after its collective)."""
    from .device import ground_fold_ok, torch
    from .evaluate import DeviceBatch, batch_partials

    t = torch()
    lib = N.lib()
    prec = ground.precision
    n = ground.n
    sp = int(lib.split_points(n))
    splits = -(-n // sp)
    fixed = batch_device_bytes(d, k_max, l, prec, splits) + _margin(n)
    budget = budget if budget is not None else ground.device_budget
    gs = GroundStream(ground, budget - fixed, device, rows=rows)
    try:
        with t.cuda.device(gs.idx):
            st = N.stream_handle(gs.dev)
            batch = DeviceBatch(values, d, k_max, l, cardinalities, prec,
                                int(lib.pad_dims(d)), gs.dev, st, sets=sets,
                                ground_fold_ok=ground_fold_ok(ground))
            own = partial is None
            if own:
                partial = t.zeros((splits, l), dtype=t.float64, device=gs.dev)
            for slot, r0, r1 in gs.slices(pack_points=batch.xs is not None):
                s0 = r0 // sp
                ptr = c_void_p(partial.data_ptr() + s0 * l * 8)
                batch_partials(slot, batch, ptr, sp, -(-(r1 - r0) // sp))
            if not own:
                return partial
            sums = t.empty(l, dtype=t.float64, device=gs.dev)
            lib.reduce_partials(N.ptr(partial), splits, l, 1.0, N.ptr(sums),
                                st)
            t.cuda.synchronize(gs.dev)
            return sums
    finally:
        gs.close()


# ------------------------------------------------------------ streamed Greedy
def stream_greedy(ground, k: int, device=None):
    """Greedy (optimize.py:33-82) over a streamed ground set.

    The optimizer-aware state stays on the device (m_i for all n points, the
    selection mask, the gains); V streams through.  Candidates are V itself,
    so they are processed in resident chunks of ``cand_rows`` rows: per step
    and candidate chunk, every point slice is streamed through K3 (SIMT or
    tcgen05) into the [splits][chunk] partials, then K6 reduces them into
    the chunk's gains.  The m-update with the previous pick (K2) is applied
    to each slice on its first pass of the next step (and in one final
    pass), and its per-block partial sums give msum exactly as the resident
    run.  Everything is bit-identical to the resident Greedy.  Returns
    (indices, msum) as host arrays.
    """
    from .device import (compute_torch_dtype, ground_fold_ok, padded_rows,
                         to_device_bytes, torch)

    t = torch()
    lib = N.lib()
    prec = ground.precision
    n, d = ground.n, ground.d
    sp = int(lib.split_points(n))
    splits = -(-n // sp)
    cs = _csize(prec)
    half = prec.is_half
    if half and not ground_fold_ok(ground):
        from .optimize import raise_fold_range

        raise_fold_range(prec)
    budget = ground.device_budget
    state = n * cs + n + 8 * n + 3 * 8 * k + _margin(n) + \
        int(lib.reduce_scratch(max(n, 1))) * 8
    free = budget - state
    # candidate chunk: half of what is left (rows, multiple of 256), the
    # other half for the streaming ring
    per_cand = layout_bytes(256, d, prec, with_src=True) // 256 + splits * 8
    cand_rows = max(256, min(-(-n // 256) * 256,
                             (free // 2) // per_cand // 256 * 256))
    cand_bytes = layout_bytes(cand_rows, d, prec, with_src=True) + \
        splits * cand_rows * 8
    gs = GroundStream(ground, free - cand_bytes, device)
    try:
        with t.cuda.device(gs.idx):
            dev = gs.dev
            st = N.stream_handle(dev)
            cdt = compute_torch_dtype(prec)
            m = t.empty(n, dtype=cdt, device=dev)
            selected = t.zeros(n, dtype=t.uint8, device=dev)
            gains = t.empty(n, dtype=t.float64, device=dev)
            sel_idx = t.zeros(k, dtype=t.int64, device=dev)
            sel_gain = t.zeros(k, dtype=t.float64, device=dev)
            msum = t.zeros(k, dtype=t.float64, device=dev)
            zero_idx = t.zeros(1, dtype=t.int64, device=dev)
            scratch = t.empty(int(lib.reduce_scratch(max(n, 1))),
                              dtype=t.float64, device=dev)
            partial = t.empty((splits, cand_rows), dtype=t.float64, device=dev)
            d_pad = int(lib.pad_dims(d))
            # chosen exemplar in a one-column SIMT layout [d_pad][256]
            chosen = t.zeros((d_pad, 256), dtype=cdt, device=dev)
            cnorm = t.empty(1, dtype=t.float64, device=dev)
            # candidate chunk layouts
            c_src = t.empty(cand_rows * d * prec.bytes_per_value,
                            dtype=t.uint8, device=dev)
            c_ld = int(lib.pad_points(cand_rows))
            c_vt = t.empty(d_pad * c_ld, dtype=cdt, device=dev)
            c_norms = t.empty(c_ld, dtype=t.float64, device=dev)
            c_aux = t.empty(c_ld, dtype=cdt, device=dev)
            c_xc = None
            if half:
                tdt = t.bfloat16 if prec.tag == N.BF16 else t.float16
                c_xc = t.empty((int(lib.tc_rows(cand_rows)),
                                int(lib.tc_kp(d))), dtype=tdt, device=dev)

            def load_candidates(c0, c1):
                rows = c1 - c0
                gs.upload(c_src, c0, rows, st)
                gs.prepare(N.ptr(c_src), rows, N.ptr(c_vt),
                           int(lib.pad_points(rows)), N.ptr(c_norms),
                           N.ptr(c_aux), N.ptr(scratch), st)
                if half:
                    lib.tc_pack_candidates(prec.tag, N.ptr(c_vt),
                                           int(lib.pad_points(rows)), rows, d,
                                           N.ptr(c_norms), N.ptr(c_xc), st)

            def update_slice(slot, r0, r1, step_prev):
                """m <- min(m, d(v, chosen)) on this slice; block partials of
                sum m at the slice's global offset."""
                lib.greedy_update(prec.tag, N.ptr(slot.vt), slot.ld, r1 - r0,
                                  d, N.ptr(slot.norms), N.ptr(chosen), 256,
                                  N.ptr(cnorm), N.ptr(zero_idx), 0,
                                  N.c_void_p(m.data_ptr() + r0 * cs), None,
                                  0, None, gs.block_ptr(r0), st)

            def finish_msum(step):
                lib.sum_fixed(N.ptr(gs.block_partials), -(-n // 256),
                              N.ptr(msum), step, st)

            # S = {}: m = aux (the resident greedy_init), streamed
            for slot, r0, r1 in gs.slices(pack_points=False):
                t_ptr = N.c_void_p(m.data_ptr() + r0 * cs)
                lib.greedy_init(prec.tag, N.ptr(slot.aux), r1 - r0, t_ptr,
                                N.ptr(cnorm), N.ptr(scratch), st)
            for step in range(k):
                for c0 in range(0, n, cand_rows):
                    c1 = min(n, c0 + cand_rows)
                    cl = c1 - c0
                    load_candidates(c0, c1)
                    for slot, r0, r1 in gs.slices(pack_points=False):
                        rows = r1 - r0
                        if step > 0 and c0 == 0:
                            update_slice(slot, r0, r1, step - 1)
                        s0, ns = r0 // sp, -(-rows // sp)
                        part = N.c_void_p(partial.data_ptr() + s0 * cl * 8)
                        m_ptr = N.c_void_p(m.data_ptr() + r0 * cs)
                        if half:
                            lib.tc_pack_points(prec.tag, N.ptr(slot.vt),
                                               slot.ld, rows, d,
                                               N.ptr(slot.norms), m_ptr,
                                               N.ptr(slot.xp0()), st)
                            lib.greedy_gains_tc(prec.tag, N.ptr(c_xc), cl,
                                                N.ptr(slot.xp0()), rows, d, sp,
                                                part, ns, st)
                        else:
                            lib.greedy_gains_simt(prec.tag, N.ptr(c_vt),
                                                  int(lib.pad_points(cl)),
                                                  N.ptr(c_norms), cl,
                                                  N.ptr(slot.vt), slot.ld,
                                                  N.ptr(slot.norms), m_ptr,
                                                  rows, d, sp, part, ns, st)
                    if step > 0 and c0 == 0:
                        finish_msum(step - 1)
                    lib.reduce_partials(N.ptr(partial), splits, cl, 2.0,
                                        N.c_void_p(gains.data_ptr() + c0 * 8),
                                        st)
                lib.argmax_select(N.ptr(gains), n, N.ptr(selected), None, step,
                                  N.ptr(sel_idx), N.ptr(sel_gain),
                                  N.ptr(scratch), st)
                c = int(sel_idx[step].item())
                if c < 0:
                    from .optimize import checked_picks

                    checked_picks(sel_idx[: step + 1].cpu().numpy(), step + 1)
                row = padded_rows(ground.matrix[c:c + 1], d_pad, prec, dev)
                chosen[:, 0].copy_(row[0])
                lib.row_norms(prec.tag, N.ptr(row), 1, d, d_pad, N.ptr(cnorm),
                              st)
            # the last pick's m-update (msum[k-1])
            for slot, r0, r1 in gs.slices(pack_points=False):
                update_slice(slot, r0, r1, k - 1)
            finish_msum(k - 1)
            return sel_idx.cpu().numpy(), msum.cpu().numpy()
    finally:
        gs.close()


def _margin(n: int) -> int:
    """Device bytes a streamed pass needs besides the ring and the batch:
    the global block-partial array, e0 and small scalars."""
    return 65536 + 8 * (int(N.lib().pad_points(n)) // 256 + 8)


def fits_resident(n: int, d: int, precision, budget) -> bool:
    return budget is None or resident_bytes(n, d, precision) <= budget


__all__ = ["StreamPlan", "plan_slices", "resident_bytes", "layout_bytes",
           "GroundStream", "stream_build", "stream_set_min",
           "stream_packed_sums", "batch_device_bytes", "fits_resident",
           "stream_greedy"]
