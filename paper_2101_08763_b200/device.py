"""HBM-resident state of a ground set and upload helpers.

A ``DeviceGround`` owns (as torch tensors -- torch is only the allocator and
stream provider) the device layouts described in DESIGN.md:

* ``vt``     [d_pad][ld]   SIMT layout, column-major like the reference's
                           F-order V (core.py:286), compute type f32/f64.
* ``norms``  [ld]  f64     ||v_i||^2 of the stored values.
* ``aux``    [ld]  compute d(v_i, e0) rounded through the storage dtype.
* ``xc``     [rows][kp]    bf16/f16 tensor-core candidate operand (lazy).
* ``xp0``    [rows][kp]    bf16/f16 tensor-core point operand, m = 0 (lazy;
                           the point side of the K4-TC batch kernel).

Everything numeric is done by the kernels of ``libexem_b200.so``.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import ExemError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda(device=None) -> int:
    """Index of the sm_100 device to use; raise loudly if there is none."""
    t = torch()
    if not t.cuda.is_available():
        raise ExemError(
            "no CUDA device is visible: the B200 evaluator has no CPU path")
    if device is None:
        idx = t.cuda.current_device()
    elif isinstance(device, int):
        idx = device
    else:
        dv = t.device(device)
        idx = dv.index if dv.index is not None else t.cuda.current_device()
    major, minor = t.cuda.get_device_capability(idx)
    if major != 10:
        raise ExemError(
            f"device {idx} is sm_{major}{minor}; libexem_b200 is built for "
            "sm_100a (B200) only")
    N.lib()  # load the native library now so a missing build fails here
    return idx


def aux_dtype(precision) -> np.dtype:
    """Dtype of GroundSet.aux_distances: the storage dtype like the reference
    (core.py:303-305), except bfloat16 which keeps binary32."""
    if precision.tag == N.BF16:
        return np.dtype(np.float32)
    return precision.dtype


def compute_torch_dtype(precision):
    t = torch()
    return t.float64 if precision.compute_dtype == np.float64 else t.float32


def to_device_bytes(arr: np.ndarray, dev):
    """Upload a numpy array's raw bytes (any dtype, incl. bf16) to ``dev``:
    one DMA straight from the array (read-only / frozen arrays included, no
    staging copy), ordered on ``dev``'s current stream."""
    t = torch()
    raw = np.ascontiguousarray(arr)
    with t.cuda.device(dev):
        out = t.empty(max(raw.nbytes, 1), dtype=t.uint8, device=dev)
        N.lib().h2d_bytes(N.ptr(out), N.c_void_p(raw.ctypes.data),
                          raw.nbytes, N.stream_handle(dev))
    return out[: raw.nbytes]


def padded_rows(rows: np.ndarray, d_pad: int, precision, dev):
    """[k][d_pad] compute-type device matrix from (k, d) storage values."""
    t = torch()
    k, d = rows.shape
    host = np.zeros((k, d_pad), dtype=precision.compute_dtype)
    host[:, :d] = np.asarray(rows, dtype=precision.dtype).astype(
        precision.compute_dtype)
    return t.from_numpy(host).to(dev)


# binary16 tensor-core operands carry ||x||^2/2 folded into three f16 pieces
# p0*2^11 + p1 + p2 (fold_pieces, exem_common.cuh) with p0 <= 65504.
F16_FOLD_MAX_NORM = 2.0 * 65504.0 * 2048.0


def fold_ok(precision, max_norm) -> bool:
    """Whether norms up to ``max_norm`` fit the folded tensor-core operands
    of ``precision`` (only binary16 has a range limit).  Beyond it the
    binary16 paths run on the CUDA cores (K3-SIMT / K4), which use the
    reference's direct form and have no such limit."""
    return precision.tag != N.F16 or float(max_norm) < F16_FOLD_MAX_NORM


def ground_fold_ok(ground, device=None) -> bool:
    """``fold_ok`` for a ground set, resident or streamed (the streamed
    build records the largest ||v||^2 it saw)."""
    if ground.precision.tag != N.F16:
        return True
    if ground.streamed:
        return fold_ok(ground.precision, ground._ext()["max_norm"])
    return device_ground(ground, device).fold_ok()


class DeviceGround:
    """Device layouts of one ground set on one CUDA device."""

    def __init__(self, n, d, precision, device_index):
        t = torch()
        lib = N.lib()
        self.n, self.d, self.precision = int(n), int(d), precision
        self.device_index = device_index
        self.dev = t.device("cuda", device_index)
        self.ld = int(lib.pad_points(self.n))
        self.d_pad = int(lib.pad_dims(self.d))
        self.split_pts = int(lib.split_points(self.n))
        self.splits = int(lib.num_splits(self.n))
        cdt = compute_torch_dtype(precision)
        self.cdtype = cdt
        # bf16/f16 ground sets keep V at its 2-byte storage type
        # (EXEM_VT_STORAGE): K1 writes it, K2 / the m-update / the TC
        # operand packers read it; the binary32 widening is materialised
        # only for the CUDA-core consumers that need it (vt_c)
        self.vt_flag = N.VT_STORAGE if precision.is_half else 0
        if self.vt_flag:
            vdt = t.bfloat16 if precision.tag == N.BF16 else t.float16
        else:
            vdt = cdt
        self.vt = t.empty((self.d_pad, self.ld), dtype=vdt, device=self.dev)
        self._vt_c = None
        self.norms = t.empty(self.ld, dtype=t.float64, device=self.dev)
        self.aux = t.empty(self.ld, dtype=cdt, device=self.dev)
        self.scratch = t.empty(int(lib.reduce_scratch(self.ld)),
                               dtype=t.float64, device=self.dev)
        self.aux_sum = t.empty(1, dtype=t.float64, device=self.dev)
        self._xc = None
        self._xp0 = None
        self.kp = int(lib.tc_kp(self.d)) if precision.is_half else 0
        self._max_norm = None

    @property
    def vt_tag(self) -> int:
        """dtype tag of the entry points that read/write ``vt``."""
        return self.precision.tag | self.vt_flag

    def vt_c(self):
        """``vt`` at the compute type: ``vt`` itself for f32/f64; for half
        ground sets a binary32 widening built on first use (exem_widen_packed
        over the whole [d_pad][ld] buffer) for the CUDA-core kernels that
        read 4-byte V (K3-SIMT, K4, the sieve's distance rows, K2 shapes the
        TMA kernel does not cover)."""
        if not self.vt_flag:
            return self.vt
        if self._vt_c is None:
            t = torch()
            lib = N.lib()
            with t.cuda.device(self.device_index):
                out = t.empty((self.d_pad, self.ld), dtype=self.cdtype,
                              device=self.dev)
                lib.widen_packed(self.precision.tag, N.ptr(self.vt), self.ld,
                                 self.ld, 1, self.d_pad, N.ptr(out),
                                 self.stream)
            self._vt_c = out
        return self._vt_c

    def column_major_storage(self) -> np.ndarray:
        """(n, d) column-major host array of the STORED values (the
        reference's GroundSet.matrix layout), read back from ``vt``: exact,
        since vt holds the storage values (or, at f32/f64, the values)."""
        t = torch()
        tag = self.precision.tag
        with t.cuda.device(self.device_index):
            v = self.vt[: self.d, : self.n]
            if tag == N.BF16:
                host = v.contiguous().view(t.int16).cpu().numpy().view(
                    self.precision.dtype)
            elif tag == N.F16:
                host = v.contiguous().cpu().numpy()
            else:
                host = v.contiguous().cpu().numpy()
        return host.T  # (d, n) C-order == (n, d) F-order

    def fold_ok(self) -> bool:
        """Folded tensor-core operands are valid for this ground set."""
        if self.precision.tag != N.F16:
            return True
        if self._max_norm is None:
            self._max_norm = float(self.norms[: self.n].max().item())
        return fold_ok(self.precision, self._max_norm)

    @property
    def stream(self):
        return N.stream_handle(self.dev)

    def xp0(self):
        """Tensor-core point operand with h_i = ||v_i||^2/2 (m = 0): the
        point side of K4-TC (built once)."""
        if self._xp0 is None:
            t = torch()
            lib = N.lib()
            rows = int(lib.tc_rows(self.n))
            tdt = t.bfloat16 if self.precision.tag == N.BF16 else t.float16
            self._xp0 = t.empty((rows, self.kp), dtype=tdt, device=self.dev)
            lib.tc_pack_points(self.vt_tag, N.ptr(self.vt), self.ld,
                               self.n, self.d, N.ptr(self.norms), None,
                               N.ptr(self._xp0), self.stream)
        return self._xp0

    def xp_batch(self):
        """Point operand of K4-TC: the m = 0 folded rows, or plain rows when
        folding would add a K chunk (exem_tc_batch_plain)."""
        lib = N.lib()
        if not lib.tc_batch_plain(self.d):
            return self.xp0()
        if getattr(self, "_xpp", None) is None:
            t = torch()
            tdt = t.bfloat16 if self.precision.tag == N.BF16 else t.float16
            self._xpp = t.empty((int(lib.tc_rows(self.n)),
                                 int(lib.tc_batch_kp(self.d))), dtype=tdt,
                                device=self.dev)
            lib.tc_pack_points_plain(self.vt_tag, N.ptr(self.vt),
                                     self.ld, self.n, self.d,
                                     N.ptr(self._xpp), self.stream)
        return self._xpp

    def xc_split(self):
        """Split-bf16 binary32 candidate operand (exem_tc_pack_split)."""
        if getattr(self, "_xcs", None) is None:
            t = torch()
            lib = N.lib()
            rows = int(lib.tc_rows(self.n))
            kp = int(lib.tc_kp(int(lib.tc_split_dim(self.d))))
            self._xcs = t.empty((rows, kp), dtype=t.bfloat16, device=self.dev)
            lib.tc_pack_split(0, N.ptr(self.vt), self.ld, self.n, self.d,
                              N.ptr(self.norms), None, N.ptr(self._xcs),
                              self.stream)
        return self._xcs

    def xc(self):
        """Tensor-core candidate operand [tc_rows][kp] (built once)."""
        if self._xc is None:
            t = torch()
            lib = N.lib()
            rows = int(lib.tc_rows(self.n))
            tdt = t.bfloat16 if self.precision.tag == N.BF16 else t.float16
            self._xc = t.empty((rows, self.kp), dtype=tdt, device=self.dev)
            lib.tc_pack_candidates(self.vt_tag, N.ptr(self.vt), self.ld,
                                   self.n, self.d, N.ptr(self.norms),
                                   N.ptr(self._xc), self.stream)
        return self._xc


def row_major(matrix: np.ndarray) -> bool:
    """True when the host matrix is C-order (and not also F-order)."""
    return bool(matrix.flags.c_contiguous and not matrix.flags.f_contiguous)


def prepare_ground(matrix: np.ndarray, aux_vec: np.ndarray, precision,
                   device=None, check_finite: bool = False):
    """Upload V in its host layout and run K1 (column-major, the reference's
    layout, or row-major); return (state, aux_dist, sum)."""
    t = torch()
    idx = require_cuda(device)
    lib = N.lib()
    n, d = matrix.shape
    with t.cuda.device(idx):
        dg = DeviceGround(n, d, precision, idx)
        e0 = to_device_bytes(aux_vec, dg.dev)
        if not (matrix.flags.c_contiguous or matrix.flags.f_contiguous):
            matrix = np.asfortranarray(matrix)
        # one DMA straight from the (read-only, frozen) host matrix: no
        # host-side staging copy; row-major sources are transposed by K1
        src = t.empty(max(matrix.nbytes, 1), dtype=t.uint8, device=dg.dev)
        lib.h2d_bytes(N.ptr(src), N.c_void_p(matrix.ctypes.data),
                      matrix.nbytes, dg.stream)
        prepare = (lib.ground_prepare_rows if row_major(matrix)
                   else lib.ground_prepare)
        prepare(dg.vt_tag, N.ptr(src), n, d, N.ptr(e0), N.ptr(dg.vt),
                dg.ld, N.ptr(dg.norms), N.ptr(dg.aux), N.ptr(dg.aux_sum),
                N.ptr(dg.scratch), int(check_finite), dg.stream)
        aux_host = dg.aux[:n].cpu().numpy().astype(aux_dtype(precision))
        aux_sum = float(dg.aux_sum.item())
        del src, e0
    return dg, aux_host, aux_sum


def device_ground(ground, device=None) -> DeviceGround:
    """Cached ``DeviceGround`` of ``ground`` on ``device`` (built on demand)."""
    idx = require_cuda(device)
    dg = ground._device.get(idx)
    if dg is None:
        dg, _, _ = prepare_ground(ground.matrix, ground.aux, ground.precision,
                                  idx)
        ground._device[idx] = dg
    return dg
