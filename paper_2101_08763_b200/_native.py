"""ctypes binding of the C-ABI in ``include/exem_b200.h``.

This is the one place the Python host touches native code.  Every entry
point takes plain device pointers (``tensor.data_ptr()``), sizes and the
``cudaStream_t`` of torch's current stream; nothing here computes on the CPU.
A missing or unloadable library raises immediately -- there is no fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import c_double, c_int, c_int64, c_void_p
from pathlib import Path

from .errors import (
    DimensionMismatchError,
    ExemError,
    InvalidDataError,
    OutOfMemoryError,
)

LIB_PATH = Path(__file__).resolve().parent / "libexem_b200.so"

# dtype tags (include/exem_b200.h)
F16, BF16, F32, F64 = 0, 1, 2, 3
# OR'd into a half tag: the vt buffer holds 2-byte storage values
VT_STORAGE = 0x100

# status codes -> reference exception classes (pkg/src/exembatch/errors.py)
OK, ERR_ARG, ERR_OOM, ERR_CUDA, ERR_DATA, ERR_UNSUPPORTED = range(6)

_P = c_void_p
_SIGNATURES = {
    "exem_last_error": (ctypes.c_char_p, []),
    "exem_abi_version": (c_int, []),
    "exem_device_info": (c_int, [c_int, _P, _P, _P, _P]),
    "exem_pad_points": (c_int64, [c_int64]),
    "exem_pad_dims": (c_int64, [c_int64]),
    "exem_split_points": (c_int64, [c_int64]),
    "exem_num_splits": (c_int64, [c_int64]),
    "exem_tc_kp": (c_int64, [c_int64]),
    "exem_tc_rows": (c_int64, [c_int64]),
    "exem_reduce_scratch": (c_int64, [c_int64]),
    "exem_ground_prepare": (c_int, [c_int, _P, c_int64, c_int64, _P, _P,
                                    c_int64, _P, _P, _P, _P, c_int, _P]),
    "exem_set_min_storage_ok": (c_int, [c_int, c_int64, c_int64, c_int]),
    "exem_set_min": (c_int, [c_int, _P, c_int64, c_int64, c_int64, _P, _P, _P,
                             _P, c_int64, c_int, _P, _P, _P, _P, _P]),
    "exem_batch_eval": (c_int, [c_int, _P, c_int64, c_int64, c_int64, _P, _P,
                                _P, _P, _P, c_int64, c_int64, c_int64, c_int64,
                                _P, c_int64, _P]),
    "exem_greedy_gains_simt": (c_int, [c_int, _P, c_int64, _P, c_int64, _P,
                                       c_int64, _P, _P, c_int64, c_int64,
                                       c_int64, _P, c_int64, _P]),
    "exem_greedy_gains_tc": (c_int, [c_int, _P, c_int64, _P, c_int64, c_int64,
                                     c_int64, _P, c_int64, _P]),
    "exem_greedy_gains_tc_ex": (c_int, [c_int, _P, c_int64, _P, c_int64,
                                        c_int64, c_int64, _P, c_int64, c_int,
                                        _P, _P]),
    "exem_tc_pack_candidates": (c_int, [c_int, _P, c_int64, c_int64, c_int64,
                                        _P, _P, _P]),
    "exem_tc_pack_points": (c_int, [c_int, _P, c_int64, c_int64, c_int64, _P,
                                    _P, _P, _P]),
    "exem_reduce_partials": (c_int, [_P, c_int64, c_int64, c_double, _P, _P]),
    "exem_argmax_select": (c_int, [_P, c_int64, _P, _P, c_int64, _P, _P, _P,
                                   _P]),
    "exem_greedy_update": (c_int, [c_int, _P, c_int64, c_int64, c_int64, _P,
                                   _P, c_int64, _P, _P, c_int64, _P, _P,
                                   c_int64, _P, _P, _P]),
    "exem_greedy_init": (c_int, [c_int, _P, c_int64, _P, _P, _P, _P]),
    "exem_distance_matrix": (c_int, [c_int, _P, _P, c_int64, _P, _P, c_int64,
                                     c_int64, c_int64, _P, _P]),
    "exem_row_norms": (c_int, [c_int, _P, c_int64, c_int64, c_int64, _P, _P]),
    "exem_packed_norms": (c_int, [c_int, _P, c_int64, c_int64, c_int64, _P,
                                  _P]),
    "exem_tc_set_geometry": (c_int, [c_int64, _P, _P, _P]),
    "exem_tc_set_rows": (c_int64, [c_int64, c_int64]),
    "exem_tc_pack_sets": (c_int, [c_int, _P, _P, _P, c_int64, c_int64,
                                  c_int64, c_int64, _P, _P, _P]),
    "exem_batch_eval_tc": (c_int, [c_int, _P, c_int64, _P, _P, _P, _P,
                                   c_int64, c_int64, c_int64, c_int64, _P,
                                   c_int64, _P]),
    "exem_tc_batch_plain": (c_int64, [c_int64]),
    "exem_tc_batch_kp": (c_int64, [c_int64]),
    "exem_tc_pack_points_plain": (c_int, [c_int, _P, c_int64, c_int64,
                                          c_int64, _P, _P]),
    "exem_host_register": (c_int, [_P, c_int64]),
    "exem_host_unregister": (c_int, [_P]),
    "exem_h2d_rows": (c_int, [_P, _P, c_int64, c_int64, c_int64, c_int64,
                              c_int64, _P]),
    "exem_sum_fixed": (c_int, [_P, c_int64, _P, c_int64, _P]),
    "exem_pack_elements": (c_int, [c_int, _P, _P, _P, c_int64, c_int64,
                                   c_int64, c_int64, _P, _P]),
    "exem_tc_split_dim": (c_int64, [c_int64]),
    "exem_tc_pack_split": (c_int, [c_int, _P, c_int64, c_int64, c_int64, _P,
                                   _P, _P, _P]),
    "exem_tc_refresh_h": (c_int, [_P, _P, c_int64, _P, c_int64, c_int64, _P]),
    "exem_sieve_gains": (c_int, [c_int, _P, c_int64, c_int64, _P, c_int64,
                                 _P, _P, _P]),
    "exem_sieve_update": (c_int, [c_int, _P, _P, c_int64, _P, _P, _P]),
    "exem_ipc_alloc": (c_int, [c_int64, _P]),
    "exem_ipc_free": (c_int, [_P]),
    "exem_ipc_handle": (c_int, [_P, _P]),
    "exem_ipc_open": (c_int, [_P, _P]),
    "exem_ipc_close": (c_int, [_P]),
    "exem_peer_publish": (c_int, [_P, ctypes.c_uint64, _P]),
    "exem_peer_argmax_select": (c_int, [_P, _P, c_int, ctypes.c_uint64,
                                        c_int64, c_double, _P, _P, c_int64,
                                        _P, _P, _P, _P]),
    "exem_ground_prepare_rows": (c_int, [c_int, _P, c_int64, c_int64, _P, _P,
                                         c_int64, _P, _P, _P, _P, c_int, _P]),
    "exem_h2d_bytes": (c_int, [_P, _P, c_int64, _P]),
    "exem_widen_packed": (c_int, [c_int, _P, c_int64, c_int64, c_int64,
                                  c_int64, _P, _P]),
    "exem_sieve_block_dist": (c_int, [c_int, _P, c_int64, c_int64, c_int64,
                                      _P, _P, _P, c_int64, _P, c_int64, _P,
                                      _P]),
    "exem_sieve_block_scratch": (c_int64, [c_int64, c_int64, c_int64]),
    "exem_sieve_block_gains": (c_int, [c_int, _P, c_int64, c_int64, _P,
                                       c_int64, c_int64, c_int64, _P, _P, _P]),
    "exem_launch_count": (c_int64, []),
}

EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


class _Lib:
    """Bound library whose calls raise the mapped reference exception."""

    def __init__(self, handle: ctypes.CDLL):
        self._h = handle
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args

    def raw(self, name):
        return getattr(self._h, name)

    def __getattr__(self, name):
        fn = getattr(self._h, "exem_" + name)
        if fn.restype is not c_int or name in ("abi_version",
                                               "set_min_storage_ok"):
            return fn

        def call(*args):
            rc = fn(*args)
            if rc != OK:
                raise_status(rc, self._h.exem_last_error().decode())
            return rc

        return call


def raise_status(rc: int, msg: str):
    if rc == ERR_OOM:
        raise OutOfMemoryError(msg)
    if rc == ERR_DATA:
        raise InvalidDataError(msg)
    if rc == ERR_ARG:
        raise DimensionMismatchError(msg)
    raise ExemError(f"native error {rc}: {msg}")


# Bumped whenever an entry point's signature or contract changes
# (2: exem_ground_prepare[_rows] gained check_finite; K4-TC set tiles are
# column-interleaved; 3: exem_greedy_gains_tc_ex; 4: EXEM_VT_STORAGE,
# exem_set_min_storage_ok).
ABI_VERSION = 4


def load_library(path: Path | str | None = None) -> _Lib:
    """Load (once) and bind ``libexem_b200.so``; raise if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # EXEM_LIB_PATH: an alternative build of the same library for A/B
        # timing experiments (tools/); it is still the native library
        p = Path(path) if path else Path(os.environ.get("EXEM_LIB_PATH",
                                                        LIB_PATH))
        if not p.exists():
            raise ExemError(
                f"native library {p} is missing; run "
                "`python -m paper_2101_08763_b200.build` (there is no CPU "
                "fallback)"
            )
        lib = _Lib(ctypes.CDLL(str(p)))
        got = int(lib.abi_version())
        if got != ABI_VERSION:
            raise ExemError(
                f"native library {p} has ABI {got}, this package needs "
                f"{ABI_VERSION}: rebuild it (python -m paper_2101_08763_b200.build)")
        if path is None:
            _lib = lib
        return lib


def lib() -> _Lib:
    return load_library()


def ptr(t) -> c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    return c_void_p(0 if t is None else t.data_ptr())


def stream_handle(device=None) -> c_void_p:
    import torch

    return c_void_p(torch.cuda.current_stream(device).cuda_stream)
