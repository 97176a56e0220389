"""Dissimilarity and the exemplar-clustering objective (mirror of
``pkg/src/exembatch/objective.py``).

f(S) = L({e0}) - L(S u {e0}),  L(S) = |V|^-1 sum_v min_{s in S} d(v, s)
(PAPER.md:98-113).  Every per-point minimum and sum runs on the device
(kernel K2, ``exem_set_min``); the host only coerces arguments and forms the
final ``acc(aux_loss) - sum/acc(n)`` scalar exactly like the reference.

Only squared Euclidean distance has a device kernel.  A custom
``Dissimilarity`` keeps working for ``Dissimilarity.distances`` (it is the
caller's own host function), but passing one to an evaluation entry point
raises: there is no CPU fallback for the evaluation path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native as N
from .core import GroundSet
from .errors import (
    DimensionMismatchError,
    EmptyEvaluationSetError,
    ExemError,
    InvalidDataError,
)


@dataclass(frozen=True)
class Dissimilarity:
    """Non-negative dissimilarity (objective.py:24-61).

    ``batch`` maps an (m, d) block and (q, d) elements to an (m, q) matrix;
    for ``SQUARED_EUCLIDEAN`` it is the device kernel ``exem_distance_matrix``.
    """

    name: str
    pairwise: Callable
    batch: Optional[Callable] = None
    requires_equal_dims: bool = True

    def __call__(self, x, y) -> float:
        return self.pairwise(x, y)

    def distances(self, block: np.ndarray, elems: np.ndarray) -> np.ndarray:
        block = np.asarray(block)
        elems = np.asarray(elems)
        if self.requires_equal_dims and block.shape[1] != elems.shape[1]:
            raise DimensionMismatchError(
                f"cannot compare {block.shape[1]}-dim and {elems.shape[1]}-dim vectors")
        if self.batch is not None:
            out = self.batch(block, elems)
        else:
            out = np.empty((block.shape[0], elems.shape[0]), dtype=block.dtype)
            for a in range(block.shape[0]):
                for b in range(elems.shape[0]):
                    out[a, b] = self.pairwise(block[a], elems[b])
        if np.isnan(out).any():
            raise InvalidDataError(f"dissimilarity {self.name!r} produced NaN")
        if __debug__ and out.size and float(np.min(out)) < 0:
            raise InvalidDataError(
                f"dissimilarity {self.name!r} produced a negative value")
        return out


def squared_euclidean(x, y) -> float:
    """||x - y||^2 of two vectors (objective.py:64-72)."""
    xa, ya = np.asarray(x), np.asarray(y)
    if xa.shape != ya.shape:
        raise DimensionMismatchError(
            f"cannot compare vectors of shapes {xa.shape} and {ya.shape}")
    diff = xa - ya
    return float(np.sum(diff * diff))


def _precision_of(dtype):
    from .core import Precision

    dt = np.dtype(dtype)
    for p in Precision:
        try:
            if p.dtype == dt:
                return p
        except ValueError:
            continue
    if dt.kind in "iub":
        return Precision.binary64
    raise InvalidDataError(f"unsupported dtype {dt}")


def _device_distances(block: np.ndarray, elems: np.ndarray) -> np.ndarray:
    """Device distance matrix in the reference's per-precision form
    (objective.py:75-90): GEMM form for f32/f64, direct form for halves."""
    from .device import padded_rows, require_cuda, torch

    t = torch()
    prec = _precision_of(block.dtype)
    idx = require_cuda()
    lib = N.lib()
    m, d = block.shape
    q = elems.shape[0]
    if m == 0 or q == 0:
        return np.zeros((m, q), dtype=prec.dtype)
    if not (np.isfinite(np.asarray(block, np.float64)).all()
            and np.isfinite(np.asarray(elems, np.float64)).all()):
        raise InvalidDataError(
            "dissimilarity 'squared_euclidean' produced NaN")
    with t.cuda.device(idx):
        dev = t.device("cuda", idx)
        d_pad = int(lib.pad_dims(d))
        a = padded_rows(np.asarray(block, prec.dtype), d_pad, prec, dev)
        b = padded_rows(np.asarray(elems, prec.dtype), d_pad, prec, dev)
        an = t.empty(m, dtype=t.float64, device=dev)
        bn = t.empty(q, dtype=t.float64, device=dev)
        st = N.stream_handle(dev)
        lib.row_norms(prec.tag, N.ptr(a), m, d, d_pad, N.ptr(an), st)
        lib.row_norms(prec.tag, N.ptr(b), q, d, d_pad, N.ptr(bn), st)
        out = t.empty((m, q), dtype=a.dtype, device=dev)
        lib.distance_matrix(prec.tag, N.ptr(a), N.ptr(an), m, N.ptr(b),
                            N.ptr(bn), q, d, d_pad, N.ptr(out), st)
        res = out.cpu().numpy()
    return res.astype(prec.dtype)


SQUARED_EUCLIDEAN = Dissimilarity(
    name="squared_euclidean",
    pairwise=squared_euclidean,
    batch=_device_distances,
)


def require_device_dissimilarity(dissimilarity) -> None:
    """Only squared Euclidean distance has a device kernel; refuse others."""
    if dissimilarity is None or dissimilarity is SQUARED_EUCLIDEAN:
        return
    if (isinstance(dissimilarity, Dissimilarity)
            and dissimilarity.name == SQUARED_EUCLIDEAN.name
            and dissimilarity.batch is SQUARED_EUCLIDEAN.batch):
        return
    raise ExemError(
        f"dissimilarity {getattr(dissimilarity, 'name', dissimilarity)!r} has "
        "no device kernel; only SQUARED_EUCLIDEAN is evaluated on the B200 "
        "(there is no CPU fallback)")


def _as_elements(ground: GroundSet, elements) -> np.ndarray:
    """(m, d) array at the ground precision (objective.py:100-110)."""
    arr = np.asarray(elements, dtype=ground.precision.dtype)
    if arr.size == 0:
        return np.empty((0, ground.d), dtype=ground.precision.dtype)
    arr = np.atleast_2d(arr)
    if arr.shape[1] != ground.d:
        raise DimensionMismatchError(
            f"set elements are {arr.shape[1]}-dim but the ground set is {ground.d}-dim")
    return arr


def device_set_min(ground: GroundSet, elems: np.ndarray, include_aux: bool,
                   want_t: bool = False, want_labels: bool = False,
                   device=None):
    """Run K2 over one explicit set; return (sum_t, t or None, labels or None).

    sum_t is the fixed-order fp64 sum of t_i = min([aux_i,] min_e d(v_i, e)).
    """
    from .device import padded_rows, torch

    if ground.streamed:
        from .streaming import stream_set_min

        return stream_set_min(ground, elems, include_aux, want_t, want_labels,
                              device)
    t = torch()
    lib = N.lib()
    dg = ground.on_device(device)
    prec = ground.precision
    k = int(elems.shape[0])
    with t.cuda.device(dg.device_index):
        st = dg.stream
        e = padded_rows(elems, dg.d_pad, prec, dg.dev)
        en = t.empty(max(k, 1), dtype=t.float64, device=dg.dev)
        if k:
            lib.row_norms(prec.tag, N.ptr(e), k, dg.d, dg.d_pad, N.ptr(en), st)
        # sets larger than one element group of the TMA K2 (64 at 4-byte,
        # 32 at 8-byte compute types) carry the running minimum through
        # t_out: give it one even when only the sum is wanted
        groups = k > (32 if dg.cdtype == t.float64 else 64)
        t_out = (t.empty(dg.n, dtype=dg.cdtype, device=dg.dev)
                 if want_t or groups else None)
        lab = t.empty(dg.n, dtype=t.int64, device=dg.dev) if want_labels else None
        s = t.empty(1, dtype=t.float64, device=dg.dev)
        # 2-byte half storage goes straight to the TMA-fed K2; shapes it
        # does not cover read the binary32 widening
        if dg.vt_flag and lib.set_min_storage_ok(dg.vt_tag, dg.d, k,
                                                 int(t_out is not None)):
            tag, vt = dg.vt_tag, dg.vt
        else:
            tag, vt = prec.tag, dg.vt_c()
        lib.set_min(tag, N.ptr(vt), dg.ld, dg.n, dg.d, N.ptr(dg.norms),
                    N.ptr(dg.aux), N.ptr(e), N.ptr(en), k, int(include_aux),
                    N.ptr(t_out), N.ptr(lab), N.ptr(s), N.ptr(dg.scratch), st)
        total = float(s.item())
        t_host = t_out.cpu().numpy() if want_t else None
        lab_host = lab.cpu().numpy() if want_labels else None
    return total, t_host, lab_host


def min_distances(ground: GroundSet, elems: np.ndarray,
                  dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN,
                  include_aux: bool = True) -> np.ndarray:
    """Per-observation minimum distance to ``elems`` (objective.py:113-141)."""
    require_device_dissimilarity(dissimilarity)
    dtype = ground.precision.dtype
    elems = np.asarray(elems, dtype=dtype)
    if elems.ndim == 1:
        elems = elems.reshape(1, -1) if elems.size else elems.reshape(0, ground.d)
    if elems.shape[0] and elems.shape[1] != ground.d:
        raise DimensionMismatchError(
            f"cannot compare {ground.d}-dim and {elems.shape[1]}-dim vectors")
    if elems.shape[0] == 0:
        t = np.full(ground.n, ground.precision.max_finite, dtype=dtype)
        if include_aux:
            t = np.minimum(t, ground.aux_distances).astype(dtype)
        return t
    _, t, _ = device_set_min(ground, elems, include_aux, want_t=True)
    return t.astype(dtype)


def kmedoids_loss(ground: GroundSet, set_vectors,
                  dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN) -> float:
    """Mean nearest-element distance (objective.py:144-153)."""
    require_device_dissimilarity(dissimilarity)
    elems = _as_elements(ground, set_vectors)
    if elems.shape[0] == 0:
        raise EmptyEvaluationSetError("the loss minimizes over a non-empty set")
    total, _, _ = device_set_min(ground, elems, include_aux=False)
    acc = ground.precision.accumulate_dtype
    return float(acc.type(total / ground.n))


def exemplar_value(ground: GroundSet, set_vectors,
                   dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN) -> float:
    """f(S) = L({e0}) - L(S u {e0}) (objective.py:156-167)."""
    require_device_dissimilarity(dissimilarity)
    elems = _as_elements(ground, set_vectors)
    if elems.shape[0] == 0:
        return 0.0
    total, _, _ = device_set_min(ground, elems, include_aux=True)
    acc = ground.precision.accumulate_dtype
    return float(acc.type(ground.aux_loss) - acc.type(total / ground.n))


def point_loss(ground: GroundSet, i: int, set_vectors,
               dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN) -> float:
    """Per-observation partial loss of S u {e0} (objective.py:170-195)."""
    require_device_dissimilarity(dissimilarity)
    if not 0 <= i < ground.n:
        raise IndexError(f"point index {i} out of range [0, {ground.n})")
    elems = _as_elements(ground, set_vectors)
    dtype = ground.precision.dtype
    if elems.shape[0]:
        _, t, _ = device_set_min(ground, elems, include_aux=True, want_t=True)
        ti = dtype.type(t[i])
    else:
        ti = ground.aux_distances[i]
    return float(dtype.type(ti) / dtype.type(ground.n))


def marginal_gain(ground: GroundSet, set_vectors, element,
                  dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN) -> float:
    """f(S u {e}) - f(S) (objective.py:198-210)."""
    base = _as_elements(ground, set_vectors)
    extra = _as_elements(ground, element)
    extended = np.vstack([base, extra]) if base.shape[0] else extra
    return exemplar_value(ground, extended, dissimilarity) - exemplar_value(
        ground, base, dissimilarity)
