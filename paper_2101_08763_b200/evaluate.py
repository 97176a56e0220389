"""Batch evaluation and memory-budget chunking (mirror of
``pkg/src/exembatch/evaluate.py``).

The reference dispatches on a backend string to three host implementations
(evaluate.py:42,282-293).  Here there is exactly one implementation per call:
the sm_100a kernels.  The reference's backend names are still accepted by
``Evaluator`` (so callers constructing ``Evaluator("parallel", ...)`` keep
working) and all of them select that single device path.

Per set j:  f(S_j) = acc(aux_loss) - acc(sum_i t_i(S_j)) / acc(n)
with t_i = min(aux_i, min_{e} d(v_i, S_j[e])) summed in fp64 in a fixed order
by kernel K4 (``exem_batch_eval``) + K6 (``exem_reduce_partials``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from .core import (
    DeviceLimits,
    EvaluationBatch,
    GroundSet,
    PackedBatch,
    Precision,
    compute_kernel_config,
)
from .errors import DimensionMismatchError, OutOfMemoryError
from .objective import (
    SQUARED_EUCLIDEAN,
    Dissimilarity,
    _as_elements,
    device_set_min,
    require_device_dissimilarity,
)

# Accepted backend names: the reference's (evaluate.py:42), in its order and
# with its default, plus "b200"; every name selects the same single device
# path, so existing ``Evaluator(backend=...)`` calls drop in unchanged.
BACKENDS = ("reference", "parallel", "tiled", "b200")


@dataclass(frozen=True)
class Evaluator:
    """Evaluation settings (evaluate.py:50-65) plus the CUDA device.

    ``limits``/``worker_count`` are kept for signature compatibility; the
    device path's tiling is fixed by the B200 kernels.
    """

    backend: str = "reference"
    limits: DeviceLimits = field(default_factory=DeviceLimits)
    worker_count: int = 1
    precision: Optional[Precision] = None
    device: Optional[int] = None
    # binary32 Greedy gains on the tensor cores via split-bf16 operands
    # (opt-in; the default binary32 path is the CUDA-core K3-SIMT)
    tensor_fp32: bool = False
    # Greedy: run the k-step loop as one CUDA graph (optimize.capture_steps)
    cuda_graph: bool = False

    def __post_init__(self):
        if self.backend not in BACKENDS:
            raise ValueError(
                f"unknown backend {self.backend!r}; expected one of {BACKENDS}")
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")


@dataclass(frozen=True)
class ChunkPlan:
    """Sets-per-chunk under a memory budget (evaluate.py:68-75)."""

    chunk_size: int
    chunk_count: int
    per_set_bytes: int
    free_bytes: int


def estimate_set_memory(n: int, k_max: int, d: int, precision: Precision) -> int:
    """mu_s = (k_max*d + n) * bytes_per_value + 16 (evaluate.py:78-83;
    PAPER.md:406-409): the packed slice, one work-matrix row and metadata."""
    if min(n, k_max, d) < 1:
        raise ValueError("n, k_max and d must all be >= 1")
    return (k_max * d + n) * precision.bytes_per_value + 16


def plan_chunks(free_bytes: int, per_set_bytes: int, l: int) -> ChunkPlan:
    """chunk_size = min(floor(phi/mu_s), l); OOM when 0 (evaluate.py:86-102)."""
    if per_set_bytes < 1 or l < 1:
        raise ValueError("per_set_bytes and l must be >= 1")
    fit = free_bytes // per_set_bytes
    if fit == 0:
        raise OutOfMemoryError(
            f"a single evaluation set needs {per_set_bytes} bytes but only "
            f"{free_bytes} are free; use a lower precision or a larger budget")
    size = min(fit, l)
    return ChunkPlan(chunk_size=size, chunk_count=math.ceil(l / size),
                     per_set_bytes=per_set_bytes, free_bytes=free_bytes)


def _check_batch(ground: GroundSet, batch: EvaluationBatch) -> None:
    if batch.d != ground.d:
        raise DimensionMismatchError(
            f"batch is {batch.d}-dim but the ground set is {ground.d}-dim")


def _effective_precision(evaluator: Evaluator, ground: GroundSet) -> Precision:
    if evaluator.precision is not None and evaluator.precision is not ground.precision:
        raise ValueError(
            "evaluator precision differs from the ground set precision; "
            "build the ground set at the desired precision")
    return ground.precision


def _finish(ground: GroundSet, sums: np.ndarray) -> np.ndarray:
    """acc(aux_loss) - acc(sum)/acc(n) per set (evaluate.py:111-112)."""
    acc = ground.precision.accumulate_dtype
    return acc.type(ground.aux_loss) - sums.astype(acc) / acc.type(ground.n)


def evaluate_single(ground: GroundSet, set_vectors,
                    dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN) -> float:
    """f of one set (evaluate.py:115-123) -- kernel K2 + fixed-order sum."""
    require_device_dissimilarity(dissimilarity)
    elems = _as_elements(ground, set_vectors)
    if elems.shape[0] == 0:
        return 0.0
    total, _, _ = device_set_min(ground, elems, include_aux=True)
    return float(_finish(ground, np.array([total]))[0])


TC_MAX_SET = 256  # K4-TC holds one set in <= 256 TMEM columns


def tc_batch_supported(precision: Precision, k_max: int) -> bool:
    """Explicit batches of half-precision ground sets run on tensor cores
    (K4-TC) when a set fits one TMEM tile; otherwise on the SIMT K4."""
    return precision.is_half and 1 <= k_max <= TC_MAX_SET


class DeviceBatch:
    """A packed batch uploaded once (packed_address order, core.py:320-328)
    plus what the batch kernels need: element norms, cardinalities and, for
    half precision, the K4-TC set-tile operand."""

    def __init__(self, values: Optional[np.ndarray], d: int, k_max: int,
                 l: int, cardinalities, precision: Precision, d_pad: int, dev,
                 stream, sets=None, ground_fold_ok: bool = True):
        """``values``: a packed (d, k_max, l) host buffer (PackedBatch), or
        None with ``sets`` = the l element arrays, which are concatenated on
        the host and interleaved on the device (exem_pack_elements)."""
        from .device import to_device_bytes, torch

        t = torch()
        lib = N.lib()
        self.d, self.k_max, self.l = d, k_max, l
        self.l_pad = int(-(-l // 128) * 128)
        self.precision = precision
        cdt = t.float64 if precision.compute_dtype == np.float64 else t.float32
        if sets is not None:
            rows = np.concatenate([np.asarray(x, dtype=precision.dtype)
                                   .reshape(-1, d) for x in sets])
            cards = np.asarray(cardinalities, dtype=np.int64)
            offsets = np.zeros(l, dtype=np.int64)
            np.cumsum(cards[:-1], out=offsets[1:])
            rows_d = to_device_bytes(rows, dev)
            offs_d = t.from_numpy(offsets).to(dev)
            card_d = t.from_numpy(cards.astype(np.int32)).to(dev)
            self.packed = t.empty((d_pad, k_max, self.l_pad), dtype=cdt,
                                  device=dev)
            lib.pack_elements(precision.tag, N.ptr(rows_d), N.ptr(offs_d),
                              N.ptr(card_d), l, self.l_pad, k_max, d,
                              N.ptr(self.packed), stream)
        else:  # raw packed bytes up, widened + padded on the device
            raw = np.ascontiguousarray(
                np.asarray(values, dtype=precision.dtype).reshape(d, k_max, l))
            raw_d = to_device_bytes(raw, dev)
            self.packed = t.empty((d_pad, k_max, self.l_pad), dtype=cdt,
                                  device=dev)
            lib.widen_packed(precision.tag, N.ptr(raw_d), l, self.l_pad, k_max,
                             d, N.ptr(self.packed), stream)
        self.pnorms = t.empty((k_max, self.l_pad), dtype=t.float64, device=dev)
        lib.packed_norms(precision.tag, N.ptr(self.packed), d, k_max,
                         self.l_pad, N.ptr(self.pnorms), stream)
        self.card = t.tensor(np.asarray(cardinalities, dtype=np.int32),
                             device=dev)
        self.xs = None
        self.bs = None
        use_tc = tc_batch_supported(precision, k_max)
        if use_tc and precision.tag == N.F16:
            # binary16 operands: every norm must be in the folded range (the
            # same rule for the plain layout, whose fp32 GEMM form cancels
            # catastrophically at such norms; the CUDA-core K4 uses the
            # reference's direct form)
            from .device import fold_ok

            use_tc = ground_fold_ok and (l == 0 or fold_ok(
                precision, self.pnorms.max().item()))
        if use_tc:
            rows = int(lib.tc_set_rows(l, k_max))
            tdt = t.bfloat16 if precision.tag == N.BF16 else t.float16
            self.xs = t.empty((rows, int(lib.tc_batch_kp(d))), dtype=tdt,
                              device=dev)
            if lib.tc_batch_plain(d):  # unfolded operands (K4-TC)
                self.bs = t.empty(rows, dtype=t.float32, device=dev)
            lib.tc_pack_sets(precision.tag, N.ptr(self.packed),
                             N.ptr(self.pnorms), N.ptr(self.card), l,
                             self.l_pad, k_max, d, N.ptr(self.xs),
                             N.ptr(self.bs), stream)


def batch_partials(dg, batch: DeviceBatch, partial, split_pts: int,
                   splits: int) -> None:
    """K4 (SIMT) or K4-TC over the ground rows held by ``dg``:
    partial[s][j] = sum over split s of t_i(S_j)."""
    lib = N.lib()
    prec = dg.precision
    pp = partial if isinstance(partial, N.c_void_p) else N.ptr(partial)
    if batch.xs is not None:
        lib.batch_eval_tc(prec.tag, N.ptr(dg.xp_batch()), dg.n, N.ptr(dg.aux),
                          N.ptr(dg.norms), N.ptr(batch.xs), N.ptr(batch.bs),
                          batch.l, batch.k_max, dg.d, split_pts, pp, splits,
                          dg.stream)
    else:
        lib.batch_eval(prec.tag, N.ptr(dg.vt_c()), dg.ld, dg.n, dg.d,
                       N.ptr(dg.norms), N.ptr(dg.aux), N.ptr(batch.packed),
                       N.ptr(batch.pnorms), N.ptr(batch.card), batch.l,
                       batch.l_pad, batch.k_max, split_pts, pp, splits,
                       dg.stream)


def device_packed_sums(ground: GroundSet, values: Optional[np.ndarray],
                       d: int, k_max: int, l: int, cardinalities, device=None,
                       sets=None):
    """Upload a batch -- a packed (d, k_max, l) buffer, or the sets' element
    arrays -- and run K4 (or K4-TC) + K6.

    Returns the device tensor of per-set fp64 sums sum_i t_i(S_j).
    """
    from .device import torch

    if ground.streamed:
        from .streaming import stream_packed_sums

        return stream_packed_sums(ground, values, d, k_max, l, cardinalities,
                                  device, sets=sets)
    t = torch()
    lib = N.lib()
    dg = ground.on_device(device)
    with t.cuda.device(dg.device_index):
        st = dg.stream
        batch = DeviceBatch(values, d, k_max, l, cardinalities,
                            ground.precision, dg.d_pad, dg.dev, st, sets=sets,
                            ground_fold_ok=dg.fold_ok())
        partial = t.empty((dg.splits, l), dtype=t.float64, device=dg.dev)
        batch_partials(dg, batch, partial, dg.split_pts, dg.splits)
        sums = t.empty(l, dtype=t.float64, device=dg.dev)
        lib.reduce_partials(N.ptr(partial), dg.splits, l, 1.0, N.ptr(sums), st)
    return sums


def tiled_evaluate(ground: GroundSet, packed: PackedBatch,
                   dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN,
                   limits: Optional[DeviceLimits] = None,
                   worker_count: int = 1, instrument: bool = False):
    """Evaluate a packed batch (evaluate.py:197-270) with kernel K4.

    The packed round-robin buffer is consumed in its own layout; blank slots
    (e >= card_j) never contribute.  With ``instrument=True`` the reference's
    staging model is reported alongside: under the paper's kernel
    configuration every ground vector is staged once per block row covering
    its column, i.e. ``grid_y`` times (core.py:349-377).
    """
    require_device_dissimilarity(dissimilarity)
    limits = limits or DeviceLimits()
    config = compute_kernel_config(ground.n, packed.l, ground.bytes_per_vector,
                                   limits)
    sums = device_packed_sums(ground, packed.values, packed.d, packed.k_max,
                              packed.l, packed.cardinalities)
    out = _finish(ground, sums.cpu().numpy())
    if instrument:
        loads = np.full(ground.n, config.grid[1], dtype=np.int64)
        return out, loads
    return out


def evaluate_batch(evaluator: Evaluator, ground: GroundSet,
                   batch: EvaluationBatch,
                   dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN) -> np.ndarray:
    """One value per set (evaluate.py:273-293) -- kernels K4 + K6."""
    require_device_dissimilarity(dissimilarity)
    _check_batch(ground, batch)
    _effective_precision(evaluator, ground)
    sums = device_packed_sums(ground, None, batch.d, batch.k_max, batch.l,
                              batch.cardinalities, evaluator.device,
                              sets=batch.sets)
    return _finish(ground, sums.cpu().numpy())


def evaluate_chunked(evaluator: Evaluator, ground: GroundSet,
                     batch: EvaluationBatch,
                     dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN,
                     budget: int = 0) -> np.ndarray:
    """Budget-sized chunks of sets, merged in order (evaluate.py:296-319).

    Per-set sums never depend on which other sets share a launch, so the
    result is bit-identical to ``evaluate_batch``.
    """
    _check_batch(ground, batch)
    precision = _effective_precision(evaluator, ground)
    mu = estimate_set_memory(ground.n, batch.k_max, batch.d, precision)
    plan = plan_chunks(budget, mu, batch.l)
    pieces = []
    for c in range(plan.chunk_count):
        lo = c * plan.chunk_size
        hi = min(lo + plan.chunk_size, batch.l)
        sub = EvaluationBatch.from_sets(batch.sets[lo:hi])
        pieces.append(evaluate_batch(evaluator, ground, sub, dissimilarity))
    return np.concatenate(pieces)
