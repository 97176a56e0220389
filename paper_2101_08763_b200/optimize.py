"""Greedy selection, the exhaustive oracle and cluster assignment (mirror of
``pkg/src/exembatch/optimize.py``).

``greedy_maximize`` keeps the reference's contract (optimize.py:33-82): k
steps, the candidates of a step are V minus the selection, ties go to the
lowest ground index, ``values[t]`` is f(S_t) and ``evaluations`` counts the
l = n - t candidate sets scored per step.  It is *optimizer-aware*: instead
of materialising the l explicit sets S u {c} (optimize.py:64, ~20 GB per step
at n=1M, k=50) it keeps m_i = min(aux_i, min_{s in S} d(v_i, s)) on device and
scores every candidate in one launch of K3,

    f(S u {c}) = f(S) + n^-1 sum_i max(0, m_i - d(v_i, c)),

which is algebraically identical (min is exact) -- see DESIGN.md.  The whole
step (K3 gains -> K6 reduce -> K5 argmax -> K2 m-update) stays on device; the
host reads the trajectory once at the end.
"""

from __future__ import annotations

import itertools
import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .core import EvaluationBatch, GroundSet
from .errors import (
    BudgetExceedsGroundSetError,
    EmptyEvaluationSetError,
    InstanceTooLargeError,
    InvalidDataError,
)
from .evaluate import (
    Evaluator,
    _effective_precision,
    evaluate_batch,
    estimate_set_memory,
    plan_chunks,
)
from .objective import (
    SQUARED_EUCLIDEAN,
    Dissimilarity,
    _as_elements,
    device_set_min,
    require_device_dissimilarity,
)

BRUTE_FORCE_LIMIT = 10**6
SPLIT32_MAX_D = 128
# K3-TC epilogue width: after the first tensor-core gains launch of a run,
# the fraction of (candidate row, 32-point chunk) sign screens that found a
# positive gain decides between 2 and 4 epilogue warps per TMEM lane quarter
# for the remaining steps (exem_greedy_gains_tc_ex).
EPI_WIDE_THRESHOLD = 0.02


@dataclass(frozen=True)
class OptimizationResult:
    """Selected indices, value trajectory, work done (optimize.py:24-30)."""

    exemplar_indices: tuple
    values: tuple
    evaluations: int


class GreedyRun:
    """Device state of one Greedy run over a (shard of a) ground set.

    ``dg``      point shard whose m_i this run owns (SIMT layout).
    ``cand``    candidate layouts (== dg on a single GPU; the full V when the
                points are row-sharded, see ``distributed.py``).
    """

    def __init__(self, dg, cand=None, k_cap: int = 1, split_pts=None,
                 tc: Optional[bool] = None, split32: bool = False):
        from .device import torch

        t = torch()
        self.t = t
        self.lib = N.lib()
        self.dg = dg
        self.cand = cand or dg
        self.prec = dg.precision
        self.tc = self.prec.is_half if tc is None else tc
        if self.tc and not (dg.fold_ok() and self.cand.fold_ok()):
            raise_fold_range(self.prec)
        # binary32 gains on the tensor cores through split-bf16 operands
        # (exem_tc_pack_split): the K3-TC kernel with d' = 6d
        # (d <= 128: beyond, the tensor core's fp32 accumulation over
        # K' = 6d + 6 terms exceeds the binary32 tolerance on the gains --
        # measured 1.09e-5 at d = 256 -- so larger d keeps the SIMT path)
        self.split32 = (bool(split32) and self.prec.tag == N.F32 and
                        dg.d <= SPLIT32_MAX_D)
        if self.split32:
            self.tc = True
        self.split_pts = int(split_pts or dg.split_pts)
        self.splits = -(-dg.n // self.split_pts)
        self.l = self.cand.n
        dev = dg.dev
        self.m = t.empty(dg.ld, dtype=dg.cdtype, device=dev)
        self.selected = t.zeros(max(self.l, 1), dtype=t.uint8, device=dev)
        self.gains = t.empty(self.l, dtype=t.float64, device=dev)
        self.sel_idx = t.zeros(k_cap, dtype=t.int64, device=dev)
        self.sel_gain = t.zeros(k_cap, dtype=t.float64, device=dev)
        self.msum = t.zeros(k_cap, dtype=t.float64, device=dev)
        self.msum0 = t.zeros(1, dtype=t.float64, device=dev)
        self.scratch = t.empty(int(self.lib.reduce_scratch(max(dg.ld, self.l))),
                               dtype=t.float64, device=dev)
        self._partial = None
        self.xp = None
        self.xc = None
        # K3-TC epilogue width (0: not decided yet) and its screen counter
        self.epi = 0
        self.hit_fraction = None
        self.hits = t.zeros(1, dtype=t.int64, device=dev)
        self.tc_tag = self.prec.tag
        self.tc_d = dg.d
        if self.split32:
            self.tc_tag = N.BF16
            self.tc_d = int(self.lib.tc_split_dim(dg.d))
            self.kp = int(self.lib.tc_kp(self.tc_d))
            rows = int(self.lib.tc_rows(dg.n))
            self.xp = t.empty((rows, self.kp), dtype=t.bfloat16, device=dev)
            self.xc = self.cand.xc_split()
        elif self.tc:
            self.kp = dg.kp
            rows = int(self.lib.tc_rows(dg.n))
            tdt = t.bfloat16 if self.prec.tag == N.BF16 else t.float16
            self.xp = t.empty((rows, dg.kp), dtype=tdt, device=dev)
            self.xc = self.cand.xc()

    def partial(self, cols: int):
        need = self.splits * cols
        if self._partial is None or self._partial.numel() < need:
            self._partial = self.t.empty(need, dtype=self.t.float64,
                                         device=self.dg.dev)
        return self._partial

    @property
    def stream(self):
        return self.dg.stream

    def start(self):
        """m <- aux (S = {}); build the TC point operand from it."""
        dg, lib = self.dg, self.lib
        lib.greedy_init(self.prec.tag, N.ptr(dg.aux), dg.n, N.ptr(self.m),
                        N.ptr(self.msum0), N.ptr(self.scratch), self.stream)
        if self.split32:
            lib.tc_pack_split(1, N.ptr(dg.vt), dg.ld, dg.n, dg.d,
                              N.ptr(dg.norms), N.ptr(self.m), N.ptr(self.xp),
                              self.stream)
        elif self.tc:
            lib.tc_pack_points(dg.vt_tag, N.ptr(dg.vt), dg.ld, dg.n, dg.d,
                               N.ptr(dg.norms), N.ptr(self.m), N.ptr(self.xp),
                               self.stream)

    def compute_gains(self, chunk: Optional[int] = None, out=None):
        """K3 + K6: gains[c] = sum_{local i} max(0, m_i - d(v_i, c)), into
        ``self.gains`` or the device buffer at pointer ``out``."""
        dg, cd, lib, st = self.dg, self.cand, self.lib, self.stream
        chunk = self.l if not chunk or chunk >= self.l else chunk
        esz = dg.vt_c().element_size() if not self.tc else 0
        for c0 in range(0, self.l, chunk):
            cl = min(chunk, self.l - c0)
            part = self.partial(cl)
            if self.tc:
                xc_ptr = N.c_void_p(self.xc.data_ptr() +
                                    c0 * self.kp * self.xc.element_size())
                probe = self.epi == 0
                lib.greedy_gains_tc_ex(self.tc_tag, xc_ptr, cl, N.ptr(self.xp),
                                       dg.n, self.tc_d, self.split_pts,
                                       N.ptr(part), self.splits,
                                       2 if probe else self.epi,
                                       N.ptr(self.hits) if probe else None, st)
            else:
                # the CUDA-core K3 reads 4/8-byte V (widened half storage)
                cvt_ptr = N.c_void_p(cd.vt_c().data_ptr() + c0 * esz)
                cn_ptr = N.c_void_p(cd.norms.data_ptr() + c0 * 8)
                lib.greedy_gains_simt(self.prec.tag, cvt_ptr, cd.ld, cn_ptr,
                                      cl, N.ptr(dg.vt_c()), dg.ld,
                                      N.ptr(dg.norms),
                                      N.ptr(self.m), dg.n, dg.d,
                                      self.split_pts, N.ptr(part),
                                      self.splits, st)
            base = self.gains.data_ptr() if out is None else out.value
            lib.reduce_partials(N.ptr(part), self.splits, cl, 2.0,
                                N.c_void_p(base + c0 * 8), st)
        if self.tc and self.epi == 0:
            self._decide_epi()

    def _decide_epi(self):
        """One host read of the screen counter after the first gains launch
        (step 0; steps replayed from a CUDA graph are captured after it)."""
        screens = (-(-self.l // 128) * 128) * (-(-self.dg.n // 256) * 8)
        self.hit_fraction = int(self.hits.item()) / max(1, screens)
        self.epi = 4 if self.hit_fraction > EPI_WIDE_THRESHOLD else 2
        forced = os.environ.get("EXEM_K3_EPI")  # timing experiments only
        if forced in ("2", "4"):
            self.epi = int(forced)

    def select(self, step: int):
        """K5: masked argmax (lowest index on ties) -> sel_idx[step]."""
        self.lib.argmax_select(N.ptr(self.gains), self.l, N.ptr(self.selected),
                               None, step, N.ptr(self.sel_idx),
                               N.ptr(self.sel_gain), N.ptr(self.scratch),
                               self.stream)

    def update(self, step: int):
        """K2: m_i <- min(m_i, d(v_i, c*)); msum[step] = sum_i m_i."""
        dg, cd = self.dg, self.cand
        assert dg.vt_flag == cd.vt_flag  # same precision: same vt layout
        self.lib.greedy_update(
            dg.vt_tag, N.ptr(dg.vt), dg.ld, dg.n, dg.d, N.ptr(dg.norms),
            N.ptr(cd.vt), cd.ld, N.ptr(cd.norms), N.ptr(self.sel_idx), step,
            N.ptr(self.m), None if self.split32 else N.ptr(self.xp), dg.kp,
            N.ptr(self.msum), N.ptr(self.scratch), self.stream)
        if self.split32:
            self.lib.tc_refresh_h(N.ptr(dg.norms), N.ptr(self.m), dg.n,
                                  N.ptr(self.xp), self.kp, self.tc_d,
                                  self.stream)

    def force(self, step: int, index: int):
        """Teacher forcing: take ``index`` as the exemplar of ``step``
        (instead of K5's argmax), then K2 as usual.  No gains are needed
        for a forced step."""
        self.sel_idx[step] = int(index)
        self.selected[int(index)] = 1
        self.update(step)

    def step(self, step: int, chunk: Optional[int] = None):
        self.compute_gains(chunk)
        self.select(step)
        self.update(step)


def capture_steps(steps, do_step):
    """Record ``do_step(t)`` for every t in ``steps`` into ONE CUDA graph and
    return it (``graph.replay()`` runs them).

    A Greedy step is K3 -> K6 -> [all-reduce] -> K5 -> K2 with no host
    synchronisation, and the step index only selects where K5/K2 write
    (sel_idx[t], msum[t]), so the whole k-step loop -- including the NCCL
    all-reduce of a row-sharded run -- is capturable: one graph launch
    replaces ~5 launches per step and takes the host out of the loop
    (SURVEY.md 8(e)).  Every kernel of the library launches on torch's
    current stream, which ``torch.cuda.graph`` makes the capture stream.
    The kernels must have run once before (module load, smem attributes).
    """
    from .device import torch

    t = torch()
    graph = t.cuda.CUDAGraph()
    with t.cuda.graph(graph):
        for step in steps:
            do_step(step)
    return graph


def raise_fold_range(precision) -> None:
    """Greedy runs half precisions on the tensor cores only; binary16 norms
    beyond the folded operand range (device.F16_FOLD_MAX_NORM) cannot be
    represented there."""
    from .device import F16_FOLD_MAX_NORM

    raise InvalidDataError(
        f"{precision.name} Greedy: squared norms reach beyond "
        f"{F16_FOLD_MAX_NORM:.3g}, the range of the binary16 tensor-core "
        "operands; use Precision.binary32 (evaluate_single / evaluate_batch "
        "handle such data at binary16 on the CUDA cores)")


def checked_picks(idx: np.ndarray, k: int) -> np.ndarray:
    """The first k device picks; K5 writes -1 when a step had no valid
    candidate (every remaining gain NaN), which is an error here rather than
    a silent duplicate exemplar."""
    idx = np.asarray(idx)[:k]
    bad = np.flatnonzero(idx < 0)
    if bad.size:
        raise InvalidDataError(
            f"greedy step {int(bad[0])} found no valid candidate "
            "(every remaining marginal gain is NaN)")
    return idx


def _chunk_for_budget(ground: GroundSet, step: int, budget: Optional[int]):
    """Candidate chunk size under the reference's mu_s rule (or None)."""
    if budget is None:
        return None
    mu = estimate_set_memory(ground.n, step + 1, ground.d, ground.precision)
    plan = plan_chunks(budget, mu, ground.n - step)
    size = plan.chunk_size
    return max(256, size // 256 * 256) if size < ground.n else None


def trajectory_values(ground: GroundSet, msum: np.ndarray) -> tuple:
    """values[t] = acc(aux_loss) - acc(sum_i m_i)/acc(n) (evaluate.py:111-112)."""
    acc = ground.precision.accumulate_dtype
    vals = acc.type(ground.aux_loss) - msum.astype(acc) / acc.type(ground.n)
    return tuple(float(v) for v in vals)


def greedy_maximize(ground: GroundSet, k: int,
                    evaluator: Optional[Evaluator] = None,
                    dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN,
                    memory_budget: Optional[int] = None) -> OptimizationResult:
    """Select up to k exemplars, one argmax-gain candidate per step."""
    require_device_dissimilarity(dissimilarity)
    if k > ground.n:
        raise BudgetExceedsGroundSetError(
            f"k={k} exceeds the {ground.n} available observations")
    evaluator = evaluator or Evaluator()
    if k <= 0:
        return OptimizationResult(exemplar_indices=(), values=(), evaluations=0)
    _effective_precision(evaluator, ground)
    if ground.streamed:
        # V over the device budget: candidates and points stream through in
        # resident chunks / split-aligned slices (streaming.py); bit-identical
        # to the resident run
        from .streaming import stream_greedy

        idx, msum = stream_greedy(ground, k, evaluator.device)
        return OptimizationResult(
            exemplar_indices=tuple(int(i) for i in checked_picks(idx, k)),
            values=trajectory_values(ground, msum[:k]),
            evaluations=sum(ground.n - i for i in range(k)),
        )
    dg = ground.on_device(evaluator.device)
    from .device import torch

    with torch().cuda.device(dg.device_index):
        run = GreedyRun(dg, k_cap=k, split32=evaluator.tensor_fp32)
        run.start()
        chunks = [_chunk_for_budget(ground, step, memory_budget)
                  for step in range(k)]
        if evaluator.cuda_graph and k > 1:
            # step 0 eagerly (loads every kernel), steps 1..k-1 as one graph
            run.step(0, chunks[0])
            capture_steps(range(1, k),
                          lambda s: run.step(s, chunks[s])).replay()
        else:
            for step in range(k):
                run.step(step, chunks[step])
        idx = run.sel_idx.cpu().numpy()
        msum = run.msum.cpu().numpy()
    return OptimizationResult(
        exemplar_indices=tuple(int(i) for i in checked_picks(idx, k)),
        values=trajectory_values(ground, msum[:k]),
        evaluations=sum(ground.n - i for i in range(k)),
    )


def brute_force_optimum(ground: GroundSet, k: int,
                        dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN):
    """Exhaustive optimum over size-k subsets (optimize.py:85-112).

    Scored in device batches of explicit sets (K4); the first maximum in
    ``itertools.combinations`` order wins, as in the reference's strict '>'.
    """
    require_device_dissimilarity(dissimilarity)
    if k > ground.n:
        raise BudgetExceedsGroundSetError(
            f"k={k} exceeds the {ground.n} available observations")
    if k <= 0:
        return (), 0.0
    if math.comb(ground.n, k) > BRUTE_FORCE_LIMIT:
        raise InstanceTooLargeError(
            f"C({ground.n}, {k}) subsets exceed the exhaustive-search guard")
    best_set, best_val = (), -math.inf
    combos = itertools.combinations(range(ground.n), k)
    while True:
        block = list(itertools.islice(combos, 65536))
        if not block:
            break
        batch = EvaluationBatch.from_sets([ground.matrix[list(c)] for c in block])
        vals = np.asarray(evaluate_batch(Evaluator(), ground, batch),
                          dtype=np.float64)
        j = int(np.argmax(vals))
        if vals[j] > best_val:
            best_set, best_val = tuple(block[j]), float(vals[j])
    return best_set, best_val


def assign_clusters(ground: GroundSet, exemplars,
                    dissimilarity: Dissimilarity = SQUARED_EUCLIDEAN) -> np.ndarray:
    """Nearest-exemplar label per observation, lowest index on ties
    (optimize.py:115-136) -- the argmin epilogue of kernel K2."""
    require_device_dissimilarity(dissimilarity)
    elems = _as_elements(ground, exemplars)
    if elems.shape[0] == 0:
        raise EmptyEvaluationSetError("cluster assignment needs at least one exemplar")
    _, _, labels = device_set_min(ground, elems, include_aux=False,
                                  want_labels=True)
    return labels.astype(np.int64)
