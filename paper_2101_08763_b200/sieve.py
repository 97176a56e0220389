"""Sieve-Streaming maximization over the device evaluator.

The north star names "the Greedy and streaming optimizers"; the reference
ships only Greedy (streaming optimizers are explicit non-goals there,
SPEC.md:9,402).  This module adds the classic
one-pass SieveStreaming (Badanidiyuru, Mirzasoleiman, Karbasi, Krause,
KDD 2014) with the on-the-fly singleton maximum, driven by the same
optimizer-aware state as the device Greedy: every sieve keeps its per-point
minimum m_i = min(aux_i, min_{s in S} d(v_i, s)) on the device, so the
marginal gain of an arriving element e for all sieves at once is one pass
of ``exem_sieve_gains`` over the distances d(v_i, e) (``exem_set_min`` with
k = 1), and accepting e is one ``exem_sieve_update``.

Per element e (stream order = ``order`` or index order):
    f({e}) = n^-1 sum_i max(0, aux_i - d(v_i, e));  m* = max(m*, f({e}))
    thresholds O = {(1+eps)^j : m* <= (1+eps)^j <= 2 k m*}  (sieves outside O
    are dropped, new ones start empty)
    for each sieve v with |S_v| < k:
        accept e  iff  Delta(e | S_v) >= (v/2 - f(S_v)) / (k - |S_v|)
The result is the best sieve; f(S) >= (1/2 - eps) OPT (the paper's bound).
The tests compare against an fp64 host restatement of the same algorithm in
the test oracle (``sieve_streaming``).
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .core import GroundSet
from .errors import BudgetExceedsGroundSetError
from .optimize import OptimizationResult


def sieve_thresholds(m_star: float, k: int, eps: float) -> list:
    """Integer exponents j with m* <= (1+eps)^j <= 2 k m*."""
    if m_star <= 0.0:
        return []
    base = math.log1p(eps)
    lo = math.ceil(math.log(m_star) / base - 1e-12)
    hi = math.floor(math.log(2.0 * k * m_star) / base + 1e-12)
    return list(range(lo, hi + 1))


def sieve_streaming_maximize(ground: GroundSet, k: int, eps: float = 0.1,
                             order: Optional[Sequence[int]] = None,
                             device=None) -> OptimizationResult:
    """One pass over the stream; returns the best sieve's exemplars (in
    acceptance order), its value trajectory f(S_1..S_|S|), and the number of
    marginal-gain evaluations (sieves probed)."""
    from .device import padded_rows, torch

    if k > ground.n:
        raise BudgetExceedsGroundSetError(
            f"k={k} exceeds the {ground.n} available observations")
    if k <= 0:
        return OptimizationResult(exemplar_indices=(), values=(), evaluations=0)
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must be in (0, 1)")
    t = torch()
    lib = N.lib()
    dg = ground.on_device(device)
    prec = ground.precision
    n = ground.n
    acc = prec.accumulate_dtype
    aux_loss = float(acc.type(ground.aux_loss))
    cap = len(sieve_thresholds(1.0, k, eps)) + 2  # sieves alive at once
    stream = range(n) if order is None else order
    with t.cuda.device(dg.device_index):
        st = dg.stream
        cdt = dg.aux.dtype
        # row 0 = aux (the empty set: gains are singleton values), rows 1.. =
        # sieve m-vectors
        M = t.empty((cap + 1, dg.ld), dtype=cdt, device=dg.dev)
        M[0].copy_(dg.aux)
        dist = t.empty(dg.ld, dtype=cdt, device=dg.dev)
        gains = t.empty(cap + 1, dtype=t.float64, device=dg.dev)
        msum = t.empty(1, dtype=t.float64, device=dg.dev)
        blocks = -(-n // 256)
        scratch = t.empty(max(blocks * (cap + 1), int(lib.reduce_scratch(n))),
                          dtype=t.float64, device=dg.dev)
        free_rows = list(range(cap, 0, -1))
        sieves = {}  # j -> dict(row, picks, values, f)
        m_star, evaluations = 0.0, 0
        for e in stream:
            e = int(e)
            row_e = padded_rows(ground.matrix[e:e + 1], dg.d_pad, prec, dg.dev)
            en = t.empty(1, dtype=t.float64, device=dg.dev)
            lib.row_norms(prec.tag, N.ptr(row_e), 1, dg.d, dg.d_pad, N.ptr(en),
                          st)
            lib.set_min(prec.tag, N.ptr(dg.vt), dg.ld, n, dg.d,
                        N.ptr(dg.norms), N.ptr(dg.aux), N.ptr(row_e),
                        N.ptr(en), 1, 0, N.ptr(dist), None, None,
                        N.ptr(scratch), st)
            lib.sieve_gains(prec.tag, N.ptr(M), dg.ld, cap + 1, N.ptr(dist),
                            n, N.ptr(gains), N.ptr(scratch), st)
            g = gains.cpu().numpy() / n
            m_star = max(m_star, float(g[0]))
            live = sieve_thresholds(m_star, k, eps)
            for j in [j for j in sieves if j not in live]:
                free_rows.append(sieves.pop(j)["row"])
            fresh = set()
            for j in live:
                if j not in sieves:
                    r = free_rows.pop()
                    M[r].copy_(dg.aux)
                    sieves[j] = {"row": r, "picks": [], "values": [], "f": 0.0}
                    fresh.add(j)
            for j in live:
                sv = sieves[j]
                size = len(sv["picks"])
                if size >= k:
                    continue
                evaluations += 1
                # a sieve created for this element is empty: its gain is the
                # singleton value (its M row was stale when gains ran)
                delta = float(g[0]) if j in fresh else float(g[sv["row"]])
                v = (1.0 + eps) ** j
                if delta >= (v / 2.0 - sv["f"]) / (k - size):
                    lib.sieve_update(prec.tag,
                                     N.c_void_p(M[sv["row"]].data_ptr()),
                                     N.ptr(dist), n, N.ptr(msum),
                                     N.ptr(scratch), st)
                    f = float(acc.type(aux_loss) - acc.type(msum.item())
                              / acc.type(n))
                    sv["picks"].append(e)
                    sv["values"].append(f)
                    sv["f"] = f
    if not sieves:
        return OptimizationResult(exemplar_indices=(), values=(),
                                  evaluations=evaluations)
    # best value; ties -> the lowest threshold
    j_best = max(sorted(sieves), key=lambda j: sieves[j]["f"])
    best = sieves[j_best]
    return OptimizationResult(exemplar_indices=tuple(best["picks"]),
                              values=tuple(best["values"]),
                              evaluations=evaluations)
