"""Sieve-Streaming maximization over the device evaluator.

The north star names "the Greedy and streaming optimizers"; the reference
ships only Greedy (streaming optimizers are explicit non-goals there,
SPEC.md:9,402).  This module adds the classic
one-pass SieveStreaming (Badanidiyuru, Mirzasoleiman, Karbasi, Krause,
KDD 2014) with the on-the-fly singleton maximum, driven by the same
optimizer-aware state as the device Greedy: every sieve keeps its per-point
minimum m_i = min(aux_i, min_{s in S} d(v_i, s)) on the device, so the
marginal gains of a block of arriving elements for all sieves at once are
one pass of ``exem_sieve_block_dist`` (K2's distances, every element's row
kept) plus one ``exem_sieve_block_gains`` launch, and accepting e is one
``exem_sieve_update``.

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
                             device=None, block: int = 64) -> OptimizationResult:
    """One pass over the stream; returns the best sieve's exemplars (in
    acceptance order), its value trajectory f(S_1..S_|S|), and the number of
    marginal-gain evaluations (sieves probed).

    The stream is processed ``block`` elements at a time: one pass of K2
    writes the block's distance rows D[b][i] = d(v_i, e_b), one launch scores
    every (sieve, element) pair, gains[s][b] = sum_i max(0, m_s[i] - D[b][i]),
    and the host walks the block in stream order.  Accepting e_b into a sieve
    changes only that sieve's m-row, so only its gains for the rest of the
    block are rescored -- the decisions are those of the element-at-a-time
    algorithm (acceptances are rare: at most k per sieve)."""
    from .device import padded_rows, torch

    if k > ground.n:
        raise BudgetExceedsGroundSetError(
            f"k={k} exceeds the {ground.n} available observations")
    if k <= 0:
        return OptimizationResult(exemplar_indices=(), values=(), evaluations=0)
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must be in (0, 1)")
    if block < 1:
        raise ValueError("block must be >= 1")
    t = torch()
    lib = N.lib()
    dg = ground.on_device(device)
    prec = ground.precision
    n = ground.n
    acc = prec.accumulate_dtype
    aux_loss = float(acc.type(ground.aux_loss))
    cap = len(sieve_thresholds(1.0, k, eps)) + 2  # sieves alive at once
    stream = (np.arange(n, dtype=np.int64) if order is None
              else np.asarray(order, dtype=np.int64).reshape(-1))
    rows = cap + 1
    with t.cuda.device(dg.device_index):
        st = dg.stream
        cdt = dg.aux.dtype
        # row 0 = aux (the empty set: gains are singleton values), rows 1.. =
        # sieve m-vectors
        M = t.empty((rows, dg.ld), dtype=cdt, device=dg.dev)
        M[0].copy_(dg.aux)
        D = t.empty((block, dg.ld), dtype=cdt, device=dg.dev)
        G = t.empty((rows, block), dtype=t.float64, device=dg.dev)
        # Gr[:block] one row's rescored gains, Gr[block] its new sum_i m_i:
        # one device -> host copy per acceptance
        Gr = t.empty(block + 1, dtype=t.float64, device=dg.dev)
        scratch = t.empty(max(int(lib.sieve_block_scratch(n, rows, block)),
                              int(lib.reduce_scratch(n)), 1),
                          dtype=t.float64, device=dg.dev)
        en = t.empty(block, dtype=t.float64, device=dg.dev)
        free_rows = list(range(cap, 0, -1))
        sieves = {}  # j -> dict(row, picks, values, f)
        m_star, evaluations = 0.0, 0

        msum_ptr = N.c_void_p(Gr.data_ptr() + 8 * block)

        def accept(r, bi, nb, rescore):
            """m_r <- min(m_r, D[bi]); rescore row r against the block's
            elements bi+1..nb-1.  Returns (sum_i m_i, gains) -- one sync."""
            lib.sieve_update(prec.tag, N.c_void_p(M[r].data_ptr()),
                             N.c_void_p(D[bi].data_ptr()), n, msum_ptr,
                             N.ptr(scratch), st)
            cnt = nb - bi - 1 if rescore else 0
            if cnt > 0:
                lib.sieve_block_gains(
                    prec.tag, N.c_void_p(M[r].data_ptr()), dg.ld, 1,
                    N.c_void_p(D[bi + 1].data_ptr()), dg.ld, cnt, n,
                    N.ptr(Gr), N.ptr(scratch), st)
            host = Gr.cpu().numpy()
            return float(host[block]), host[:cnt] / n

        for b0 in range(0, len(stream), block):
            idx = stream[b0:b0 + block]
            nb = len(idx)
            E = padded_rows(ground.matrix[idx], dg.d_pad, prec, dg.dev)
            lib.row_norms(prec.tag, N.ptr(E), nb, dg.d, dg.d_pad, N.ptr(en), st)
            lib.sieve_block_dist(prec.tag, N.ptr(dg.vt_c()), dg.ld, n, dg.d,
                                 N.ptr(dg.norms), N.ptr(E), N.ptr(en), nb,
                                 N.ptr(D), dg.ld, N.ptr(scratch), st)
            lib.sieve_block_gains(prec.tag, N.ptr(M), dg.ld, rows, N.ptr(D),
                                  dg.ld, nb, n, N.ptr(G), N.ptr(scratch), st)
            g = G.view(-1)[: rows * nb].view(rows, nb).cpu().numpy() / n
            # rows reset to aux inside this block and not yet grown: their
            # block gains are the singleton column g[0] (M was stale when
            # the block was scored)
            fresh = set()
            for bi in range(nb):
                e = int(idx[bi])
                m_star = max(m_star, float(g[0, bi]))
                live = sieve_thresholds(m_star, k, eps)
                for j in [j for j in sieves if j not in live]:
                    free_rows.append(sieves.pop(j)["row"])
                for j in live:
                    if j not in sieves:
                        r = free_rows.pop()
                        M[r].copy_(dg.aux)
                        sieves[j] = {"row": r, "picks": [], "values": [],
                                     "f": 0.0}
                        fresh.add(r)
                for j in live:
                    sv = sieves[j]
                    size = len(sv["picks"])
                    if size >= k:
                        continue
                    evaluations += 1
                    r = sv["row"]
                    delta = float(g[0, bi]) if r in fresh else float(g[r, bi])
                    v = (1.0 + eps) ** j
                    if delta >= (v / 2.0 - sv["f"]) / (k - size):
                        total, fresh_g = accept(r, bi, nb, size + 1 < k)
                        f = float(acc.type(aux_loss) - acc.type(total)
                                  / acc.type(n))
                        sv["picks"].append(e)
                        sv["values"].append(f)
                        sv["f"] = f
                        fresh.discard(r)
                        if len(fresh_g):
                            g[r, bi + 1:nb] = fresh_g
    if not sieves:
        return OptimizationResult(exemplar_indices=(), values=(),
                                  evaluations=evaluations)
    # best value; ties -> the lowest threshold
    j_best = max(sorted(sieves), key=lambda j: sieves[j]["f"])
    best = sieves[j_best]
    return OptimizationResult(exemplar_indices=tuple(best["picks"]),
                              values=tuple(best["values"]),
                              evaluations=evaluations)
