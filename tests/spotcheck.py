"""Teacher-forced Greedy parity helpers (SURVEY.md 8(c) "Large-n parity").

The reference is infeasible at the benchmark sizes (C4: months of CPU), so
at a set of Greedy steps the device's state is re-derived independently on
the host in fp64 from the STORED values and the device's own picks so far
(teacher forcing: a near-tie never ends the comparison):

    m_i  = min(aux_i, min_{s in S_t} d(v_i, s))        (objective.py:113-141)
    G_c  = sum_i max(0, m_i - d(v_i, c))               (the K3 quantity)
    f(S) = aux_loss - sum_i m_i / n                    (evaluate.py:105-112)

and compared with the device's gains for its argmax, its runner-up and
random candidates, and with the device's trajectory values.  The pick must
be the argmax of the host gains over the checked candidates within the
stated gain tolerance (a documented near-tie otherwise).

Errors are appended as JSON lines to $EXEM_PARITY_LOG when set (the
measured maxima behind the tolerances in DESIGN.md section 4).
"""

from __future__ import annotations

import json
import os

import numpy as np

import exem_oracle as O  # checker only


def log(record: dict) -> None:
    path = os.environ.get("EXEM_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(record) + "\n")


def d64(x: np.ndarray, c: np.ndarray, block: int = 1 << 16) -> np.ndarray:
    """fp64 squared distances of every row of x to the vector c (direct
    form, blocked to bound memory)."""
    out = np.empty(x.shape[0])
    for lo in range(0, x.shape[0], block):
        diff = x[lo:lo + block] - c[None, :]
        out[lo:lo + block] = np.einsum("ij,ij->i", diff, diff)
    return out


def host_m(x: np.ndarray, aux: np.ndarray, picks) -> np.ndarray:
    m = np.asarray(aux, np.float64).copy()
    for s in picks:
        np.minimum(m, d64(x, x[s]), out=m)
    return m


def host_gains(x: np.ndarray, m: np.ndarray, cands) -> np.ndarray:
    return np.array([np.maximum(m - d64(x, x[c]), 0.0).sum() for c in cands])


def device_greedy_with_checks(g, k: int, check_steps, n_random: int = 16,
                              seed: int = 0, split32: bool = False,
                              forced=None):
    """Run k Greedy steps on the device (K3 -> K6 -> K5 -> K2) and capture,
    at each step in ``check_steps`` (0-based), the device gains of the
    argmax, the runner-up and ``n_random`` random unselected candidates.
    ``forced`` (optional list) overrides the device's picks (teacher
    forcing from given exemplars).  Returns (picks, values, captures)."""
    import torch

    from paper_2101_08763_b200.optimize import GreedyRun, trajectory_values

    rng = np.random.default_rng(seed)
    dg = g.on_device()
    caps = []
    with torch.cuda.device(dg.device_index):
        run = GreedyRun(dg, k_cap=k, split32=split32)
        run.start()
        for step in range(k):
            run.compute_gains()
            if step in check_steps:
                G = run.gains.cpu().numpy().copy()
                sel = run.selected[: run.l].cpu().numpy().astype(bool)
                Gm = np.where(sel, -np.inf, G)
                order = np.argsort(-Gm, kind="stable")
                top, second = int(order[0]), int(order[1])
                free = np.flatnonzero(~sel)
                rand = rng.choice(free, size=min(n_random, free.size),
                                  replace=False)
                cands = [top, second] + [int(c) for c in rand
                                         if c not in (top, second)]
                caps.append({"step": step, "cands": cands,
                             "G_dev": G[cands], "top": top})
            if forced is None:
                run.select(step)
                run.update(step)
            else:
                run.force(step, int(forced[step]))
        picks = run.sel_idx.cpu().numpy()[:k].tolist()
        msum = run.msum.cpu().numpy()[:k]
    return picks, list(trajectory_values(g, msum)), caps


def check_captures(g, picks, values, caps, gain_tol, value_tol, label=""):
    """Host fp64 re-derivation at the captured steps.  ``gain_tol(G)`` and
    ``value_tol(f)`` give the absolute bounds.  Returns the measured maxima
    (relative gain error, value error relative to max(1,|f|))."""
    x = np.asarray(g.matrix, np.float64)
    n = x.shape[0]
    aux = np.asarray(g.aux_distances, np.float64)
    worst_g, worst_v = 0.0, 0.0
    for cap in caps:
        t = cap["step"]
        m = host_m(x, aux, picks[:t])
        Gh = host_gains(x, m, cap["cands"])
        Gd = np.asarray(cap["G_dev"])
        err = np.abs(Gd - Gh)
        tol = np.array([gain_tol(v) for v in Gh])
        assert np.all(err <= tol), (label, t, err.max(), (err / tol).max())
        worst_g = max(worst_g, float((err / np.maximum(1.0, np.abs(Gh))).max()))
        # the device pick is the argmax of the host gains within tolerance
        best = float(Gh.max())
        assert Gh[0] >= best - gain_tol(best), (label, t, Gh[0], best)
        # the trajectory value after this step's pick
        m1 = np.minimum(m, d64(x, x[picks[t]]))
        f_host = g.aux_loss - m1.sum() / n
        ev = abs(values[t] - f_host)
        assert ev <= value_tol(f_host), (label, t, values[t], f_host)
        worst_v = max(worst_v, ev / max(1.0, abs(f_host)))
    log({"check": label, "n": n, "d": x.shape[1], "steps": [c["step"]
         for c in caps], "max_rel_gain_err": worst_g,
         "max_rel_value_err": worst_v})
    return worst_g, worst_v


def teacher_forced_trajectory(g, res, gain_tol, value_tol, label=""):
    """Every step of a small Greedy: host fp64 gains over ALL candidates
    given the device's S_t; the device's pick must be a maximiser within
    ``gain_tol`` (near-ties documented by the tolerance, the comparison
    continues from the device's S), and its value must match f(S_{t+1})."""
    x = np.asarray(g.matrix, np.float64)
    n = x.shape[0]
    aux = np.asarray(g.aux_distances, np.float64)
    m = aux.copy()
    chosen = np.zeros(n, bool)
    ties = 0
    worst_v = 0.0
    for t, c in enumerate(res.exemplar_indices):
        G = O.gains_m(x, m, x)  # fp64, all candidates
        G[chosen] = -np.inf
        best = int(np.argmax(G))
        assert not chosen[c]
        assert G[c] >= G[best] - gain_tol(G[best]), (label, t, c, best,
                                                     G[c], G[best])
        ties += int(c != best)
        chosen[c] = True
        np.minimum(m, d64(x, x[c]), out=m)
        f_host = g.aux_loss - m.sum() / n
        assert abs(res.values[t] - f_host) <= value_tol(f_host), (
            label, t, res.values[t], f_host)
        worst_v = max(worst_v, abs(res.values[t] - f_host) /
                      max(1.0, abs(f_host)))
    log({"check": label, "n": n, "d": x.shape[1], "k": len(res.exemplar_indices),
         "near_ties": ties, "max_rel_value_err": worst_v})
    return ties
