"""Parity at the BASELINE scales (SURVEY.md 8(c) "Large-n parity").

C4 (n = 1M, d = 100): the device Greedy in every precision path -- bf16 and
f16 tcgen05 (K3-TC), binary32 on the CUDA cores (K3-SIMT) and binary32 on the
tensor cores (split-bf16) -- is spot-checked at steps {1, 5, k}: the gains of
the device's argmax, its runner-up and 16 random candidates are recomputed
in fp64 on the host from the stored values and the device's own picks
(teacher forced), the pick must be the host argmax over them within the gain
tolerance, and the recorded value must equal the host f(S_t).

C2 (n = 100k, d = 100, binary32, |S u c| = 20): with S = 19 seeded
exemplars forced on the device, f(S u {c}) = f(S) + G_c / n for the argmax,
the runner-up and ~200 random candidates equals the ORACLE's explicit
evaluation of S u {c} in the reference's own fp32 op order
(oracle.evaluate_batch = evaluate.py:142-149) within the binary32 contract,
and equals the device's explicit-set kernel (K4) on the same sets.

C3 SIMT shapes (d = 512 / 1024 at binary32 and binary64, d = 100 at
binary64): every Greedy step teacher-forced against fp64 truth, and explicit
batches against the oracle.

Tolerances (parity contract):
  binary64  gains 1e-11 * max(1,G); values 1e-12 * max(1,|f|)
  binary32  gains 1e-5 * max(1,G);  values 1e-5 * max(1,|f|) + 2 ulp32(aux_loss)
  half      gains HALF_GAIN * max(1,G); values HALF_VALUE * max(1,|f|)
            + 2 ulp32(aux_loss)  (tests/contract.py)
"""

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import EvaluationBatch, Evaluator, Precision
from spotcheck import (check_captures, device_greedy_with_checks,
                       teacher_forced_trajectory)

pytestmark = pytest.mark.gpu

P16, BF16, P32, P64 = (Precision.binary16, Precision.bfloat16,
                       Precision.binary32, Precision.binary64)

from contract import HALF_F_REL as HALF_VALUE  # noqa: E402
from contract import HALF_G_REL as HALF_GAIN  # noqa: E402
from contract import SPLIT32_G_REL  # noqa: E402


def _ulp32(x):
    return float(np.spacing(np.float32(abs(x))))


def _tols(prec, aux_loss):
    slack = 2 * _ulp32(aux_loss)
    if prec is P64:
        return (lambda G: 1e-11 * max(1.0, abs(G)),
                lambda f: 1e-12 * max(1.0, abs(f)))
    if prec is P32:
        return (lambda G: 1e-5 * max(1.0, abs(G)),
                lambda f: 1e-5 * max(1.0, abs(f)) + slack)
    return (lambda G: HALF_GAIN * max(1.0, abs(G)),
            lambda f: HALF_VALUE * max(1.0, abs(f)) + slack)


@pytest.fixture(scope="module")
def c4_data():
    return np.random.default_rng(0).standard_normal((1_000_000, 100),
                                                    dtype=np.float32)


@pytest.mark.parametrize("prec,split32,k", [
    (BF16, False, 10), (P16, False, 10), (P32, True, 10), (P32, False, 5)])
def test_c4_spot_checks(c4_data, prec, split32, k):
    g = pb.build_ground_set(c4_data, precision=prec)
    steps = sorted({0, 4, k - 1})
    picks, values, caps = device_greedy_with_checks(g, k, steps, seed=k,
                                                    split32=split32)
    assert len(set(picks)) == k
    gt, vt = _tols(prec, g.aux_loss)
    if split32:  # binary32 values; gains carry the tensor core's fp32 sums
        gt = lambda G: SPLIT32_G_REL * max(1.0, abs(G))  # noqa: E731
    check_captures(g, picks, values, caps, gt, vt,
                   label=f"C4 {prec.name}{' split32' if split32 else ''}")
    # the public API returns the same trajectory
    res = pb.greedy_maximize(g, k=k, evaluator=Evaluator(tensor_fp32=split32))
    assert list(res.exemplar_indices) == picks
    assert list(res.values) == values


def test_c2_forced_step_vs_oracle_explicit_sets():
    n, d = 100_000, 100
    rng = np.random.default_rng(2)
    V = rng.standard_normal((n, d), dtype=np.float32)
    g = pb.build_ground_set(V, precision=P32)
    S = [int(i) for i in rng.choice(n, size=19, replace=False)]
    k = 20
    # steps 0..18 forced to S; step 19 = the C2 batch (all l = n - 19 sets)
    picks, values, caps = device_greedy_with_checks(
        g, k, [k - 1], n_random=198, seed=3, forced=S + [S[0]])
    assert picks[:19] == S
    cap = caps[0]
    cands = cap["cands"]
    fS = values[18]
    dev_f = fS + np.asarray(cap["G_dev"]) / n  # f(S u {c}) from K3 gains
    # the oracle: explicit sets S u {c} in the reference's fp32 op order
    og = O.Ground(V, np.float32)
    sets = [og.matrix[S + [c]] for c in cands]
    ref = O.evaluate_batch(og, sets, workers=8)
    slack = 2 * _ulp32(g.aux_loss)
    err = np.abs(dev_f - ref)
    assert np.all(err <= 1e-5 * np.maximum(1.0, np.abs(ref)) + slack), \
        err.max()
    # the device's explicit-set kernel (K4) on the same sets
    k4 = pb.evaluate_batch(Evaluator(), g,
                           EvaluationBatch.from_sets([g.matrix[S + [c]]
                                                      for c in cands]))
    assert np.all(np.abs(k4 - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref))
                  + slack)
    # the argmax of the device gains is the argmax of the oracle's values
    # over the checked candidates, up to the binary32 tolerance
    assert ref[0] >= ref.max() - (1e-5 * max(1.0, abs(ref.max())) + slack)


@pytest.mark.parametrize("prec,n,d", [(P32, 6000, 512), (P32, 3000, 1024),
                                      (P64, 8000, 100), (P64, 4000, 512),
                                      (P64, 2500, 1024)])
def test_simt_large_d_teacher_forced(prec, n, d):
    rng = np.random.default_rng(n + d)
    data = rng.standard_normal((n, d)).astype(prec.dtype)
    g = pb.build_ground_set(data, precision=prec)
    k = 4
    res = pb.greedy_maximize(g, k=k)
    gt, vt = _tols(prec, g.aux_loss)
    teacher_forced_trajectory(g, res, gt, vt, label=f"SIMT {prec.name} d={d}")
    # explicit batches (K4 SIMT) against the oracle in the reference order
    sets = [np.sort(rng.choice(n, size=int(rng.integers(1, 60)),
                               replace=False)) for _ in range(24)]
    vals = pb.evaluate_batch(Evaluator(), g,
                             EvaluationBatch.from_sets([g.matrix[i]
                                                        for i in sets]))
    og = O.Ground(g.matrix, prec.dtype)
    ref = O.evaluate_batch(og, [og.matrix[i] for i in sets], workers=8)
    slack = 0.0 if prec is P64 else 2 * _ulp32(g.aux_loss)
    tol = 1e-12 if prec is P64 else 1e-5
    assert np.all(np.abs(vals - ref) <= tol * np.maximum(1.0, np.abs(ref))
                  + slack)
