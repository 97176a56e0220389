"""The half-precision parity contract, in one place.

binary16 / bfloat16 values are compared with the fp64 oracle evaluated on
the IDENTICAL inputs the device holds: the stored (half-rounded) values,
the stored aux distances (binary16 rounds them like the reference,
core.py:303-305) and the device's aux_loss.  What remains is the device's
own arithmetic -- fp32 accumulation in the tensor core, the folded norm
constants (~24 bits) -- plus the final rounding of f to the accumulate
dtype (binary32, core.py:55-60), which is at most ~1 ulp32 of aux_loss:

    |f_dev - f_ref| <= HALF_F_REL * max(1, |f_ref|) + 2 ulp32(aux_loss)
    |G_dev - G_ref| <= HALF_G_REL * max(1, |G_ref|)     (Greedy gains)

HALF_F_REL / HALF_G_REL are about twice the largest errors measured on
B200 over the parity suite (profiles/r02_parity_errors.jsonl).  The
reference's own half bound against binary32 (5e-2,
tests/test_evaluate.py:230-243) is checked separately.
"""

from __future__ import annotations

import numpy as np

import exem_oracle as O  # checker only
from spotcheck import log

# measured maxima (B200, round 2): f 2.1e-6 beyond the slack (K4-TC f16,
# d = 700); G 1.07e-5 (K3-TC f16, d = 1024); split-bf16 binary32 gains
# 1.8e-5 (C4)
HALF_F_REL = 5e-6
HALF_G_REL = 2e-5
SPLIT32_G_REL = 4e-5


def ulp32(x) -> float:
    return float(np.spacing(np.float32(abs(x))))


def oracle_on_device_inputs(g):
    """fp64 oracle ground set holding exactly what the device holds."""
    og = O.Ground(np.asarray(g.matrix, np.float64), np.float64,
                  aux=np.asarray(g.aux, np.float64))
    og.aux_distances = np.asarray(g.aux_distances, np.float64)
    og.aux_loss = float(g.aux_loss)
    return og


def check_half_values(g, got, ref, label=""):
    """``got`` device f values, ``ref`` oracle f on the same inputs."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.maximum(1.0, np.abs(ref))
    slack = 2 * ulp32(g.aux_loss)
    err = np.abs(got - ref)
    rel = np.maximum(err - slack, 0.0) / scale
    log({"check": label, "kind": "half f", "max_abs_err": float(err.max()),
         "max_rel_err_beyond_slack": float(rel.max()),
         "max_rel_err": float((err / scale).max()), "slack": slack})
    assert np.all(err <= HALF_F_REL * scale + slack), (
        label, float(err.max()), float((err / scale).max()))


def check_half_gains(G, ref, label=""):
    G = np.asarray(G, np.float64)
    ref = np.asarray(ref, np.float64)
    ok = np.isfinite(ref)
    scale = np.maximum(1.0, np.abs(ref[ok]))
    err = np.abs(G[ok] - ref[ok])
    log({"check": label, "kind": "half G",
         "max_rel_err": float((err / scale).max())})
    assert np.all(err <= HALF_G_REL * scale), (label,
                                               float((err / scale).max()))
