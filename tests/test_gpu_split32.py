"""Binary32 Greedy gains on tensor cores (opt-in ``Evaluator(tensor_fp32=
True)``): every fp32 coordinate split into three bf16 pieces laid out along
K (exem_tc_pack_split), so the unchanged K3-TC kernel computes the gains at
binary32 accuracy.  Checked like the CUDA-core binary32 path: gains against
fp64 truth on the same fp32 inputs, and the BASELINE config-1 Greedy
trajectory against the reference's own golden picks/values."""

import numpy as np
import pytest

import exem_oracle as O
import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import Evaluator, Precision
from paper_2101_08763_b200.optimize import GreedyRun

pytestmark = pytest.mark.gpu
P32 = Precision.binary32


@pytest.mark.parametrize("n,d", [(5000, 100), (3000, 2), (2000, 37), (1500, 128)])
def test_split32_gains_vs_fp64(n, d):
    rng = np.random.default_rng(n + d)
    data = rng.standard_normal((n, d)).astype(np.float32)
    g = pb.build_ground_set(data, precision=P32)
    x = g.matrix.astype(np.float64)
    dg = g.on_device()
    for split in (True, False):
        run = GreedyRun(dg, k_cap=2, split32=split)
        run.start()
        run.compute_gains()
        G = run.gains.cpu().numpy()
        ref = O.gains_m(x, g.aux_distances.astype(np.float64), x)
        scale = max(1.0, np.abs(ref).max())
        err = np.max(np.abs(G - ref)) / scale
        assert err <= 1e-5, (split, err)
        if split:
            err_split = err
        else:
            err_simt = err
        # one step later: K2 m-update, then the -h columns refreshed
        run.select(0)
        run.update(0)
        c = int(run.sel_idx[0].item())
        run.compute_gains()
        m2 = np.minimum(g.aux_distances.astype(np.float64),
                        ((x - x[c]) ** 2).sum(1))
        ref2 = O.gains_m(x, m2, x)
        assert np.max(np.abs(run.gains.cpu().numpy() - ref2)) <= 1e-5 * scale
    # both within the binary32 contract; the split path's gains carry the
    # tensor core's fp32 accumulation over K' = 6d + 6 terms (measured ~10x
    # the CUDA-core path's error, still well inside 1e-5)
    assert max(err_split, err_simt) <= 1e-5


def test_split32_c1_greedy_matches_reference(golden):
    V = np.random.default_rng(1234).standard_normal((10000, 100), dtype=np.float32)
    g = pb.build_ground_set(V, precision=P32)
    res = pb.greedy_maximize(g, k=10, evaluator=Evaluator(tensor_fp32=True))
    assert list(res.exemplar_indices) == golden["c1_f32_picks"].tolist()
    ref = golden["c1_f32_values"]
    slack = 2 * float(np.spacing(np.float32(g.aux_loss)))
    assert np.all(np.abs(np.array(res.values) - ref) <= 1e-5 * np.maximum(1, np.abs(ref)) + slack)


def test_split32_falls_back_beyond_128_dims():
    g = pb.build_ground_set(np.random.default_rng(1).standard_normal((600, 129)),
                            precision=P32)
    assert not GreedyRun(g.on_device(), split32=True).split32
    assert GreedyRun(pb.build_ground_set(np.ones((300, 4)), precision=P32)
                     .on_device(), split32=True).split32
