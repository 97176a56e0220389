"""Low-memory regime (streaming.py, north-star item c): a ground set over its
device budget stays in host memory and streams through a two-slot device
ring in split-aligned slices.  Everything computed on a streamed ground set
must be BIT-IDENTICAL to the resident computation (same per-split / per-block
partials, same fixed-order reductions), and row-sharded batch evaluation
(distributed.py) must reproduce the single-GPU sums exactly.
"""

import numpy as np
import pytest

import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import EvaluationBatch, Evaluator, Precision
from paper_2101_08763_b200 import _native as N
from paper_2101_08763_b200 import streaming as S
from paper_2101_08763_b200.distributed import shard_rows

pytestmark = pytest.mark.gpu

P16, BF16, P32, P64 = (Precision.binary16, Precision.bfloat16,
                       Precision.binary32, Precision.binary64)


def _budget(n, d, prec, l, k_max, splits_per_slice=3):
    lib = N.lib()
    sp = int(lib.split_points(n))
    fixed = S.batch_device_bytes(d, k_max, l, prec, -(-n // sp)) + S._margin(n)
    slot = S.layout_bytes(splits_per_slice * sp, d, prec, with_src=True)
    b = fixed + 2 * slot + 4096
    assert b < S.resident_bytes(n, d, prec)
    plan = S.plan_slices(n, d, prec, b - fixed, sp)
    assert len(plan.slices) > 1
    return b


@pytest.mark.parametrize("prec", [P32, P64, BF16, P16])
def test_streamed_matches_resident_bit_exact(prec):
    rng = np.random.default_rng(21)
    n, d, l = 20_000, 37, 60
    data = rng.standard_normal((n, d)) * (0.5 if prec is P16 else 1.0)
    idx = [np.sort(rng.choice(n, size=int(rng.integers(1, 13)), replace=False))
           for _ in range(l)]
    budget = _budget(n, d, prec, l, 12)
    gr = pb.build_ground_set(data, precision=prec)
    gs = pb.build_ground_set(data, precision=prec, device_budget=budget)
    assert gs.streamed and not gr.streamed
    assert gs.aux_loss == gr.aux_loss
    assert np.array_equal(gs.aux_distances, gr.aux_distances)
    br = EvaluationBatch.from_sets([gr.matrix[i] for i in idx])
    vr = pb.evaluate_batch(Evaluator(), gr, br)
    vs = pb.evaluate_batch(Evaluator(), gs, br)
    assert np.array_equal(vr, vs)
    mu = pb.estimate_set_memory(n, br.k_max, d, prec)
    assert np.array_equal(pb.evaluate_chunked(Evaluator(), gs, br, budget=mu * 17), vr)
    S0 = gr.matrix[idx[3]]
    assert pb.evaluate_single(gs, S0) == pb.evaluate_single(gr, S0)
    assert np.array_equal(pb.min_distances(gs, S0), pb.min_distances(gr, S0))
    assert np.array_equal(pb.assign_clusters(gs, S0), pb.assign_clusters(gr, S0))


def test_sharded_batch_partials_match_single_gpu():
    """Each simulated rank streams its shard into its own partial rows; the
    sum of the rank matrices (what all-reduce computes) reduced in fixed
    order equals the resident single-GPU sums bit for bit."""
    import torch

    rng = np.random.default_rng(5)
    n, d, l = 30_000, 20, 40
    data = rng.standard_normal((n, d))
    g = pb.build_ground_set(data, precision=BF16)
    sets = [g.matrix[np.sort(rng.choice(n, size=int(rng.integers(1, 30)),
                                        replace=False))] for _ in range(l)]
    batch = EvaluationBatch.from_sets(sets)
    ref = pb.evaluate_batch(Evaluator(), g, batch)
    packed = pb.pack_batch(batch, g.precision)
    lib = N.lib()
    sp = int(lib.split_points(n))
    splits = -(-n // sp)
    for world in (2, 3, 4):
        total = torch.zeros((splits, l), dtype=torch.float64, device="cuda")
        for rank in range(world):
            part = torch.zeros_like(total)
            r0, r1 = shard_rows(n, world, rank, sp)
            if r1 > r0:
                S.stream_packed_sums(g, packed.values, d, packed.k_max, l,
                                     packed.cardinalities, rows=(r0, r1),
                                     partial=part, budget=1 << 30)
            assert torch.all(part[: r0 // sp] == 0)
            total += part
        sums = torch.empty(l, dtype=torch.float64, device="cuda")
        lib.reduce_partials(N.ptr(total), splits, l, 1.0, N.ptr(sums),
                            N.stream_handle())
        acc = g.precision.accumulate_dtype
        vals = acc.type(g.aux_loss) - sums.cpu().numpy().astype(acc) / acc.type(n)
        assert np.array_equal(vals, ref), world


def test_streamed_budget_errors():
    rng = np.random.default_rng(1)
    data = rng.standard_normal((5000, 8))
    with pytest.raises(pb.OutOfMemoryError):
        pb.build_ground_set(data, precision=P32, device_budget=2 << 20 >> 4)
    g = pb.build_ground_set(data, precision=P32,
                            device_budget=S.resident_bytes(5000, 8, P32) - 1)
    assert g.streamed
    with pytest.raises(pb.OutOfMemoryError):
        g.on_device()


@pytest.mark.parametrize("prec", [BF16, P32, P64])
def test_streamed_greedy_matches_resident(prec):
    """Greedy over a streamed ground set (candidate chunks x point slices,
    m kept on device) picks the same exemplars with bit-identical values."""
    rng = np.random.default_rng(8)
    n, d, k = 12_000, 24, 4
    data = rng.standard_normal((n, d))
    gr = pb.build_ground_set(data, precision=prec)
    ref = pb.greedy_maximize(gr, k=k)
    lib = N.lib()
    sp = int(lib.split_points(n))
    budget = int(0.9 * S.resident_bytes(n, d, prec))
    gs = pb.build_ground_set(data, precision=prec, device_budget=budget)
    assert gs.streamed
    res = pb.greedy_maximize(gs, k=k)
    assert res.exemplar_indices == ref.exemplar_indices
    assert res.values == ref.values
    assert res.evaluations == ref.evaluations
    assert sp > 0


@pytest.mark.parametrize("prec", [P32, P64, BF16, P16])
def test_row_major_input_matches_column_major(prec):
    """A large C-order input is uploaded untransposed and K1's row-major
    variant (exem_ground_prepare_rows) transposes on the device (resident;
    streamed ground sets transpose on the host); GroundSet.matrix is
    column-major either way, and everything derived from it -- aux
    distances, L({e0}), batch sums, Greedy -- is bit-identical to the
    column-major (reference layout) path, resident and streamed."""
    rng = np.random.default_rng(5)
    n, d, l, k = 30_003, 45, 40, 3
    assert n * d >= 1 << 20  # the device-transpose size class
    data = rng.standard_normal((n, d)) * (0.5 if prec is P16 else 1.0)
    rows = np.ascontiguousarray(data.astype(prec.dtype))
    cols = np.asfortranarray(rows)
    idx = [np.sort(rng.choice(n, size=int(rng.integers(1, 11)), replace=False))
           for _ in range(l)]
    budget = _budget(n, d, prec, l, 10)
    ref = None
    for src in (cols, rows):
        for kw in ({}, {"device_budget": budget}):
            g = pb.build_ground_set(src, precision=prec, **kw)
            assert g.matrix.flags.f_contiguous
            assert np.array_equal(g.matrix, rows)
            b = EvaluationBatch.from_sets([g.matrix[i] for i in idx])
            got = (g.aux_loss, g.aux_distances.copy(),
                   pb.evaluate_batch(Evaluator(), g, b),
                   pb.greedy_maximize(g, k=k))
            if ref is None:
                ref = got
                continue
            assert got[0] == ref[0]
            assert np.array_equal(got[1], ref[1])
            assert np.array_equal(got[2], ref[2])
            assert got[3].exemplar_indices == ref[3].exemplar_indices
            assert got[3].values == ref[3].values


@pytest.mark.parametrize("prec", [P32, BF16])
@pytest.mark.parametrize("streamed", [False, True])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_detected_on_device(prec, streamed, bad):
    """binary32 storage of a float32 matrix and bfloat16 storage skip the
    host scan: K1 turns a non-finite stored value into a NaN aux sum and
    build_ground_set raises the reference's InvalidDataError (core.py:282-283)
    -- wherever the value sits (first / last point, a late streamed slice)."""
    rng = np.random.default_rng(2)
    n, d = 20_003, 37
    budget = _budget(n, d, prec, 4, 4) if streamed else None
    for i, k in ((0, 0), (n - 1, d - 1), (15_000, 11)):
        V = rng.standard_normal((n, d)).astype(np.float32)
        V[i, k] = bad
        with pytest.raises(pb.InvalidDataError):
            pb.build_ground_set(V, precision=prec, device_budget=budget)
    # finite data passes, and float64 input overflowing binary32 keeps the
    # reference semantics (validated on the host, stored as inf, accepted)
    V = rng.standard_normal((n, d)).astype(np.float32)
    g = pb.build_ground_set(V, precision=prec, device_budget=budget)
    assert np.isfinite(g.aux_loss)
    if prec is P32:
        W = V.astype(np.float64)
        W[5, 3] = 1e39
        g = pb.build_ground_set(W, precision=prec)
        assert np.isinf(g.matrix[5, 3]) and np.isinf(g.aux_loss)
