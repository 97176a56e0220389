"""Host-side logic and the C-ABI boundary (CPU only, no kernel launches).

Mirrors the reference's host/unit tests (pkg/tests/test_core.py,
test_evaluate.py:170-197, test_acceptance.py:113-175) for the parts of the
API that are pure host arithmetic, and checks that libexem_b200.so loads and
exports every symbol include/exem_b200.h declares.
"""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import (
    DeviceLimits,
    DimensionMismatchError,
    EmptyEvaluationSetError,
    EmptyGroundSetError,
    EvaluationBatch,
    Evaluator,
    InvalidDataError,
    OutOfMemoryError,
    Precision,
    SharedMemoryOverflowError,
    compute_kernel_config,
    count_transactions,
    estimate_set_memory,
    pack_batch,
    packed_address,
    plan_chunks,
)

ROOT = Path(__file__).resolve().parents[1]


# ------------------------------------------------------------------ C-ABI
def _header_symbols():
    text = (ROOT / "include" / "exem_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(exem_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(native_lib):
    import ctypes

    handle = ctypes.CDLL(str(ROOT / "paper_2101_08763_b200" / "libexem_b200.so"))
    syms = _header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(handle, s)]
    assert not missing, missing


def test_binding_covers_header(native_lib):
    from paper_2101_08763_b200 import _native

    assert sorted(_native.EXPORTED) == _header_symbols()


def test_header_constants_match_binding():
    from paper_2101_08763_b200 import _native

    text = (ROOT / "include" / "exem_b200.h").read_text()
    consts = dict(re.findall(r"#define (EXEM_[A-Z0-9_]+) (0x[0-9a-fA-F]+|\d+)",
                             text))
    val = {k: int(v, 0) for k, v in consts.items()}
    assert val["EXEM_VT_STORAGE"] == _native.VT_STORAGE
    assert (val["EXEM_F16"], val["EXEM_BF16"], val["EXEM_F32"],
            val["EXEM_F64"]) == (_native.F16, _native.BF16, _native.F32,
                                 _native.F64)
    # the flag never collides with a tag
    assert all(t & _native.VT_STORAGE == 0 for t in range(4))


def test_storage_ok_predicate(native_lib):
    """exem_set_min_storage_ok is pure host arithmetic (no device work)."""
    from paper_2101_08763_b200 import _native as N

    ok = native_lib.set_min_storage_ok
    assert ok(N.F32 | N.VT_STORAGE, 100, 10, 0) == 0
    assert ok(N.F32, 100, 10, 0) == 0
    assert ok(N.BF16 | N.VT_STORAGE, 100, 0, 0) == 0


def test_layout_helpers(native_lib):
    lib = native_lib
    from paper_2101_08763_b200._native import ABI_VERSION
    assert lib.abi_version() == ABI_VERSION == 4
    assert lib.pad_points(1) == 256 and lib.pad_points(257) == 512
    assert lib.pad_dims(100) == 104 and lib.pad_dims(2) == 8
    assert lib.tc_kp(100) == 128 and lib.tc_kp(2) == 64 and lib.tc_kp(1024) == 1088
    assert lib.tc_rows(1_000_000) % 256 == 0
    for n in (1, 10, 1000, 10_000, 100_000, 1_000_000, 50_000_000):
        sp = lib.split_points(n)
        assert sp % 256 == 0 and 1024 <= sp <= 32768
        assert lib.num_splits(n) == -(-n // sp)
    assert lib.reduce_scratch(10) >= 2 * 296


def test_status_mapping():
    from paper_2101_08763_b200 import _native as N

    with pytest.raises(OutOfMemoryError):
        N.raise_status(N.ERR_OOM, "x")
    with pytest.raises(InvalidDataError):
        N.raise_status(N.ERR_DATA, "x")
    with pytest.raises(DimensionMismatchError):
        N.raise_status(N.ERR_ARG, "x")
    with pytest.raises(pb.ExemError):
        N.raise_status(N.ERR_CUDA, "x")


def test_bad_args_fail_without_gpu(native_lib):
    """Argument validation in the C-ABI runs before any device work."""
    from paper_2101_08763_b200 import _native as N

    with pytest.raises(DimensionMismatchError):
        native_lib.ground_prepare(N.F32, None, 0, 3, None, None, 256, None,
                                  None, None, None, 0, None)
    with pytest.raises(DimensionMismatchError):
        native_lib.greedy_gains_simt(N.F32, None, 256, None, 10, None, 256,
                                     None, None, 10, 3, 100, None, 1, None)


def test_missing_library_fails_loudly(tmp_path):
    from paper_2101_08763_b200 import _native

    with pytest.raises(pb.ExemError, match="no CPU"):
        _native.load_library(tmp_path / "nope.so")


# ------------------------------------------------------------------ core
def test_precision_aliases():
    assert Precision.from_name("FP32") is Precision.binary32
    assert Precision.from_name(" half ") is Precision.binary16
    assert Precision.from_name("bf16") is Precision.bfloat16
    assert Precision.from_name("double") is Precision.binary64
    with pytest.raises(ValueError):
        Precision.from_name("fp8")
    assert Precision.binary16.accumulate_dtype == np.float32
    assert Precision.bfloat16.accumulate_dtype == np.float32
    assert Precision.binary64.accumulate_dtype == np.float64
    assert [p.bytes_per_value for p in Precision] == [2, 2, 4, 8]
    assert Precision.bfloat16.dtype.itemsize == 2
    assert Precision.binary32.max_finite == float(np.finfo(np.float32).max)


def test_device_limits_validation():
    with pytest.raises(ValueError):
        DeviceLimits(max_threads_per_block=0)
    with pytest.raises(ValueError):
        DeviceLimits(max_threads_per_block=100, warp_size=32)


@pytest.mark.parametrize("obs,err", [
    ([], EmptyGroundSetError),
    ([[1.0, 2.0], [3.0]], DimensionMismatchError),
    ([[1.0, np.nan]], InvalidDataError),
    ([[1.0, np.inf]], InvalidDataError),
    (np.zeros((2, 2, 2)), DimensionMismatchError),
])
def test_build_ground_set_validation_precedes_device(obs, err):
    with pytest.raises(err):
        pb.build_ground_set(obs)


def test_build_ground_set_aux_validation():
    with pytest.raises(DimensionMismatchError):
        pb.build_ground_set([[1.0, 2.0]], aux=[1.0])
    with pytest.raises(ValueError):
        pb.build_ground_set([[1.0]], aux="one")
    with pytest.raises(InvalidDataError):
        pb.build_ground_set([[1.0]], aux=[np.nan])


def test_evaluation_batch():
    b = EvaluationBatch.from_sets([[[1.0, 2.0]], [[1.0, 2.0], [3.0, 4.0]]])
    assert (b.l, b.d, b.k_max, b.cardinalities) == (2, 2, 2, (1, 2))
    with pytest.raises(EmptyEvaluationSetError):
        EvaluationBatch.from_sets([])
    with pytest.raises(EmptyEvaluationSetError):
        EvaluationBatch.from_sets([np.empty((0, 2))])
    with pytest.raises(DimensionMismatchError):
        EvaluationBatch.from_sets([[[1.0]], [[1.0, 2.0]]])


def test_packed_address_bijection():
    l, k_max, d = 3, 4, 2
    seen = {packed_address(j, e, dim, l, k_max, d)
            for j in range(l) for e in range(k_max) for dim in range(d)}
    assert seen == set(range(l * k_max * d))
    assert packed_address(2, 1, 1, 3, 4) == 1 * 12 + 1 * 3 + 2
    with pytest.raises(IndexError):
        packed_address(3, 0, 0, 3, 4)
    with pytest.raises(IndexError):
        packed_address(0, 0, 2, 3, 4, d=2)


def test_pack_batch_round_robin():
    b = EvaluationBatch.from_sets([[[10.0], [11.0]], [[20.0], [21.0]]])
    p = pack_batch(b, Precision.binary64)
    assert p.values.tolist() == [10.0, 20.0, 11.0, 21.0]
    b2 = EvaluationBatch.from_sets([[[1.0, 2.0]], [[3.0, 4.0], [5.0, 6.0]]])
    p2 = pack_batch(b2, Precision.binary32)
    assert p2.blank_slots == 2
    assert np.array_equal(p2.set_elements(1), np.array([[3, 4], [5, 6]], np.float32))
    assert pack_batch(b2, Precision.binary16).values.nbytes * 2 == p2.values.nbytes


def test_kernel_config_table():
    # tests/test_acceptance.py:147-158 worked examples
    cases = [((50000, 5000, 400), (1, 1024, 1), (50000, 5, 1)),
             ((1000, 1, 400), (122, 1, 1), (9, 1, 1)),
             ((64, 2048, 4), (1, 1024, 1), (64, 2, 1))]
    for (n, l, gamma), block, grid in cases:
        cfg = compute_kernel_config(n, l, gamma)
        assert (cfg.block, cfg.grid) == (block, grid)
    with pytest.raises(SharedMemoryOverflowError):
        compute_kernel_config(10, 10, 10**6)
    with pytest.raises(ValueError):
        compute_kernel_config(0, 1, 1)


def test_coalescing_model():
    assert count_transactions([(0, 8), (8, 8), (16, 8), (24, 8)]) == 1
    assert count_transactions([(0, 8), (32, 8), (64, 8), (96, 8)]) == 4
    l, k_max, d, bpv, e, dim = 32, 4, 2, 4, 1, 1
    packed = count_transactions(
        [(packed_address(j, e, dim, l, k_max) * bpv, bpv) for j in range(32)])
    per_set = count_transactions(
        [((j * k_max * d + e * d + dim) * bpv, bpv) for j in range(32)])
    assert (packed, per_set) == (4, 32)
    with pytest.raises(ValueError):
        count_transactions([(0, 4)] * 33)


def test_memory_estimate_and_plan(hand):
    assert [estimate_set_memory(50000, 10, 100, Precision.binary32),
            estimate_set_memory(1, 1, 1, Precision.binary16)] == hand["mu_examples"]
    plan = plan_chunks(1000, 300, 10)
    assert [plan.chunk_size, plan.chunk_count] == hand["plan_example"]
    assert (plan_chunks(10**9, 300, 10).chunk_size, plan_chunks(10**9, 300, 10).chunk_count) == (10, 1)
    with pytest.raises(OutOfMemoryError):
        plan_chunks(100, 300, 10)
    with pytest.raises(ValueError):
        estimate_set_memory(0, 1, 1, Precision.binary32)
    # attainable chunk counts for l=10 (test_acceptance.py:125-129)
    assert {-(-10 // s) for s in range(1, 11)} == {1, 2, 3, 4, 5, 10}


def test_evaluator_validation():
    with pytest.raises(ValueError):
        Evaluator(backend="gpu")
    with pytest.raises(ValueError):
        Evaluator(worker_count=0)
    for name in pb.BACKENDS:
        Evaluator(backend=name)


def test_custom_dissimilarity_rejected_on_evaluation_path():
    from paper_2101_08763_b200.objective import require_device_dissimilarity

    manhattan = pb.Dissimilarity("manhattan",
                                 pairwise=lambda x, y: float(np.abs(x - y).sum()))
    with pytest.raises(pb.ExemError, match="no device kernel"):
        require_device_dissimilarity(manhattan)
    require_device_dissimilarity(pb.SQUARED_EUCLIDEAN)
    # the user's own pairwise function still works as a host utility
    assert manhattan.distances(np.array([[0.0], [3.0]]), np.array([[1.0]])).tolist() == [[1.0], [2.0]]


def test_squared_euclidean_pairwise():
    assert pb.squared_euclidean([1.0, 2.0], [3.0, 4.0]) == 8.0
    with pytest.raises(DimensionMismatchError):
        pb.squared_euclidean([1.0], [1.0, 2.0])


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2101_08763_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "exem_oracle" not in text and "import oracle" not in text, py
        assert "from oracle" not in text, py


def test_stream_plan_is_split_aligned(native_lib):
    """Low-memory regime planning (streaming.py): slices are whole
    partial-sum splits covering [0, n) in order, sized so two ring slots fit
    the budget; below one split per slot -> OutOfMemoryError."""
    from paper_2101_08763_b200 import streaming as S

    P = pb.Precision
    for n, d, prec in ((20_000, 37, P.binary32), (1_000_000, 100, P.bfloat16),
                       (50_000_000, 256, P.bfloat16), (5000, 8, P.binary64)):
        sp = int(native_lib.split_points(n))
        one = S.layout_bytes(sp, d, prec, with_src=True)
        for budget in (2 * one, 5 * one + 17, 40 * one):
            plan = S.plan_slices(n, d, prec, budget, sp)
            assert plan.slices[0][0] == 0 and plan.slices[-1][1] == n
            for (a0, a1), (b0, b1) in zip(plan.slices, plan.slices[1:]):
                assert a1 == b0 and a1 % sp == 0
            assert 2 * plan.slot_bytes <= budget
            assert plan.rows_per_slice % sp == 0 or plan.rows_per_slice == n
        with pytest.raises(pb.OutOfMemoryError):
            S.plan_slices(n, d, prec, 2 * one - 1, sp)
        assert S.resident_bytes(n, d, prec) > S.layout_bytes(n, d, prec)
        assert S.fits_resident(n, d, prec, None)
        assert not S.fits_resident(n, d, prec, S.resident_bytes(n, d, prec) - 1)


def test_resident_bytes_count_two_byte_vt(native_lib):
    """Resident half ground sets keep vt at the 2-byte storage type
    (EXEM_VT_STORAGE); streamed slots keep the binary32 widening."""
    from paper_2101_08763_b200 import streaming as S

    P = pb.Precision
    n, d = 1_000_000, 100
    ld = int(native_lib.pad_points(n))
    d_pad = int(native_lib.pad_dims(d))
    for prec in (P.bfloat16, P.binary16):
        wide = S.layout_bytes(n, d, prec)
        narrow = S.layout_bytes(n, d, prec, vt_storage=True)
        assert wide - narrow == d_pad * ld * 2
    for prec in (P.binary32, P.binary64):  # no storage flag for wide types
        assert S.layout_bytes(n, d, prec) == \
            S.layout_bytes(n, d, prec, vt_storage=True)
    # C4 bf16: vt 208 MB + two half operands + norms/aux + scratch < 1 GB
    assert S.resident_bytes(n, d, P.bfloat16) < 1.0e9


def test_tc_set_geometry(native_lib):
    """K4-TC set tiles: w = k_max slots per set (column-interleaved), as many
    sets as fit 256 TMEM columns (<= 16; <= 32 in the small-set kernel,
    k_max <= 10),
    MMA N = round_up(spt*w, 16)."""
    import ctypes

    geo = native_lib.raw("exem_tc_set_geometry")
    for k in (1, 7, 8, 9, 50, 51, 128, 129, 256):
        spt, w, nc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        assert geo(k, ctypes.byref(spt), ctypes.byref(w), ctypes.byref(nc)) == 0
        assert w.value == k
        assert spt.value == (min(32, 256 // k) if k <= 10 else min(16, 256 // k))
        assert nc.value == -(-spt.value * k // 16) * 16 <= 256
        rows = native_lib.tc_set_rows(1000, k)
        assert rows == -(-1000 // spt.value) * nc.value
    spt, w, nc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert geo(257, ctypes.byref(spt), ctypes.byref(w), ctypes.byref(nc)) == 5


def test_groundset_fields_match_reference():
    """Same dataclass fields as the reference's GroundSet (core.py:127-143);
    device state lives outside the fields."""
    import dataclasses

    import paper_2101_08763_b200 as pb

    names = [f.name for f in dataclasses.fields(pb.GroundSet)]
    assert names == ["matrix", "precision", "aux", "aux_distances", "aux_loss"]


def test_checked_picks_sentinel():
    from paper_2101_08763_b200.errors import InvalidDataError
    from paper_2101_08763_b200.optimize import checked_picks

    assert list(checked_picks(np.array([4, 2, 9]), 2)) == [4, 2]
    with pytest.raises(InvalidDataError):
        checked_picks(np.array([4, -1, 9]), 3)
