"""Dataset files (paper_2101_08763_b200/io.py), mirroring the reference's
tests/test_io.py: the .exem container round trip and header layout
(pkg/tests/test_io.py:16-60), its validation errors and CSV ingestion --
plus the B200 loader's properties: the payload is memory-mapped, not
copied, and (GPU) loads to the same ground set as build_ground_set,
resident or streamed."""

import numpy as np
import pytest

import paper_2101_08763_b200 as pb
from paper_2101_08763_b200 import (
    InvalidDataError,
    Precision,
    load_ground_set,
    read_csv_observations,
    read_ground_file,
    write_ground_file,
)


@pytest.mark.parametrize("precision", list(Precision))
def test_round_trip(tmp_path, precision):
    rng = np.random.default_rng(7)
    matrix = rng.random((13, 4)).astype(precision.dtype)
    path = tmp_path / "data.exem"
    write_ground_file(path, matrix, precision)
    back, stored = read_ground_file(path)
    assert stored is precision
    assert np.array_equal(np.asarray(back), matrix)
    assert isinstance(back, np.memmap) and not back.flags.writeable
    assert back.flags.f_contiguous


def test_header_layout_matches_reference(tmp_path):
    path = tmp_path / "data.exem"
    write_ground_file(path, [[1.0, 2.0]], Precision.binary32)
    raw = path.read_bytes()
    assert raw[:4] == b"EXEM" and raw[4] == 1 and raw[5] == 1
    assert len(raw) == 14 + 2 * 4
    # column-major payload: the [d][n] buffer kernel K1 consumes
    write_ground_file(path, [[1.0, 2.0], [3.0, 4.0]], Precision.binary64)
    vals = np.frombuffer(path.read_bytes()[14:], dtype=np.float64)
    assert vals.tolist() == [1.0, 3.0, 2.0, 4.0]


@pytest.mark.parametrize("patch,where", [(b"NOPE", 0), (bytes([9]), 4), (bytes([7]), 5)])
def test_bad_header(tmp_path, patch, where):
    good = tmp_path / "good.exem"
    write_ground_file(good, [[1.0]], Precision.binary32)
    raw = bytearray(good.read_bytes())
    raw[where:where + len(patch)] = patch
    bad = tmp_path / "bad.exem"
    bad.write_bytes(bytes(raw))
    with pytest.raises(InvalidDataError):
        read_ground_file(bad)


def test_truncated_and_size_mismatch(tmp_path):
    p = tmp_path / "t.exem"
    p.write_bytes(b"EXE")
    with pytest.raises(InvalidDataError):
        read_ground_file(p)
    write_ground_file(p, [[1.0, 2.0]], Precision.binary32)
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(InvalidDataError):
        read_ground_file(p)


def test_csv(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text("a,b\n1,2\n\n3, 4\n")
    assert read_csv_observations(p).tolist() == [[1.0, 2.0], [3.0, 4.0]]
    p.write_text("1,2\nx,4\n")
    with pytest.raises(InvalidDataError):
        read_csv_observations(p)
    p.write_text("a,b\n")
    with pytest.raises(InvalidDataError):
        read_csv_observations(p)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [Precision.binary32, Precision.bfloat16])
def test_load_ground_set_to_device(tmp_path, precision):
    from paper_2101_08763_b200 import streaming as S

    rng = np.random.default_rng(3)
    data = rng.standard_normal((9000, 12))
    path = tmp_path / "v.exem"
    write_ground_file(path, data, precision)
    ref = pb.build_ground_set(data, precision=precision)
    g = load_ground_set(path)
    assert g.precision is precision
    assert g.aux_loss == ref.aux_loss
    assert np.array_equal(g.aux_distances, ref.aux_distances)
    assert pb.greedy_maximize(g, k=3) == pb.greedy_maximize(ref, k=3)
    gs = load_ground_set(path, device_budget=S.resident_bytes(9000, 12, precision) - 1)
    assert gs.streamed and gs.aux_loss == ref.aux_loss
    csv = tmp_path / "v.csv"
    csv.write_text("\n".join(",".join(repr(float(x)) for x in r) for r in data[:50]))
    gc = load_ground_set(csv)
    assert gc.precision is Precision.binary32 and gc.n == 50
