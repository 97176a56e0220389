"""The command-line front end (cli.py), mirroring the reference's
tests/test_cli.py: same commands, outputs and exit codes.  The known answers
are the reference's (V = {(1), (3)}, e0 = 0: f({3}) = 4.5, f({1,3}) = 5.0,
Greedy k = 2 picks (1, 0); tests/test_cli.py:83-90, :52-62).  Commands that
evaluate need the device and are marked gpu; usage and parsing run on CPU.
"""

import numpy as np
import pytest

from paper_2101_08763_b200 import Precision, read_csv, write_ground_file
from paper_2101_08763_b200.cli import main, read_sets_csv
from paper_2101_08763_b200.errors import ExemError


@pytest.fixture
def data_csv(tmp_path):
    path = tmp_path / "data.csv"
    path.write_text("1.0\n3.0\n")
    return path


def test_info_prints_defaults(capsys):
    assert main(["info"]) == 0
    out = capsys.readouterr().out
    assert "max_threads_per_block = 1024" in out
    assert "shared_memory_bytes   = 49152" in out
    assert "warp_size             = 32" in out


@pytest.mark.parametrize("argv", [
    [],
    ["bench", "--vary", "d", "--values", "1", "--out", "x.csv"],
    ["bench", "--vary", "n", "--values", "8", "--backend", "cuda",
     "--out", "x.csv"],
    ["eval", "--input", "a.csv", "--sets", "s.csv", "--precision", "fp8"],
])
def test_usage_errors_exit_1(argv):
    with pytest.raises(SystemExit) as exc:
        main(argv)
    assert exc.value.code == 1


def test_missing_input_is_exit_1(tmp_path):
    assert main(["cluster", "--input", str(tmp_path / "absent.csv"),
                 "--k", "1", "--out", str(tmp_path / "o.csv")]) == 1


def test_sets_csv_grouping_header_and_errors(tmp_path):
    p = tmp_path / "sets.csv"
    p.write_text("set_id,x0,x1\n7,1,2\n3,0,0\n7,3,4\n\n3,5,6\n")
    sets = read_sets_csv(p)
    assert [s.tolist() for s in sets] == [[[1, 2], [3, 4]], [[0, 0], [5, 6]]]
    p.write_text("0,3.0\nbad,row,here\n")
    with pytest.raises(ExemError, match="malformed row 2"):
        read_sets_csv(p)
    p.write_text("set_id,x0\n")
    with pytest.raises(ExemError, match="no sets"):
        read_sets_csv(p)


@pytest.mark.gpu
def test_malformed_sets_is_exit_1(data_csv, tmp_path):
    sets = tmp_path / "sets.csv"
    sets.write_text("0,3.0\nbad,row,here\n")
    assert main(["eval", "--input", str(data_csv), "--sets", str(sets)]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp32", "bf16"])
def test_eval_values_printed(data_csv, tmp_path, capsys, prec):
    sets = tmp_path / "sets.csv"
    sets.write_text("set_id,x0\n0,3.0\n1,1.0\n1,3.0\n")
    assert main(["eval", "--input", str(data_csv), "--sets", str(sets),
                 "--precision", prec]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert [float(v) for v in lines] == [4.5, 5.0]


@pytest.mark.gpu
def test_cluster_selects_exemplars(data_csv, tmp_path, capsys):
    out, labels = tmp_path / "exemplars.csv", tmp_path / "labels.csv"
    assert main(["cluster", "--input", str(data_csv), "--k", "2",
                 "--precision", "fp64", "--out", str(out),
                 "--labels", str(labels)]) == 0
    rows = [line.split(",") for line in out.read_text().splitlines()]
    assert [int(r[0]) for r in rows] == [1, 0]
    assert [float(r[1]) for r in rows] == [3.0, 1.0]
    assert labels.read_text().splitlines() == ["1", "0"]
    assert "selected 2 exemplars (value 5, 3 evaluations)" in \
        capsys.readouterr().out


@pytest.mark.gpu
def test_cluster_exem_input_and_streamed(tmp_path, capsys):
    rng = np.random.default_rng(3)
    V = rng.standard_normal((12_000, 24))
    path = tmp_path / "data.exem"
    write_ground_file(path, V, Precision.binary64)
    outs = []
    from paper_2101_08763_b200.streaming import resident_bytes

    budget = int(0.9 * resident_bytes(12_000, 24, Precision.binary64))
    for extra in ([], ["--device-budget", str(budget)]):
        out = tmp_path / f"ex{len(outs)}.csv"
        assert main(["cluster", "--input", str(path), "--k", "4",
                     "--precision", "fp64", "--out", str(out), *extra]) == 0
        outs.append(out.read_text())
    assert outs[0] == outs[1]  # streamed Greedy is bit-identical
    assert len(outs[0].splitlines()) == 4


@pytest.mark.gpu
def test_budget_too_small_is_exit_2(data_csv, tmp_path):
    assert main(["cluster", "--input", str(data_csv), "--k", "1",
                 "--memory-budget", "1", "--out", str(tmp_path / "o.csv")]) == 2


@pytest.mark.gpu
def test_bench_writes_schema_csv(tmp_path, capsys):
    out = tmp_path / "bench.csv"
    assert main(["bench", "--vary", "n", "--values", "64,128", "--l", "4",
                 "--k", "2", "--d", "3", "--backend", "tiled", "--reps", "1",
                 "--out", str(out)]) == 0
    records = read_csv(out)
    assert [r.n for r in records] == [64, 128]
    assert all(r.backend == "tiled" for r in records)
    assert all(r.runtime_seconds > 0 for r in records)
