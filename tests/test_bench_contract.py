"""bench.py launched the way the round-end driver launches it.

* ``--impl reference`` under ``torch.distributed.run`` with two processes
  (CPU only): rank 0 alone prints ONE JSON line with the contract's keys,
  the other rank exits 0 without work.
* the GPU arm at N = 2 (``-m gpu``): both ranks share cuda:0 over gloo
  (EXEM_BENCH_SHARE_GPU=1 -- the box has one GPU), the line reports
  n_gpus = 2, the communicator it ran on, and the same picks as N = 1.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data",
        "config", "e2e"}


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(nproc, args, env=None, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={_port()}", "bench.py", *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True,
                          timeout=timeout, env=dict(os.environ, **(env or {})))


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_under_torchrun_prints_one_line():
    p = _torchrun(2, ["--impl", "reference", "--gpus", "2", "--points",
                      "20000", "--steps", "2", "--warmup", "3",
                      "--cpu-seconds", "2"])
    assert p.returncode == 0, p.stderr[-3000:]
    lines = _lines(p.stdout)
    assert len(lines) == 1, p.stdout[-2000:]
    line = lines[0]
    assert KEYS <= set(line)
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["value"] > 0


@pytest.mark.gpu
def test_gpu_arm_two_ranks_sharing_one_gpu():
    args = ["--points", "40000", "--dim", "32", "--steps", "3", "--warmup",
            "3", "--no-cpu", "--no-sub"]
    one = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-3000:]
    ref = _lines(one.stdout)[-1]
    p = _torchrun(2, ["--gpus", "2", *args],
                  env={"EXEM_BENCH_SHARE_GPU": "1"})
    assert p.returncode == 0, p.stderr[-3000:]
    lines = _lines(p.stdout)
    assert len(lines) == 1, p.stdout[-2000:]
    line = lines[0]
    assert KEYS <= set(line) and line["n_gpus"] == 2
    assert line["communicator"]["nranks"] == 2
    assert line["picks_head"] == ref["picks_head"]
    assert line["e2e"]["picks_match_device_run"] is True
    assert line["gpu_launches"] > 0
