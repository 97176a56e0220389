"""The Greedy step loop as one CUDA graph (optimize.capture_steps,
SURVEY.md 8(e) "the k-step loop can be a CUDA graph").

A replayed graph must give exactly the eager run's picks and values: the
same kernels with the same arguments run in the same stream order.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2101_08763_b200 as pb

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("prec", [pb.Precision.bfloat16, pb.Precision.binary32,
                                  pb.Precision.binary64])
@pytest.mark.parametrize("budget", [None, 600_000])
def test_graphed_greedy_equals_eager(prec, budget):
    rng = np.random.default_rng(5)
    g = pb.build_ground_set(rng.standard_normal((3000, 24)), precision=prec)
    eager = pb.greedy_maximize(g, k=12, memory_budget=budget)
    graphed = pb.greedy_maximize(g, k=12, memory_budget=budget,
                                 evaluator=pb.Evaluator(cuda_graph=True))
    assert graphed.exemplar_indices == eager.exemplar_indices
    assert graphed.values == eager.values
    assert graphed.evaluations == eager.evaluations


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_greedy_graph_with_nccl_allreduce():
    """The row-sharded loop with its NCCL all-reduce captured in the graph
    (world size 1: the one-GPU box cannot host two NCCL ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2101_08763_b200.distributed import (build_sharded_ground,
                                                   communicator_record,
                                                   pin_nccl_env,
                                                   sharded_greedy)

    rng = np.random.default_rng(6)
    V = rng.standard_normal((5000, 40))
    ref = pb.greedy_maximize(pb.build_ground_set(V, precision=pb.Precision.bfloat16),
                             k=8)
    pin_nccl_env()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}",
                            rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        assert communicator_record()["nranks"] == 1
        sg = build_sharded_ground(V, pb.Precision.bfloat16, 0, 1, device=0)
        eager = sharded_greedy(sg, 8)
        graphed = sharded_greedy(sg, 8, graph=True)
    finally:
        dist.destroy_process_group()
    assert eager[0] == ref.exemplar_indices
    assert graphed == eager


def test_bench_graph_mode_matches_eager():
    def run(extra):
        out = subprocess.run(
            [sys.executable, "bench.py", "--points", "30000", "--steps", "3",
             "--warmup", "3", "--no-e2e", "--no-cpu", "--no-sub", *extra],
            cwd=ROOT, capture_output=True, text=True, timeout=600,
            env=dict(os.environ))
        assert out.returncode == 0, out.stderr[-3000:]
        return json.loads(out.stdout.strip().splitlines()[-1])

    eager, graphed = run([]), run(["--graph"])
    assert graphed["cuda_graph"] is True
    assert graphed["picks_head"] == eager["picks_head"]
    assert graphed["gpu_launches"] == eager["gpu_launches"] > 0
    assert graphed["roofline"]["kernel_ms_avg"] > 0
