"""Benchmark: BASELINE config 4 -- full Greedy, n=1,000,000, d=100, k=50.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" is one Greedy iteration over l = n - t candidate sets S u {c}
(kernel K3 over every candidate, K6 reduce, K5 argmax, K2 m-update).  The
device run is one Greedy of W + K steps: the first W steps are untimed
warm-up, the next K are timed (default 3 + 47 = 50 = BASELINE's k); the e2e
leg always runs the full k = 50 Greedy through the public API.  Unless
--no-sub, the other BASELINE configs follow as sub-records ("configs",
tools/bench_configs.py: C2, C3, C5 and the other C4 precisions).  N > 1 runs under
torchrun: V is row-sharded, the l partial gains are all-reduced over NCCL
each step (strong scaling: the problem is fixed, N GPUs share it).

Prints ONE JSON line on rank 0 (contract in the task statement): value =
candidate-set evaluations per second for the whole job; ``e2e`` is the same
metric through the public API (build_ground_set + greedy_maximize from host
numpy, H2D/D2H inside the timed region); ``roofline`` refers to the dominant
kernel (gains_tc_kernel, tcgen05); ``cpu_baseline`` times the CPU oracle
port of the reference's path (oracle/exem_oracle.py) on a bounded sample.

``--impl reference`` times that CPU port alone (all host threads) on the
same config and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("candidate-set evals/sec & dist-evals/s vs roofline "
          "(n=1M,d=100,k=50) at 1/2/4/8 GPU")
UNIT = "candidate-set evals/s"
PRECISION_CHOICES = ("bf16", "fp16", "fp32", "fp64")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=47)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--points", dest="n", type=int, default=1_000_000)
    ap.add_argument("--dim", dest="d", type=int, default=100)
    ap.add_argument("--precision", default="bf16", choices=PRECISION_CHOICES)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--tensor-fp32", action="store_true",
                    help="fp32 gains on tensor cores via split-bf16 operands")
    ap.add_argument("--graph", action="store_true",
                    help="replay the timed steps from one CUDA graph "
                    "(optimize.capture_steps; NCCL all-reduce captured too)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-sub", action="store_true",
                    help="skip the other BASELINE configs (sub-records)")
    ap.add_argument("--sub-cpu-seconds", type=float, default=2.0)
    return ap.parse_args()


K_FULL = 50  # BASELINE config 4: Greedy k = 50


def synthetic(n, d, seed):
    """Gaussian N(0, I) float32; e0 = 0."""
    return np.random.default_rng(seed).standard_normal((n, d), dtype=np.float32)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
            "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU leg
def cpu_sample(n, d, seed, set_size, seconds, threads, V=None):
    """Time the oracle port of the reference's evaluate path (fp32, parallel
    row split like evaluate.py:162-170) on sets of ``set_size`` at the
    full n: returns (sets/s, sets timed)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import exem_oracle as O  # CPU baseline leg only

    if V is None:
        V = synthetic(n, d, seed)
    g = O.Ground(V, np.float32)
    rng = np.random.default_rng(seed + 1)
    done, t_total = 0, 0.0
    while True:  # at least one batch of `threads` sets
        sets = [g.matrix[np.sort(rng.choice(n, size=set_size, replace=False))]
                for _ in range(threads)]
        t0 = time.perf_counter()
        O.evaluate_batch(g, sets, workers=threads)
        t_total += time.perf_counter() - t0
        done += len(sets)
        if t_total >= seconds:
            return done / t_total, done, t_total


def run_reference(args, rank, world):
    """--impl reference: the CPU port on the host cores, rank 0 only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n, d = args.n, args.d
    V = synthetic(n, d, args.seed)
    total_sets, total_t = 0, 0.0
    per_step = max(1.0, min(args.cpu_seconds / 4, 4.0))
    for step in range(args.warmup):  # untimed: worker pool, page-in of V
        cpu_sample(n, d, args.seed + step, step + 1, 0.25, threads, V)
    for i, step in enumerate(range(args.warmup, args.warmup + args.steps)):
        # the timed steps sample the set sizes of the whole k = 50 Greedy
        # (|S u {c}| = 1..50): the CPU's per-set cost grows with |S|, the
        # device's per-step cost does not
        set_size = 1 + int(round(i * (K_FULL - 1) / max(1, args.steps - 1)))
        rate, cnt, t = cpu_sample(n, d, args.seed + step, set_size, per_step,
                                  threads, V)
        total_sets += cnt
        total_t += t
    value = total_sets / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * (n - args.warmup - args.steps / 2) / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "fp32", "data": "synthetic Gaussian N(0,1), seed "
        f"{args.seed}",
        "config": {"workload": "C4 Greedy n=1M d=100 k=50 (CPU port of the "
                   "reference, bounded sample per step)", "n": n, "d": d,
                   "k": K_FULL},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port",
                         "sample": f"{total_sets} sets, sizes spread over "
                         f"1..{K_FULL} (the whole k={K_FULL} Greedy) across "
                         f"the {args.steps} steps, full n, numpy/OpenBLAS "
                         "restatement, 1 BLAS thread per worker"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    assert args.warmup >= 3, "W >= 3 warm-up steps"

    import torch
    import torch.distributed as dist

    import paper_2101_08763_b200 as pb
    from paper_2101_08763_b200 import _native as N
    from paper_2101_08763_b200.distributed import (DeviceShardOps,
                                                   build_sharded_ground,
                                                   communicator_record,
                                                   pin_nccl_env)
    from paper_2101_08763_b200.optimize import GreedyRun

    # EXEM_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 over gloo,
    # to exercise the N > 1 code path on a one-GPU box
    share = os.environ.get("EXEM_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if share:
            dist.init_process_group("gloo")
        else:
            pin_nccl_env()  # fixed algo/proto; INIT log (nRanks) on stderr
            dist.init_process_group("nccl",
                                    device_id=torch.device("cuda", local))
        comm = communicator_record()
        if rank == 0:
            print(f"communicator: {json.dumps(comm)}", file=sys.stderr,
                  flush=True)
    prec = pb.Precision.from_name(args.precision)
    n, d = args.n, args.d
    k = args.warmup + args.steps
    V = synthetic(n, d, args.seed)
    lib = N.lib()

    sg = build_sharded_ground(V, prec, rank, world, device=local)
    sp = int(lib.split_points(n))
    run = GreedyRun(sg.local, cand=sg.cand, k_cap=k, split_pts=sp,
                    split32=args.tensor_fp32)
    ops = DeviceShardOps(run)
    stream = torch.cuda.current_stream()

    def all_reduce(t):
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

    def barrier():
        if world > 1:
            dist.barrier()

    # K3 timing: events on the launching (current) stream around each launch
    ev = []
    orig = run.compute_gains

    def timed_gains(chunk=None, out=None):
        # external events: recorded as graph nodes under --graph capture
        cur = torch.cuda.current_stream()
        a = torch.cuda.Event(enable_timing=True, external=args.graph)
        b = torch.cuda.Event(enable_timing=True, external=args.graph)
        a.record(cur)
        orig(chunk, out=out)
        b.record(cur)
        ev.append((a, b))

    # EXEM_PEER_REDUCE=1 (N > 1): per-step exchange over CUDA-IPC peer memory
    # (distributed.PeerGains: fixed-order sum fused into the argmax) instead
    # of the NCCL all-reduce
    peer = None
    if world > 1 and os.environ.get("EXEM_PEER_REDUCE") == "1":
        from paper_2101_08763_b200.distributed import PeerGains

        peer = PeerGains(run.l, run.dg.dev)

    def do_step(step):
        if peer is None:
            ops.local_gains()
            all_reduce(ops.gains_buffer())
            ops.select(step)
        else:
            run.compute_gains(out=peer.local_buffer(step))
            peer.publish(step, run.stream)
            peer.select(run, step)
        ops.update(step)

    ops.start()
    for step in range(args.warmup):
        do_step(step)
    torch.cuda.synchronize()
    barrier()
    run.compute_gains = timed_gains
    launches0 = lib.launch_count()
    graph = None
    if args.graph:
        from paper_2101_08763_b200.optimize import capture_steps

        graph = capture_steps(range(args.warmup, k), do_step)
        captured = lib.launch_count() - launches0
        torch.cuda.synchronize()
        barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for step in range(args.warmup, k):
                do_step(step)
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
    # kernels launched in the timed region (a replay runs the captured ones)
    launches = (captured if graph is not None
                else lib.launch_count() - launches0)
    ms_local = t0.elapsed_time(t1)
    run.compute_gains = orig
    if peer is not None:
        peer.close()
    all_reduce(ops.msum_buffer())
    ms_t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    gains_ms = [a.elapsed_time(b) for a, b in ev]
    gains_ms_local = float(np.mean(gains_ms))

    picks = run.sel_idx.cpu().numpy()[:k]
    l_steps = [n - t for t in range(args.warmup, k)]
    evals = float(sum(l_steps))
    value = evals / (ms / 1e3)
    n_local = sg.rows[1] - sg.rows[0]

    # roofline of the dominant kernel: 2*n_local*l*d algorithmic flop/launch
    peaks, peak_src = load_peaks()
    half = prec.is_half or run.split32
    flop = 2.0 * n_local * float(np.mean(l_steps)) * d
    achieved = flop / (gains_ms_local / 1e3) / 1e12
    if half:
        peak = float(peaks.get("bf16_tflops_sustained",
                               peaks.get("bf16_tflops")))
        bound = "tensor"
    else:
        simt = ROOT / "profiles" / "simt_peak.json"
        sp_j = json.loads(simt.read_text()) if simt.exists() else {}
        peak = float(sp_j.get("fp64_dfma_tflops", 37.2)
                     if prec is pb.Precision.binary64
                     else sp_j.get("fp32_ffma_tflops", 74.4))
        bound = "fp32-pipe" if prec is pb.Precision.binary32 else "fp64-pipe"
    traffic = None
    tfile = ROOT / "profiles" / "gains_tc_traffic.json"
    if half and tfile.exists():
        try:
            tj = json.loads(tfile.read_text())
            # the ncu capture is of one C4 launch on one GPU: only valid for
            # that configuration
            if (tj.get("n"), tj.get("d"), tj.get("world")) == (n, d, world):
                traffic = tj.get("bytes_per_launch")
        except Exception:
            traffic = None

    result = None
    if rank == 0:
        cpu = None
        if not args.no_cpu and world >= 1:
            threads = os.cpu_count() or 1
            mid = (K_FULL + 1) // 2 + 1  # mean |S u c| of the k=50 Greedy
            rate, cnt, secs = cpu_sample(n, d, args.seed, mid, args.cpu_seconds,
                                         threads, V)
            cpu = {"value": rate, "unit": UNIT, "cores": threads,
                   "kind": "port",
                   "sample": f"{cnt} sets of size {mid} (mean |S u c| of the "
                   f"k={K_FULL} Greedy) at full n={n}, d={d}, fp32, "
                   f"{secs:.1f}s; "
                   "oracle/exem_oracle.py numpy/OpenBLAS restatement of "
                   "evaluate.py:142-170"}
        clocks = clk.summary()
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step":
            ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.precision,
            "data": f"synthetic Gaussian N(0,1) float32 seed {args.seed}, "
                    f"stored as {args.precision}",
            "communicator": comm if world > 1 else None,
            "exchange": "peer memory (CUDA IPC, fused sum+argmax)" if peer
            is not None else (f"{dist.get_backend()} all-reduce" if world > 1
                              else "none"),
            "config": {"workload": "C4 full Greedy k=50: one step = all l=n-t "
                       "candidate sets S u {c} (K3 gains + K6 + K5 argmax + "
                       "K2 m-update)" + (" [fp32 gains on tensor cores, "
                                         "split-bf16]" if run.split32 else ""),
                       "n": n, "d": d, "k": K_FULL,
                       "device_timed_steps": f"{args.warmup}..{k - 1} of a "
                       f"{k}-step run (per-step work depends only on "
                       "l = n - t); e2e runs the full k",
                       "parallelism": f"row-shard x{world}" if world > 1 else
                       "1 GPU", "l2": "inputs larger than L2 (V operands "
                       f"{2 * n * 128 * 2 / 2**20:.0f} MiB)"},
            "dist_evals_per_s": {"executed": n * evals / (ms / 1e3),
                                 "reference_equivalent": n * sum(
                                     (n - t) * (t + 1) for t in
                                     range(args.warmup, k)) / (ms / 1e3)},
            "roofline": {"bound": bound, "kernel": "gains_tc_kernel" if half
                         else "gains_simt_kernel", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_source": f"{peak_src} "
                         f"{'bf16_tflops_sustained' if half else 'profiles/simt_peak.json'}",
                         "traffic": traffic, "algorithmic_flop_per_launch": flop,
                         "kernel_ms_avg": gains_ms_local,
                         "kernel_share_of_step": gains_ms_local * args.steps / ms},
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "cuda_graph": bool(args.graph),
            "k3_epilogue": ({"groups": run.epi,
                             "screen_hit_fraction": run.hit_fraction}
                            if run.tc else None),
            "clocks": clocks,
            "picks_head": [int(x) for x in picks[:5]],
        }
    # ---- e2e through the public API (1 GPU: build_ground_set + greedy)
    if world == 1 and not args.no_e2e:
        del run, ops, sg
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        ke = max(K_FULL, k)  # the full k = 50 Greedy through the public API
        t_start = time.perf_counter()
        g = pb.build_ground_set(V, precision=prec)
        res = pb.greedy_maximize(
            g, k=ke, evaluator=pb.Evaluator(tensor_fp32=args.tensor_fp32))
        t_e2e = time.perf_counter() - t_start
        e2e_evals = float(sum(n - t for t in range(ke)))
        # H2D: V (storage dtype, row-major as generated) + e0; D2H: the
        # column-major GroundSet.matrix (transposed on the device), the
        # aux distances, aux sum, picks and trajectory sums
        vb = n * d * prec.bytes_per_value
        h2d = vb + d * prec.bytes_per_value
        d2h = vb + n * np.dtype(np.float32).itemsize + 2 * 8 * ke + 8
        result["e2e"] = {"value": e2e_evals / t_e2e, "unit": UNIT,
                         "h2d_bytes_per_step": h2d / ke,
                         "d2h_bytes_per_step": d2h / ke,
                         "seconds": t_e2e, "steps": ke,
                         "api": "build_ground_set(numpy C-order float32) + "
                                f"greedy_maximize(k={ke})",
                         "picks_match_device_run":
                         list(res.exemplar_indices[:k]) ==
                         [int(x) for x in picks]}
    elif world > 1 and not args.no_e2e:
        # e2e through the public multi-GPU API: every rank uploads V from host
        # memory (build_sharded_ground: candidate replica + its row shard) and
        # runs the row-sharded Greedy (NCCL all-reduce per step); the result
        # picks/values come back to the host.  Device time = max over ranks.
        from paper_2101_08763_b200.distributed import sharded_greedy

        del run, ops, sg
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        dist.barrier()
        t_start = time.perf_counter()
        sg2 = build_sharded_ground(V, prec, rank, world, device=local)
        picks2, _ = sharded_greedy(sg2, k)
        torch.cuda.synchronize()
        t_e2e = torch.tensor([time.perf_counter() - t_start],
                             dtype=torch.float64, device="cuda")
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        if rank == 0:
            e2e_evals = float(sum(n - t for t in range(k)))
            h2d = world * (n * d * prec.bytes_per_value +
                           d * prec.bytes_per_value)
            d2h = world * (2 * 8 * k + 8)
            result["e2e"] = {"value": e2e_evals / float(t_e2e.item()),
                             "unit": UNIT, "h2d_bytes_per_step": h2d / k,
                             "d2h_bytes_per_step": d2h / k,
                             "seconds": float(t_e2e.item()), "steps": k,
                             "api": "build_sharded_ground(numpy) + "
                                    "sharded_greedy(k) on every rank",
                             "picks_match_device_run":
                             list(picks2) == [int(x) for x in picks]}
    elif rank == 0:
        result["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0, "note": "--no-e2e"}
    if rank == 0 and world == 1 and not args.no_sub:
        # the other BASELINE configs, a few steps each (tools/bench_configs)
        sys.path.insert(0, str(ROOT / "tools"))
        import bench_configs

        torch.cuda.empty_cache()
        with ClockSampler(local) as clk2:
            result["configs"] = bench_configs.all_records(
                cpu_seconds=args.sub_cpu_seconds,
                headline_precision=args.precision, log=sys.stderr)
        result["configs_clocks"] = clk2.summary()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
