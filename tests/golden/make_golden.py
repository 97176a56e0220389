"""Generate the golden vectors in tests/golden/ by running the REFERENCE.

Imports the unmodified reference package from /root/reference/pkg/src (this
container only -- /root/reference does not exist on the GPU box) and records
its outputs on seeded inputs.  The committed ``golden.npz`` is what the
oracle (oracle/exem_oracle.py) and the device path are checked against.

    python tests/golden/make_golden.py          # small cases (~seconds)
    python tests/golden/make_golden.py --c1     # + BASELINE config 1 (~2 min)
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def c1_data():
    """BASELINE config 1: Gaussian n=10,000, d=100, fp32, seed 1234."""
    rng = np.random.default_rng(1234)
    V = rng.standard_normal((10000, 100), dtype=np.float32)
    S = np.sort(rng.choice(10000, size=10, replace=False))
    return V, S


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main(argv):
    sys.path.insert(0, str(REF))
    import exembatch as eb
    from exembatch import Evaluator, EvaluationBatch, Precision

    g = {}
    hand = {}
    P64, P32, P16 = Precision.binary64, Precision.binary32, Precision.binary16

    # ---- hand cases (tests/test_core.py:56-59, test_evaluate.py:72-77, ...)
    line = eb.build_ground_set([[1.0], [3.0]], precision=P64)
    hand["line_aux_loss"] = line.aux_loss
    hand["line_f3"] = eb.evaluate_single(line, [[3.0]])
    hand["line_f1"] = eb.evaluate_single(line, [[1.0]])
    hand["line_f13"] = eb.evaluate_single(line, [[1.0], [3.0]])
    hand["line_batch"] = eb.evaluate_batch(
        Evaluator("reference"), line,
        EvaluationBatch.from_sets([[[3.0]], [[1.0]], [[1.0], [3.0]]])).tolist()
    r1 = eb.greedy_maximize(line, k=1)
    r2 = eb.greedy_maximize(line, k=2)
    hand["line_greedy1"] = [list(r1.exemplar_indices), list(r1.values), r1.evaluations]
    hand["line_greedy2"] = [list(r2.exemplar_indices), list(r2.values), r2.evaluations]
    tie = eb.build_ground_set([[2.0], [2.0], [1.0]], precision=P64)
    hand["tie_greedy1"] = list(eb.greedy_maximize(tie, k=1).exemplar_indices)
    zero2 = eb.build_ground_set([[0.0], [2.0]], precision=P64)
    hand["zero2_f2"] = eb.evaluate_single(zero2, [[2.0]])
    auxg = eb.build_ground_set([[1.0]], aux=[2.0], precision=P64)
    hand["custom_aux_loss"] = auxg.aux_loss
    hand["kmedoids_line_0"] = eb.kmedoids_loss(line, [[0.0]])
    hand["point_loss_line"] = [eb.point_loss(line, 0, [[3.0]]),
                               eb.point_loss(line, 1, [[3.0]])]
    hand["marginal_line"] = [eb.marginal_gain(line, [], [[3.0]]),
                             eb.marginal_gain(line, [[3.0]], [[1.0]])]
    g4 = eb.build_ground_set([[0.0], [1.0], [9.0], [10.0]], precision=P64)
    hand["assign_hand"] = eb.assign_clusters(g4, [[0.5], [9.5]]).tolist()
    hand["mu_examples"] = [eb.estimate_set_memory(50000, 10, 100, P32),
                           eb.estimate_set_memory(1, 1, 1, P16)]
    pl = eb.plan_chunks(1000, 300, 10)
    hand["plan_example"] = [pl.chunk_size, pl.chunk_count]

    # ---- random small instances (tests/_util.py:28-42 generator)
    for tag, prec in (("f64", P64), ("f32", P32)):
        rng = np.random.default_rng(2024 if tag == "f64" else 2025)
        for it in range(12):
            n = int(rng.integers(2, 65))
            d = int(rng.integers(1, 9))
            l = int(rng.integers(1, 17))
            data = rng.random((n, d))
            grd = eb.build_ground_set(data, precision=prec)
            sets_idx = []
            for _ in range(l):
                m = min(int(rng.integers(1, 9)), n)
                sets_idx.append(np.sort(rng.choice(n, size=m, replace=False)))
            batch = EvaluationBatch.from_sets([grd.matrix[i] for i in sets_idx])
            vals = eb.evaluate_batch(Evaluator("reference"), grd, batch)
            key = f"rand_{tag}_{it}"
            g[key + "_data"] = data
            g[key + "_card"] = np.array([len(s) for s in sets_idx])
            g[key + "_idx"] = np.concatenate(sets_idx)
            g[key + "_vals"] = np.asarray(vals)
            g[key + "_auxd"] = grd.aux_distances
            g[key + "_auxloss"] = np.array([grd.aux_loss])
            g[key + "_mind0"] = eb.min_distances(grd, grd.matrix[sets_idx[0]])
            g[key + "_labels0"] = eb.assign_clusters(grd, grd.matrix[sets_idx[0]])

    # ---- greedy trajectories (uniform [0,1) and Gaussian)
    specs = [("g_u64", 60, 4, 5, P64, "u", 107), ("g_u32", 80, 3, 6, P32, "u", 109),
             ("g_n32", 300, 16, 6, P32, "n", 111), ("g_n64", 300, 16, 6, P64, "n", 113),
             ("g_n32d100", 1500, 100, 4, P32, "n", 115)]
    for key, n, d, k, prec, kind, seed in specs:
        rng = np.random.default_rng(seed)
        data = rng.random((n, d)) if kind == "u" else rng.standard_normal((n, d))
        grd = eb.build_ground_set(data, precision=prec)
        res = eb.greedy_maximize(grd, k=k, evaluator=Evaluator("parallel", worker_count=8))
        g[key + "_data"] = data
        g[key + "_picks"] = np.array(res.exemplar_indices)
        g[key + "_values"] = np.array(res.values)
        g[key + "_evals"] = np.array([res.evaluations])

    # ---- half precision (tests/test_evaluate.py:230-243 shape)
    rng = np.random.default_rng(89)
    data = rng.random((64, 32), dtype=np.float32)
    sets_idx = [np.sort(rng.choice(64, size=5, replace=False)) for _ in range(8)]
    g16 = eb.build_ground_set(data, precision=P16)
    g32 = eb.build_ground_set(data, precision=P32)
    g["half_data"] = data
    g["half_idx"] = np.stack(sets_idx)
    g["half_vals16"] = eb.evaluate_batch(Evaluator("reference"), g16,
                                         EvaluationBatch.from_sets([g16.matrix[i] for i in sets_idx]))
    g["half_vals32"] = eb.evaluate_batch(Evaluator("reference"), g32,
                                         EvaluationBatch.from_sets([g32.matrix[i] for i in sets_idx]))

    # ---- BASELINE config 1 (slow: reference parallel backend, 8 workers)
    if "--c1" in argv:
        V, S = c1_data()
        g["c1_sha"] = np.array([sha(V)])
        g["c1_S"] = S
        t0 = time.perf_counter()
        for tag, prec in (("f32", P32), ("f64", P64)):
            grd = eb.build_ground_set(V, precision=prec)
            g[f"c1_{tag}_fS"] = np.array([eb.evaluate_single(grd, grd.matrix[S])])
            g[f"c1_{tag}_auxloss"] = np.array([grd.aux_loss])
            res = eb.greedy_maximize(grd, k=10,
                                     evaluator=Evaluator("parallel", worker_count=8))
            g[f"c1_{tag}_picks"] = np.array(res.exemplar_indices)
            g[f"c1_{tag}_values"] = np.array(res.values)
            print(f"c1 {tag}: {res.exemplar_indices} {time.perf_counter()-t0:.1f}s",
                  flush=True)
    else:
        old = OUT / "golden.npz"
        if old.exists():
            with np.load(old) as z:
                for key in z.files:
                    if key.startswith("c1_"):
                        g[key] = z[key]

    # ---- the reference's benchmark problem generator (src/bench.py:66-93)
    from exembatch.bench import generate_problem

    for tag, prec in (("32", P32), ("64", P64), ("16", P16)):
        ground, batch = generate_problem(50, 4, 3, 5, 11, prec)
        g[f"gen{tag}_values"] = np.asarray(ground.matrix)
        g[f"gen{tag}_sets"] = np.stack([np.asarray(s) for s in batch.sets])

    np.savez_compressed(OUT / "golden.npz", **g)
    (OUT / "hand.json").write_text(json.dumps(hand, indent=1) + "\n")
    print(f"wrote {len(g)} arrays, {len(hand)} hand cases")


if __name__ == "__main__":
    main(sys.argv[1:])
