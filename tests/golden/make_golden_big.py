"""Generates the BASELINE-size golden fixtures (C2-C5) from the CPU oracle.

Run from the repo root (CPU only; ORC_NATIVE=1 builds/loads the oracle for this host's
vector ISA — same sums, bitwise the portable build's results, just faster):

    ORC_NATIVE=1 python tests/golden/make_golden_big.py pivots      # C2..C5 pivot sequences  (~5 min)
    ORC_NATIVE=1 python tests/golden/make_golden_big.py mvm         # MVM row subsets C2..C5  (~3 min)
    ORC_NATIVE=1 python tests/golden/make_golden_big.py c2 --rank 100   # C2 evaluate_mll     (~20 min)

Outputs (tests/golden/):
  big_pivots.json        pivot sequence of the pivoted Cholesky (preconditioners.hpp:236-264) at
                         C2 (k=100, 500), C3 (k=200), C4 (k=500), C5 (k=500), with the per-step
                         pivot values and the relative gap to the runner-up candidate (how close
                         the argmax came to a tie: a GPU pivot mismatch is only excusable at a gap
                         at rounding level, and none is)
  big_mvm_rows.npz       rows of (K + sigma^2 I) V for 512 sampled rows (first, last, 128-row
                         block edges, seeded random) at every config; V ~ N(0,1) seeded
  c2_oracle_rank{R}.json evaluate_mll (gp_likelihood.hpp:51-103) at C2 with the reference
                         default solver (max_iters 200, rel_tol 1e-6), probes
                         make_probes(n, 50, mix_seed(17, 1)), the pivoted-Cholesky preconditioner
                         of rank R with frozen-pivot derivative factors (experiments.hpp:30-68);
                         the operator is MatrixFree (optimizer.hpp:427 picks it for n > 4096);
                         all solves of a phase run as one lock-step batch whose columns are bitwise
                         the oracle's per-column pcg_solve (tests/test_oracle_lockstep.py)

The fixtures are inputs-by-seed: the GPU tests regenerate X, y, Z and V with
paper_2107_00243_b200.workloads / numpy's seeded generators and compare outputs only.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2107_00243_b200 import workloads  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
PIVOT_CASES = [("C2", 100), ("C2", 500), ("C3", 200), ("C4", 500), ("C5", 500)]
MVM_CASES = ["C2", "C3", "C4", "C5"]
MVM_ROWS = 512


def params(w):
    return oracle.Params(w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise)


def checksum(x):
    x = np.asarray(x, dtype=np.float64).ravel(order="C")
    return float(np.dot(x, np.cos(np.arange(x.size, dtype=np.float64) * 1e-3)))


def mvm_rows(n, seed=4242):
    """First and last row, both sides of every 16th 128-row block edge, and seeded random rows."""
    fixed = {0, n - 1}
    for b in range(128, n, 128 * 16):
        fixed.update((b - 1, b))
    rng = np.random.default_rng(seed + n)
    rest = rng.choice(n, MVM_ROWS, replace=False)
    rows = sorted(fixed)
    for r in rest:
        if len(rows) >= MVM_ROWS:
            break
        if r not in fixed:
            rows.append(int(r))
    return np.array(sorted(rows[:MVM_ROWS]), dtype=np.int64)


def mvm_v(w, t):
    return np.asfortranarray(np.random.default_rng(777 + w.data_seed).standard_normal((w.n, t)))


def do_pivots():
    out = {}
    for name, k in PIVOT_CASES:
        w = workloads.config(name, rank=k)
        x, _ = workloads.generate(w)
        p = params(w)
        t0 = time.time()
        pc = oracle.pivoted_cholesky(k, family=w.family, x=x, p=p)
        L = pc["L"]
        piv = pc["pivots"]
        # per-step diagonal (numpy restatement of the reference's d -= l^2 update) -> runner-up gap
        dg = np.full(w.n, w.outputscale ** 2)
        gaps, vals = [], []
        for s in range(pc["rank"]):
            top2 = np.partition(dg, -2)[-2:]
            vals.append(float(dg[piv[s]]))
            gaps.append(float((top2[1] - top2[0]) / top2[1]))
            dg -= L[:, s] ** 2
        # step 0 is a tie by construction (the diagonal is o^2 everywhere; the strict '>' scan
        # takes index 0, preconditioners.hpp:247-249), so the closeness measure starts at step 1
        later = gaps[1:] if len(gaps) > 1 else [float("inf")]
        out[f"{name}_{k}"] = {"workload": name, "n": w.n, "d": w.d, "rank": k, "pivots": piv.tolist(),
                              "pivot_values": vals, "min_relative_gap": min(later),
                              "argmin_gap_step": 1 + int(np.argmin(later)),
                              "remaining_max": float(pc["remaining"].max()), "x_checksum": checksum(x),
                              "seconds": time.time() - t0}
        print(name, k, "pivots", piv[:8], "min gap (steps >= 1)", min(later), f"{time.time() - t0:.1f}s", flush=True)
        del L, pc
    with open(os.path.join(OUT, "big_pivots.json"), "w") as f:
        json.dump(out, f)


def do_mvm():
    arrays = {}
    meta = {}
    for name in MVM_CASES:
        w = workloads.config(name)
        x, _ = workloads.generate(w)
        t = w.probes + 1
        v = mvm_v(w, t)
        rows = mvm_rows(w.n)
        t0 = time.time()
        got = oracle.kernel_apply_rows(w.family, x, params(w), rows, v)
        arrays[f"{name}_rows"] = rows
        arrays[f"{name}_out"] = got
        meta[name] = {"n": w.n, "t": t, "x_checksum": checksum(x), "v_checksum": checksum(v[:4096])}
        print(name, "mvm rows", got.shape, f"{time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(OUT, "big_mvm_rows.npz"), meta=json.dumps(meta), **arrays)


def do_c2(rank):
    w = workloads.config("C2", rank=rank)
    x, y = workloads.generate(w)
    p = params(w)
    seed = oracle.mix_seed(workloads.PROBE_SEED, 1)
    z = oracle.make_probes(w.n, w.probes, seed)
    t0 = time.time()
    prec = "pivchol"  # rank 0 = sigma^2 I (pivoted_cholesky of rank 0, experiments.hpp:37-38)
    r = oracle.evaluate_mll(w.family, x, p, y, z, seed=seed, prec=prec, rank=rank, mode=oracle.CACHED,
                            max_iters=w.max_iters, rel_tol=w.rel_tol, lockstep=True)
    secs = time.time() - t0
    g = {"workload": "C2", "n": w.n, "d": w.d, "l": w.probes, "rank": rank, "preconditioner": prec,
         "max_iters": w.max_iters, "rel_tol": w.rel_tol, "probe_seed": seed,
         "x_checksum": checksum(x), "y_checksum": checksum(y),
         "value": r["value"], "logdet": r["logdet"], "quad": r["quad"], "logdet_precond": r["logdet_precond"],
         "gradient": r["gradient"].tolist(), "forward_gammas": r["forward_gammas"].tolist(),
         "backward_gammas": r["backward_gammas"].tolist(),
         "forward_cg_iterations": r["forward_cg_iterations"].tolist(), "solve_iterations": r["solve_iterations"],
         "total_cg_iterations": r["total_cg_iterations"], "value_sample_variance": r["value_sample_variance"],
         "pivots": r["pivots"].tolist() if r["pivots"] is not None else [], "oracle_seconds": secs,
         "oracle_threads": oracle.num_threads()}
    with open(os.path.join(OUT, f"c2_oracle_rank{rank}.json"), "w") as f:
        json.dump(g, f, indent=1)
    np.save(os.path.join(OUT, f"c2_oracle_rank{rank}_u.npy"), r["u"])
    print("C2 rank", rank, "value", r["value"], "iters", r["total_cg_iterations"], f"{secs:.0f}s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["pivots", "mvm", "c2"])
    ap.add_argument("--rank", type=int, default=100)
    a = ap.parse_args()
    {"pivots": do_pivots, "mvm": do_mvm, "c2": lambda: do_c2(a.rank)}[a.what]()
