"""Generates tests/golden/*.json: oracle outputs on the BASELINE C1 workload and a
small multi-family grid.  Run from the repo root:  python tests/golden/make_golden.py

The oracle (oracle/, test infrastructure) is the Eigen-free restatement of the
reference pinned by tests/test_oracle_*.py; these fixtures let the GPU tests
compare against it without recomputing on the GPU box."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2107_00243_b200 import workloads  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def c1(max_iters=None):
    w = workloads.config("C1")
    x, y = workloads.generate(w)
    p = oracle.Params(w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise)
    seed = oracle.mix_seed(workloads.PROBE_SEED, 1)
    z = oracle.make_probes(w.n, w.probes, seed)
    r = oracle.evaluate_mll(w.family, x, p, y, z, seed=seed, prec="pivchol", rank=w.rank, mode=oracle.DENSE,
                            max_iters=max_iters or w.max_iters, rel_tol=w.rel_tol)
    pc = oracle.pivoted_cholesky(w.rank, family=w.family, x=x, p=p)
    return {
        "workload": "C1", "n": w.n, "d": w.d, "l": w.probes, "rank": w.rank, "probe_seed": seed,
        "x_sha": float(np.sum(x * np.arange(1, x.size + 1).reshape(x.shape))), "y_sum": float(y.sum()),
        "value": r["value"], "logdet": r["logdet"], "quad": r["quad"], "logdet_precond": r["logdet_precond"],
        "gradient": r["gradient"].tolist(), "forward_gammas": r["forward_gammas"].tolist(),
        "backward_gammas": r["backward_gammas"].tolist(), "forward_cg_iterations": r["forward_cg_iterations"].tolist(),
        "solve_iterations": r["solve_iterations"], "total_cg_iterations": r["total_cg_iterations"],
        "value_sample_variance": r["value_sample_variance"], "pivots": pc["pivots"].tolist(),
    }


def grid():
    cases = []
    for fam in (0, 1, 2, 3):
        for rank in (0, 8):
            n, d, l = 300, 2, 4
            x = oracle.random_matrix(n, d, 900 + fam)
            y = np.sin(2 * x[:, 0]) + 0.1 * oracle.random_matrix(n, 1, 901 + fam)[:, 0]
            p = oracle.Params(d, 1.1, 0.8, 0.05)
            z = oracle.make_probes(n, l, 17 + fam)
            r = oracle.evaluate_mll(fam, x, p, y, z, seed=17 + fam, prec="pivchol", rank=rank,
                                    mode=oracle.DENSE, max_iters=200, rel_tol=1e-8)
            cases.append({"family": fam, "rank": rank, "n": n, "d": d, "l": l, "x_seed": 900 + fam,
                          "y_seed": 901 + fam, "probe_seed": 17 + fam, "value": r["value"], "logdet": r["logdet"],
                          "gradient": r["gradient"].tolist(), "backward_gammas": r["backward_gammas"].tolist(),
                          "forward_gammas": r["forward_gammas"].tolist()})
    return cases


if __name__ == "__main__":
    with open(os.path.join(OUT, "c1_oracle.json"), "w") as f:
        json.dump(c1(), f, indent=1)
    # C1 with solves run to convergence (the BASELINE C1 max of 100 iterations truncates every solve)
    with open(os.path.join(OUT, "c1_converged_oracle.json"), "w") as f:
        json.dump(c1(max_iters=1000), f, indent=1)
    with open(os.path.join(OUT, "grid_oracle.json"), "w") as f:
        json.dump(grid(), f, indent=1)
    print("wrote", OUT)
