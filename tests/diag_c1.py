"""Diagnostic (run on a GPU box): relative errors of the GPU evaluate_mll vs the
C1 golden fixture in every precision/backward mode, plus true residuals."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_00243_b200 as gk  # noqa: E402
from paper_2107_00243_b200 import workloads  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "c1_oracle.json")))
w = workloads.config("C1")
x, y = workloads.generate(w)
hp = gk.Hyperparameters.from_raw(w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise)
seed = gk.mix_seed(workloads.PROBE_SEED, 1)
z = gk.make_probes(w.n, w.probes, seed)
op = gk.KernelOperator(gk.KernelSpec("rbf"), x, hp)
pc = gk.pivoted_cholesky_with_derivatives(op, w.rank)
print("pivots identical:", pc.pivots() == g["pivots"])
for mi in (100, 1000):
    for prec in ("fp64", "fp32"):
        for bw in ("faithful", "fused"):
            cfg = gk.MllConfig(gk.CgConfig(mi, w.rel_tol, False, prec, 2), True, bw)
            r = gk.evaluate_mll(y, op, pc, z, cfg)
            if mi == 100:
                ev = abs(r.value - g["value"]) / abs(g["value"])
                el = abs(r.logdet - g["logdet"]) / abs(g["logdet"])
                eg = np.abs(r.gradient - np.array(g["gradient"])) / np.abs(g["gradient"])
                print(f"max_iters={mi} {prec} {bw}: value {ev:.2e} logdet {el:.2e} quad {abs(r.quad-g['quad'])/g['quad']:.2e}"
                      f" grad max {eg.max():.2e} {np.array2string(eg, precision=1)} iters {r.solve_iterations} "
                      f"refine {r.refine_passes} res {r.max_true_rel_residual:.2e} t={r.seconds_total:.3f}s")
            else:
                print(f"max_iters={mi} {prec} {bw}: value {r.value:.8f} logdet {r.logdet:.6f} grad "
                      f"{np.array2string(r.gradient, precision=6)} iters {r.solve_iterations} "
                      f"fwd {r.forward_cg_iterations} res {r.max_true_rel_residual:.2e}")
