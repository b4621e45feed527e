"""Wall time of the optimize() step driver (optimizer.hpp:404-505) at a BASELINE workload on one GPU:
Adam steps (one objective evaluation each) with the per-step preconditioner rebuild and device-side
probe rotation, no validation set.  python tools/opt_step_time.py [workload] [steps]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_00243_b200 as gk  # noqa: E402
from paper_2107_00243_b200 import workloads  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
w = workloads.config(wl)
x, y = workloads.generate(w)
fam = ["rbf", "matern12", "matern32", "matern52"][w.family]
init = gk.Hyperparameters.from_raw(w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise)
opts = gk.OptOptions(method="adam", max_steps=steps, adam_lr=0.02, early_stop_patience=steps + 1)
cfg = gk.MllConfig(gk.CgConfig(w.max_iters, w.rel_tol, False, "tf32x3", 2), True, "auto")
t0 = time.perf_counter()
res = gk.optimize(gk.Dataset(x, y), None, gk.KernelSpec(fam), init, gk.PivotedCholeskyBuilder(w.rank),
                  w.probes, opts, cfg, seed=17)
t1 = time.perf_counter()
walls = [float(s.wall_time_s) for s in res.trace.steps]
per = np.diff([0.0] + walls)
print(json.dumps({"workload": w.name, "n": w.n, "method": "adam", "steps": len(walls), "total_s": t1 - t0,
                  "step_wall_s": [round(float(v), 5) for v in per], "median_step_s": float(np.median(per[1:])),
                  "objective": [round(float(s.objective), 4) for s in res.trace.steps],
                  "evaluations": len(res.trace.evaluations), "total_cg_iterations": int(res.total_cg_iterations), "seconds_total": float(res.seconds_total)}))
