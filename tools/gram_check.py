"""Accuracy of the Gram (expanded-distance) tensor-core MVM vs the direct-difference one against
the fp64 MVM, on a BASELINE config's data at reduced n (default C5): relative error of K V per
column, and the max centred pre-scaled |x|^2 the auto-selection bound looks at.
python tools/gram_check.py [workload] [n] [t]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_00243_b200 as gk  # noqa: E402
from paper_2107_00243_b200 import workloads  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
t = int(sys.argv[3]) if len(sys.argv) > 3 else 16
w = workloads.config(wl, n=n)
x, y = workloads.generate(w)
fam = {0: "rbf", 1: "matern12", 2: "matern32", 3: "matern52"}[w.family]
lo, lls, ln = w.log_params
op = gk.KernelOperator(gk.KernelSpec(fam), x, gk.Hyperparameters(lo, np.asarray(lls), ln))
rng = np.random.default_rng(1)
v = np.asfortranarray(np.concatenate([y[:, None], rng.choice([-1.0, 1.0], size=(n, t - 1)) / np.sqrt(n)], axis=1))
ref = op.apply(v, precision="fp64")
out = {}
for var in ("direct", "gram"):
    op.set_mvm_variant(var)
    got = op.apply(v, precision="tf32x3")
    err = np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0)
    out[var] = (op.mvm_variant(), float(err.max()), float(np.median(err)))
print(f"{wl} n={n} d={w.d} {fam}: max centred pre-scaled |x|^2 = {out['gram'][0][1]:.1f}")
for var, (mv, emax, emed) in out.items():
    print(f"  forced {var:6s} -> kernel {mv[0]:6s}: rel err max {emax:.2e}, median {emed:.2e}")
