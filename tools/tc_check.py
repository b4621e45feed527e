"""tcgen05 MVM check: accuracy vs the fp64 MVM and timing vs the SIMT fp32 kernel."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_00243_b200 as gk  # noqa: E402

cases = [(1000, 3, 9, "rbf"), (2051, 9, 51, "matern32"), (700, 18, 65, "matern52"), (16384, 18, 51, "matern32"),
         (65536, 11, 65, "matern32"), (65536, 3, 51, "matern52")]
for n, d, t, fam in cases:
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((n, d))
    v = rng.standard_normal((n, t))
    op = gk.KernelOperator(gk.KernelSpec(fam), x, gk.Hyperparameters.from_raw(d, 1.0, 0.6 * np.sqrt(d), 0.01))
    ref = op.apply(v, precision="fp64")
    res = {}
    for prec in ("fp32", "tf32x3"):
        got = op.apply(v, precision=prec)
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        colerr = max(np.linalg.norm(got[:, c] - ref[:, c]) / np.linalg.norm(ref[:, c]) for c in range(t))
        lib = op.ctx.lib
        lib.gpk_profile_enable(op.ctx.h, 1)
        lib.gpk_profile_reset(op.ctx.h)
        reps = 5 if n > 10000 else 2
        for _ in range(reps):
            op.apply(v, precision=prec)
        ms, cnt, fl, en = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
        lib.gpk_profile_read(op.ctx.h, 0, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en))
        lib.gpk_profile_enable(op.ctx.h, 0)
        res[prec] = (err, colerr, ms.value / cnt.value, fl.value / ms.value * 1e3 / 1e12)
    print(f"n={n} d={d} t={t} {fam}: " + " | ".join(
        f"{p}: err {e:.2e} colmax {c:.2e} {m:.3f} ms {tf:.1f} TF" for p, (e, c, m, tf) in res.items()), flush=True)
