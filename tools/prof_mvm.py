"""Standalone fused-MVM driver for ncu / timing: python tools/prof_mvm.py [n d t family precision reps variant]."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_00243_b200 as gk  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].upper().startswith("C"):  # a BASELINE workload's own data
    from paper_2107_00243_b200 import workloads

    w = workloads.config(sys.argv[1])
    xw, _ = workloads.generate(w)
    fam = os.environ.get("GPK_PROF_FAMILY") or ["rbf", "matern12", "matern32", "matern52"][w.family]
    prec = sys.argv[2] if len(sys.argv) > 2 else "tf32x3"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    v = np.random.default_rng(0).standard_normal((w.n, w.probes + 1))
    op = gk.KernelOperator(gk.KernelSpec(fam), xw, gk.Hyperparameters.from_raw(
        w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise))
    if os.environ.get("GPK_PROF_VARIANT"):
        op.set_mvm_variant(os.environ["GPK_PROF_VARIANT"])
    import ctypes as C
    for r in range(2):
        op.apply(v, precision=prec)
    op.ctx.lib.gpk_profile_enable(op.ctx.h, 1)
    for r in range(reps):
        op.apply(v, precision=prec)
    ms, cnt, fl, en = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
    op.ctx.lib.gpk_profile_read(op.ctx.h, 0, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en))
    print(f"[{op.mvm_variant()[0]}] {w.name} n={w.n} d={w.d} t={w.probes + 1} {fam} {prec}: "
          f"{ms.value/cnt.value:.3f} ms/launch, {fl.value/ms.value*1e3/1e12:.2f} TFLOP/s "
          f"({en.value/ms.value*1e3/1e9:.1f} G entries/s) over {cnt.value} launches")
    sys.exit(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d = int(sys.argv[2]) if len(sys.argv) > 2 else 18
t = int(sys.argv[3]) if len(sys.argv) > 3 else 51
fam = sys.argv[4] if len(sys.argv) > 4 else "matern32"
prec = sys.argv[5] if len(sys.argv) > 5 else "fp32"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
rng = np.random.default_rng(0)
x = rng.standard_normal((n, d))
v = rng.standard_normal((n, t))
op = gk.KernelOperator(gk.KernelSpec(fam), x, gk.Hyperparameters.from_raw(d, 1.0, 2.0, 0.01))
if len(sys.argv) > 7:
    op.set_mvm_variant(sys.argv[7])  # auto | direct | gram
lib = op.ctx.lib
import ctypes as C
for r in range(2):  # warm-up: module load, workspace allocation
    op.apply(v, precision=prec)
lib.gpk_profile_enable(op.ctx.h, 1)
for r in range(reps):
    op.apply(v, precision=prec)
ms, cnt, fl, en = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
lib.gpk_profile_read(op.ctx.h, 0, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en))
print(f"[{op.mvm_variant()[0]}] n={n} d={d} t={t} {fam} {prec}: {ms.value/cnt.value:.3f} ms/launch, {fl.value/ms.value*1e3/1e12:.2f} TFLOP/s "
      f"({en.value/ms.value*1e3/1e9:.1f} G entries/s) over {cnt.value} launches")
