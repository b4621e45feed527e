"""Per-tile clock64 trace of one CTA of the Gram tensor-core MVM (experimental build with -DGPK_TCG_TRACE,
loaded via GPK_LIB_PATH)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_00243_b200 as gk  # noqa: E402

n, d, t = 16384, 18, 51
rng = np.random.default_rng(0)
x = rng.standard_normal((n, d))
v = rng.standard_normal((n, t))
op = gk.KernelOperator(gk.KernelSpec("matern32"), x, gk.Hyperparameters.from_raw(d, 1.0, 2.0, 0.01))
op.set_mvm_variant("gram")
for _ in range(3):
    op.apply(v, precision="tf32x3")
buf = (C.c_longlong * (8 * 1024))()
op.ctx.lib.gpk_tcg_trace.argtypes = [C.c_void_p, C.c_int]
op.ctx.lib.gpk_tcg_trace(buf, 8 * 1024)
a = np.frombuffer(buf, dtype=np.int64).reshape(8, 1024)
t0 = a[0, 0]
print("alloc", a[0, 1] - t0, "end", a[0, 2] - t0)
nt = int((a[1] > 0).sum())
print("it  p_before_gfull p_after_gfull mma_saw_afull mma_after_Vissue mma_after_gram(it) | a_full arrivals per warp (rel. to min)")
for it in range(nt):
    arr = a[4, it * 16: it * 16 + 16] - t0 if it < 64 else np.zeros(16, dtype=np.int64)
    m = arr.min()
    print(it, *(int(a[k, it] - t0) if a[k, it] else -1 for k in (1, 2, 3, 6, 7)), "|", int(m), list(map(int, arr - m)))
