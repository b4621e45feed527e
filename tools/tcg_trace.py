"""Per-tile clock64 trace of CTA 0 of the Gram tensor-core MVM at the C2 shape (experimental build with
-DGPK_TCG_TRACE, loaded via GPK_LIB_PATH): producer warp 4 (first producer) and the MMA warp."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_00243_b200 as gk  # noqa: E402

n, d, t = 16384, 18, 51
fam = sys.argv[1] if len(sys.argv) > 1 else "matern32"
rng = np.random.default_rng(0)
x = rng.standard_normal((n, d))
v = rng.standard_normal((n, t))
op = gk.KernelOperator(gk.KernelSpec(fam), x, gk.Hyperparameters.from_raw(d, 1.0, 2.0, 0.01))
op.set_mvm_variant("gram")
for _ in range(3):
    op.apply(v, precision="tf32x3")
buf = (C.c_longlong * (8 * 1024))()
op.ctx.lib.gpk_tcg_trace.argtypes = [C.c_void_p, C.c_int]
op.ctx.lib.gpk_tcg_trace(buf, 8 * 1024)
a = np.frombuffer(buf, dtype=np.int64).reshape(8, 1024)
nt = int((a[1] > 0).sum())
print(fam, "tiles traced", nt)
print("it | producer warp 4: wait_gfull  (a_empty+ld)  compute+st->arrive  arrive->next | mma: a_full seen (after last arrival)  V issue  gram issue | arrival spread of 16 warps")
rows = []
for it in range(min(nt - 1, 63)):
    arr = a[4, it * 16: it * 16 + 16]
    w0 = arr[0]
    r = dict(wait_g=a[2, it] - a[1, it], ld=a[5, it] - a[2, it], comp=w0 - a[5, it], tail=a[1, it + 1] - w0,
             period=a[1, it + 1] - a[1, it], mma_lag=a[3, it] - arr.max(), v_issue=a[6, it] - a[3, it],
             gram_issue=a[7, it + 1] - a[6, it] if a[7, it + 1] else 0, spread=arr.max() - arr.min())
    rows.append(r)
    if it < 40:
        print(it, "|", r["wait_g"], r["ld"], r["comp"], r["tail"], "period", r["period"], "|", r["mma_lag"], r["v_issue"],
              r["gram_issue"], "|", r["spread"])
ss = rows[8:56]
print("steady-state means (tiles 8..55):", {k: round(float(np.mean([r[k] for r in ss])), 1) for k in rows[0]})
