"""One warm evaluation step bracketed by cuProfilerStart/Stop (for ncu --profile-from-start off).
python tools/one_eval.py [workload] [rank] [precision]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00243_b200 import capi, workloads  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prec = {"fp64": capi.GPK_PREC_FP64, "fp32": capi.GPK_PREC_FP32, "tf32x3": capi.GPK_PREC_TF32X3}[sys.argv[3] if len(sys.argv) > 3 else "tf32x3"]
cuda = C.CDLL("libcuda.so.1")
lib = capi.lib()
w = workloads.config(wl)
x, y = workloads.generate(w)
n, d, l = w.n, w.d, w.probes
Dp = C.POINTER(C.c_double)
seed = int(lib.gpk_mix_seed(17, 1))
z = np.empty((n, l), order="F")
lib.gpk_make_probes(n, l, C.c_uint64(seed), z.ctypes.data_as(Dp))
xf = np.asfortranarray(x)
lo, lls, ln = w.log_params
lls = np.ascontiguousarray(lls)
ctx = C.c_void_p()
assert lib.gpk_create(0, C.byref(ctx)) == 0
cfg = capi.gpk_mll_cfg(capi.gpk_cg_cfg(w.max_iters, w.rel_tol, 0, prec, 2), 1, 1, 0)
g = np.zeros(d + 2)
res = capi.gpk_mll_result()
res.gradient = g.ctypes.data_as(Dp)
for rep in range(2):
    if rep == 1:
        cuda.cuProfilerStart()
    lib.gpk_set_data(ctx, xf.ctypes.data_as(Dp), n, d, n)
    lib.gpk_set_params(ctx, w.family, 1.0, lo, lls.ctypes.data_as(Dp), ln)
    assert lib.gpk_pivoted_cholesky(ctx, rank, 0.0, w.noise, None, None, None) == 0
    assert lib.gpk_precond_deriv_factors(ctx) == 0
    assert lib.gpk_evaluate_mll(ctx, y.ctypes.data_as(Dp), z.ctypes.data_as(Dp), n, l, C.c_uint64(seed),
                                C.byref(cfg), C.byref(res)) == 0
    if rep == 1:
        cuda.cuProfilerStop()
print(f"value {res.value:.8f} iters {res.total_cg_iterations} launches {res.gpu_launches} total {res.seconds_total:.4f}s")
lib.gpk_destroy(ctx)
