"""Per-phase wall-clock of one evaluation step through the C-ABI (every call is
synchronous): python tools/phase_times.py [workload] [rank ...]; env PRECS=fp32,tf32x3,fp64"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00243_b200 import capi, workloads  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
ranks = [int(a) for a in sys.argv[2:]] or [0, 100, 500]
precs = os.environ.get("PRECS", "fp32,fp64").split(",")
PMAP = {"fp64": capi.GPK_PREC_FP64, "fp32": capi.GPK_PREC_FP32, "tf32x3": capi.GPK_PREC_TF32X3}
lib = capi.lib()
w = workloads.config(wl)
x, y = workloads.generate(w)
n, d, l = w.n, w.d, w.probes
seed = int(lib.gpk_mix_seed(17, 1))
z = np.empty((n, l), order="F")
Dp = C.POINTER(C.c_double)
lib.gpk_make_probes(n, l, C.c_uint64(seed), z.ctypes.data_as(Dp))
xf = np.asfortranarray(x)
lo, lls, ln = w.log_params
lls = np.ascontiguousarray(lls)
ctx = C.c_void_p()
assert lib.gpk_create(0, C.byref(ctx)) == 0
for pname in precs:
    prec = PMAP[pname]
    for rank in ranks:
        for rep in range(2):
            t = {}
            t0 = time.perf_counter()
            lib.gpk_set_data(ctx, xf.ctypes.data_as(Dp), n, d, n)
            lib.gpk_set_params(ctx, w.family, 1.0, lo, lls.ctypes.data_as(Dp), ln)
            t["data+params"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            assert lib.gpk_pivoted_cholesky(ctx, rank, 0.0, w.noise, None, None, None) == 0
            t["pchol"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            assert lib.gpk_precond_deriv_factors(ctx) == 0
            t["dfactors"] = time.perf_counter() - t0
            cfg = capi.gpk_mll_cfg(capi.gpk_cg_cfg(w.max_iters, w.rel_tol, 0, prec, 2), 1, 1, 0)
            g = np.zeros(d + 2)
            res = capi.gpk_mll_result()
            res.gradient = g.ctypes.data_as(Dp)
            t0 = time.perf_counter()
            rc = lib.gpk_evaluate_mll(ctx, y.ctypes.data_as(Dp), z.ctypes.data_as(Dp), n, l, C.c_uint64(seed),
                                      C.byref(cfg), C.byref(res))
            assert rc == 0, lib.gpk_last_error(ctx)
            t["evaluate"] = time.perf_counter() - t0
            if rep == 1:
                print(f"{wl} rank={rank} {pname}: " + " ".join(f"{k}={v*1e3:.1f}ms" for k, v in t.items()) +
                      f" | solve={res.seconds_solve*1e3:.1f}ms bwd={res.seconds_backward*1e3:.1f}ms "
                      f"iters={res.total_cg_iterations} y_iters={res.solve_iterations} refine={res.refine_passes} "
                      f"res={res.max_true_rel_residual:.1e} launches={res.gpu_launches} value={res.value:.8f} "
                      f"grad0={g[0]:.6f} grad1={g[1]:.6f} gradN={g[-1]:.6f}", flush=True)
lib.gpk_destroy(ctx)
