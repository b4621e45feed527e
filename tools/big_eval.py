"""One full-size mLL + gradient evaluation of a BASELINE config on one GPU (device-resident
inputs), for the configs too large for bench.py's warm-up / e2e protocol (C4, C5).  Modules are
loaded by a small warm-up evaluation first; the timed evaluation is bracketed by CUDA events.
python tools/big_eval.py C5 [rank] [backward: fused|faithful|auto] [precision] > profiles/r2_big_c5.json"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00243_b200 import capi, workloads  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C5"
rank = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
backward = sys.argv[3] if len(sys.argv) > 3 else "fused"
precision = sys.argv[4] if len(sys.argv) > 4 else "tf32x3"
BMODE = {"fused": 0, "faithful": 1, "auto": 2}[backward]
PMODE = {"fp64": capi.GPK_PREC_FP64, "fp32": capi.GPK_PREC_FP32, "tf32x3": capi.GPK_PREC_TF32X3}[precision]
lib = capi.lib()
Dp = C.POINTER(C.c_double)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    HBM = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    HBM = 6453.4
try:
    F64 = float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["fp64_tflops"])
except Exception:
    F64 = 40.0
dev = torch.device("cuda", 0)


def run(w, timed):
    x, y = workloads.generate(w)
    n, d, l = w.n, w.d, w.probes
    seed = int(lib.gpk_mix_seed(workloads.PROBE_SEED, 1))
    z = np.empty((n, l), order="F")
    t0 = time.perf_counter()
    assert lib.gpk_make_probes(n, l, C.c_uint64(seed), z.ctypes.data_as(Dp)) == 0
    t_probes = time.perf_counter() - t0
    X_d = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(x).T)).to(dev)
    y_d = torch.from_numpy(y.copy()).to(dev)
    Z_d = torch.from_numpy(np.ascontiguousarray(z.T)).to(dev)
    del z
    lo, lls, ln = w.log_params
    lls = np.ascontiguousarray(lls)
    ctx = C.c_void_p()
    assert lib.gpk_create(0, C.byref(ctx)) == 0
    cfg = capi.gpk_mll_cfg(capi.gpk_cg_cfg(w.max_iters, w.rel_tol, 0, PMODE, 2), 1, 1, BMODE)
    g = np.zeros(d + 2)
    fi = np.zeros(l, dtype=np.int32)
    res = capi.gpk_mll_result()
    res.gradient = g.ctypes.data_as(Dp)
    res.forward_cg_iterations = fi.ctypes.data_as(C.POINTER(C.c_int))
    lib.gpk_profile_enable(ctx, 15)  # every kernel kind (a long evaluation: event cost negligible)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    assert lib.gpk_set_data_device(ctx, C.c_void_p(X_d.data_ptr()), n, d, n) == 0
    assert lib.gpk_set_params(ctx, w.family, 1.0, lo, lls.ctypes.data_as(Dp), ln) == 0
    torch.cuda.synchronize()
    e[1].record()
    if w.rank > 0:
        assert lib.gpk_pivoted_cholesky(ctx, w.rank, 0.0, w.noise, None, None, None) == 0, lib.gpk_last_error(ctx)
        assert lib.gpk_precond_deriv_factors(ctx) == 0, lib.gpk_last_error(ctx)
    else:
        assert lib.gpk_precond_identity(ctx) == 0
    torch.cuda.synchronize()
    e[2].record()
    rc = lib.gpk_evaluate_mll_device(ctx, C.c_void_p(y_d.data_ptr()), C.c_void_p(Z_d.data_ptr()), n, l,
                                     C.c_uint64(seed), C.byref(cfg), C.byref(res))
    assert rc == 0, lib.gpk_last_error(ctx)
    torch.cuda.synchronize()
    e[3].record()
    torch.cuda.synchronize()
    ms, cnt, fl, en = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
    lib.gpk_profile_read(ctx, 0, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en))
    vms, vcnt, vby, ven = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
    lib.gpk_profile_read(ctx, 3, C.byref(vms), C.byref(vcnt), C.byref(vby), C.byref(ven))
    fms, fcnt, ffl, fen = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
    lib.gpk_profile_read(ctx, 2, C.byref(fms), C.byref(fcnt), C.byref(ffl), C.byref(fen))
    out = None
    if timed:
        out = dict(workload=w.name, n=n, d=d, probes=l, precond_rank=w.rank, max_iters=w.max_iters,
                   rel_tol=w.rel_tol, precision=precision, backward=backward, gpus=1,
                   s_per_eval=(e[0].elapsed_time(e[3])) / 1e3,
                   s_setup=e[0].elapsed_time(e[1]) / 1e3, s_precond=e[1].elapsed_time(e[2]) / 1e3,
                   s_evaluate=e[2].elapsed_time(e[3]) / 1e3, s_probe_generation_host=t_probes,
                   value=res.value, logdet=res.logdet, gradient=list(g), solve_iterations=res.solve_iterations,
                   total_cg_iterations=res.total_cg_iterations, refine_passes=res.refine_passes,
                   max_true_rel_residual=res.max_true_rel_residual,
                   max_cg_rel_residual=res.max_cg_rel_residual, unconverged_columns=res.unconverged_columns,
                   backward_mode_used=("fused", "faithful")[res.backward_mode_used],
                   forward_cg_iterations_mean=float(np.mean(fi)),
                   mvm=dict(launches=cnt.value, avg_launch_ms=ms.value / max(cnt.value, 1),
                            tflops_algorithmic=fl.value / ms.value * 1e3 / 1e12 if ms.value else 0.0,
                            entries_per_s=en.value / ms.value * 1e3 if ms.value else 0.0,
                            share_of_eval=ms.value / 1e3 / ((e[2].elapsed_time(e[3])) / 1e3)),
                   cg_vector_phase=dict(iterations=vcnt.value, avg_ms=vms.value / max(vcnt.value, 1),
                                        bytes_per_iteration=vby.value / max(vcnt.value, 1),
                                        achieved_gbs=vby.value / (vms.value / 1e3) / 1e9 if vms.value else 0.0,
                                        hbm_frac=(vby.value / (vms.value / 1e3) / 1e9) / HBM if vms.value else 0.0,
                                        woodbury_fp64_flops_per_iteration=4.0 * n * w.rank * ven.value
                                        / max(vcnt.value, 1),
                                        fp64_tensor_frac=(4.0 * n * w.rank * ven.value / (vms.value / 1e3) / 1e12)
                                        / F64 if vms.value else 0.0,
                                        share_of_eval=vms.value / 1e3 / ((e[2].elapsed_time(e[3])) / 1e3)),
                   fp64_mvm=dict(launches=fcnt.value, avg_launch_ms=fms.value / max(fcnt.value, 1),
                                 entries_per_s=fen.value / fms.value * 1e3 if fms.value else 0.0),
                   gpu=torch.cuda.get_device_name(0))
    lib.gpk_destroy(ctx)
    return out


w0 = workloads.config(wl, n=4096)  # warm-up: loads every module of the path
w0.max_iters = 10
run(w0, False)
w = workloads.config(wl, rank=rank)
print(json.dumps(run(w, True)))
