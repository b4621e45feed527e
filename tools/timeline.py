"""Kernel timeline of one warm C2 evaluation step (device-resident inputs) under
torch.profiler (CUPTI activity records: every kernel / memcpy of the process, our
library's included).  Reports device busy time, idle gaps between consecutive
device activities attributed to the activity that FOLLOWS the gap, and per-name
totals.  python tools/timeline.py [workload] [rank] [out.json]"""
import collections
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_00243_b200 import capi, workloads  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 100
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/timeline.json"
lib = capi.lib()
w = workloads.config(wl, rank=rank)
x, y = workloads.generate(w)
n, d, l = w.n, w.d, w.probes
Dp = C.POINTER(C.c_double)
seed = int(lib.gpk_mix_seed(17, 1))
z = np.empty((n, l), order="F")
lib.gpk_make_probes(n, l, C.c_uint64(seed), z.ctypes.data_as(Dp))
dev = torch.device("cuda", 0)
X_d = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(x).T)).to(dev)
y_d = torch.from_numpy(y.copy()).to(dev)
Z_d = torch.from_numpy(np.ascontiguousarray(z.T)).to(dev)
lo, lls, ln = w.log_params
lls = np.ascontiguousarray(lls)
ctx = C.c_void_p()
assert lib.gpk_create(0, C.byref(ctx)) == 0
cfg = capi.gpk_mll_cfg(capi.gpk_cg_cfg(w.max_iters, w.rel_tol, 0, capi.GPK_PREC_TF32X3, 2), 1, 1, 0)
g = np.zeros(d + 2)
res = capi.gpk_mll_result()
res.gradient = g.ctypes.data_as(Dp)


def step():
    assert lib.gpk_set_data_device(ctx, C.c_void_p(X_d.data_ptr()), n, d, n) == 0
    assert lib.gpk_set_params(ctx, w.family, 1.0, lo, lls.ctypes.data_as(Dp), ln) == 0
    assert lib.gpk_pivoted_cholesky(ctx, rank, 0.0, w.noise, None, None, None) == 0
    assert lib.gpk_precond_deriv_factors(ctx) == 0
    assert lib.gpk_evaluate_mll_device(ctx, C.c_void_p(y_d.data_ptr()), C.c_void_p(Z_d.data_ptr()), n, l,
                                       C.c_uint64(seed), C.byref(cfg), C.byref(res)) == 0


for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
acts = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0, t1 = acts[0]["ts"], acts[-1]["ts"] + acts[-1]["dur"]
busy = sum(e["dur"] for e in acts)
gaps = collections.defaultdict(lambda: [0.0, 0])
tot = collections.defaultdict(lambda: [0.0, 0])
end = acts[0]["ts"]
for e in acts:
    nm = e["name"].split("(")[0].replace("void ", "")[:60]
    gap = max(0.0, e["ts"] - end)
    gaps[nm][0] += gap
    gaps[nm][1] += 1
    tot[nm][0] += e["dur"]
    tot[nm][1] += 1
    end = max(end, e["ts"] + e["dur"])
print(f"span {(t1 - t0) / 1e3:.2f} ms, device busy {busy / 1e3:.2f} ms, idle {(t1 - t0 - busy) / 1e3:.2f} ms, "
      f"{len(acts)} device activities; mll {res.value:.6f}")
print("\nidle time before each activity kind (ms, count):")
for k, (v, c) in sorted(gaps.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {v / 1e3:8.3f}  {c:5d}  {k}")
print("\ndevice time per kind (ms, count):")
for k, (v, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {v / 1e3:8.3f}  {c:5d}  {k}")
