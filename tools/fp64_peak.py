"""Measured FP64 tensor-core (DMMA) peak of this B200: cuBLAS DGEMM through torch.matmul on
float64 8192^3 (2 N^3 flops), best of 10 after warm-up, CUDA events.  The roofline denominator
of the fp64 Woodbury products (G1 = L^T r, G2 = C W: 4 n k t flops per CG iteration), which at
k = 500 bind before HBM does.  Writes profiles/fp64_peak.json."""
import json
import os
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = a @ b
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
tf = 2.0 * n ** 3 / best / 1e12
out = {"fp64_tflops": tf, "how": f"torch.matmul float64 {n}^3 (cuBLAS DGEMM), best of 10, CUDA events",
       "gpu": torch.cuda.get_device_name(0)}
print(json.dumps(out))
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "fp64_peak.json"), "w"), indent=1)
