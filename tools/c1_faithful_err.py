"""Relative gradient error of the truncated C1 fp64 reference-faithful evaluation vs the golden
oracle fixture (rounding-path sensitivity check of the CG kernels; run on a GPU box)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_mll import _c1_eval  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "c1_oracle.json")))
pc, r = _c1_eval(100, "fp64", "faithful")
e = np.abs(r.gradient - g["gradient"]) / np.abs(g["gradient"])
print(os.environ.get("TAG", ""), "value %.2e" % (abs(r.value - g["value"]) / abs(g["value"])), "grad", np.array2string(e, precision=2))
