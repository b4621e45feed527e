#!/bin/bash
cd "$(dirname "$0")/.."
timeout 60 python tools/prof_mvm.py 2048 9 51 matern32 tf32x3 3 || { echo HANG; exit 1; }
for w in C3 C2 C5; do
  echo "== $w divergent guard recompute"; timeout 200 python tools/prof_mvm.py $w tf32x3 10 || { echo HANG; exit 1; }
  echo "== $w previous"; GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libgpk_prev.so timeout 200 python tools/prof_mvm.py $w tf32x3 10 2>&1 | grep -v Warn
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "mvm or tcg" 2>&1 | tail -3
