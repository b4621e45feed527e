#!/bin/bash
cd "$(dirname "$0")/.."
for w in C2 C5; do
  echo "== $w in-tree (two-level for every NC8)"; timeout 200 python tools/prof_mvm.py $w tf32x3 10
  echo "== $w spin waits"; GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libgpk_spin.so timeout 200 python tools/prof_mvm.py $w tf32x3 10 2>&1 | grep -v Warn
done
timeout 200 python tools/gram_check.py C5 32768 65
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "mvm or tcg" 2>&1 | tail -3
