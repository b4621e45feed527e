# new (in-tree) vs the round-1 MVM (lib_exp/libgpk_old.so): hang check, per-launch times, parity tests
timeout 60 ./tools/ubench_umma.bin > gpurun_out/ubench_umma2.txt 2>&1; tail -12 gpurun_out/ubench_umma2.txt
timeout 60 python tools/prof_mvm.py 2048 9 51 matern32 tf32x3 3 || { echo "HANG/FAIL small gram"; exit 1; }
timeout 60 python tools/prof_mvm.py 2048 3 51 matern52 tf32x3 3 || { echo "HANG/FAIL small direct"; exit 1; }
for w in C2 C3 C5 C4; do
  echo "== $w new"; timeout 200 python tools/prof_mvm.py $w tf32x3 10 || { echo "HANG/FAIL $w"; exit 1; }
  echo "== $w old"; GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libgpk_old.so timeout 200 python tools/prof_mvm.py $w tf32x3 10 2>&1 | grep -v Warn
done
timeout 200 python tools/gram_check.py C2 16384 51
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_optimize.py -m gpu -x -q 2>&1 | tail -8
