# A/B timing of experimental builds under paper_2107_00243_b200/lib_exp/<name>/ (see csrc/Makefile BUILD/OUT)
for s in "16384 18 51" "16384 18 8" "65536 11 65" "16384 18 96"; do
 for L in base $(ls paper_2107_00243_b200/lib_exp); do
  if [ $L = base ]; then unset GPK_LIB_PATH; else export GPK_LIB_PATH=$PWD/paper_2107_00243_b200/lib_exp/$L/libgpkrylov_cuda.so; fi
  echo -n "$L "; timeout 60 python tools/prof_mvm.py $s matern32 tf32x3 20 gram
 done
done
