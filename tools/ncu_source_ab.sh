# ncu source counters (per-SASS instructions executed) of the tcg MVM at the C2 shape: the lib_exp
# build (an older commit) vs the in-tree build; the .ncu-rep stay on the box.
H=$PWD/paper_2107_00243_b200/lib_exp/libgpkrylov_cuda.so
for v in ${VARIANTS:-head p1}; do
  if [ $v = head ]; then E="GPK_LIB_PATH=$H"; else E="GPK_TCG_PERSIST=1"; fi
  env $E timeout 300 ncu --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:fused_kmvm_tcg -s 2 -c 1 -f -o /tmp/src_$v python tools/prof_mvm.py 16384 18 51 matern32 tf32x3 1 > /tmp/ncu_$v.log 2>&1
  ncu -i /tmp/src_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${v}_sass.csv 2>&1
done
