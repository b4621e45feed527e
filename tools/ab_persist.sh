# A/B of the tcg MVM variants at C2 shape (timing + ncu details/raw CSV; the .ncu-rep stay on the box)
P="python tools/prof_mvm.py 16384 18 51 matern32 tf32x3 60"
H=$PWD/paper_2107_00243_b200/lib_exp/libgpkrylov_cuda.so
for r in 1 2; do
  echo head; GPK_LIB_PATH=$H timeout 120 $P
  echo p0; GPK_TCG_PERSIST=0 timeout 120 $P
  echo p1; GPK_TCG_PERSIST=1 timeout 120 $P
done
for v in none; do
  if [ $v = head ]; then E="GPK_LIB_PATH=$H"; elif [ $v = p0 ]; then E="GPK_TCG_PERSIST=0"; else E="GPK_TCG_PERSIST=1"; fi
  env $E timeout 300 ncu --set full --clock-control none --import-source on -k regex:fused_kmvm_tcg -s 2 -c 1 -f -o /tmp/mvm_$v python tools/prof_mvm.py 16384 18 51 matern32 tf32x3 1 > /tmp/ncu_$v.log 2>&1
  tail -2 /tmp/ncu_$v.log
  ncu -i /tmp/mvm_$v.ncu-rep --page details --csv > gpurun_out/mvm_${v}_details.csv 2>&1
  ncu -i /tmp/mvm_$v.ncu-rep --page raw --csv > gpurun_out/mvm_${v}_raw.csv 2>&1
done
ls -la gpurun_out
