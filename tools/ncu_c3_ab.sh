# ncu of the Gram MVM on C3 data: current build vs the round-1 build (same command)
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none -k regex:fused_kmvm_tcg --launch-skip 2 -c 1 -o gpurun_out/c3_new -f \
  python tools/prof_mvm.py C3 tf32x3 1 > gpurun_out/c3_new.log 2>&1
GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libgpk_old.so $NCU --set full --clock-control none -k regex:fused_kmvm_tcg \
  --launch-skip 2 -c 1 -o gpurun_out/c3_old -f python tools/prof_mvm.py C3 tf32x3 1 > gpurun_out/c3_old.log 2>&1
ls -la gpurun_out/*.ncu-rep
for v in new old; do
  $NCU -i gpurun_out/c3_$v.ncu-rep --page details --csv > gpurun_out/c3_${v}_details.csv 2>&1
  $NCU -i gpurun_out/c3_$v.ncu-rep --page raw --csv > gpurun_out/c3_${v}_raw.csv 2>&1
  $NCU -i gpurun_out/c3_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/c3_${v}_sass.csv 2>&1
  rm -f gpurun_out/c3_$v.ncu-rep
done
ls -la gpurun_out/
