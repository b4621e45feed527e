#!/bin/bash
# ncu --set full of one MVM launch at C3 and C5 with the final round-2 kernel (text summaries only)
cd "$(dirname "$0")/.."
T=/tmp/gpk_ncu; mkdir -p $T
for w in C3 C5; do
  timeout 900 ncu --set full --clock-control none -k regex:fused_kmvm_tcg -s 1 -c 1 -f -o $T/mvm_$w python tools/prof_mvm.py $w tf32x3 1 > gpurun_out/ncu_$w.log 2>&1
  (echo "ncu --set full --clock-control none, ONE fused_kmvm_tcg_kernel launch at $w, final round-2 kernel (strided unit order where it applies, lane-local guard recompute for KS <= 2)"; echo
   python tools/ncu_summary.py $T/mvm_$w.ncu-rep; ncu -i $T/mvm_$w.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for name in ['dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','sm__inst_executed_pipe_xu.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','gpu__time_duration.sum']:
    for i,c in enumerate(h):
        if c.startswith(name): print('  ',c, r[1][i], v[i])
") > gpurun_out/r2_mvm_${w}_final_ncu.txt 2>&1
done
rm -rf $T; tail -9 gpurun_out/r2_mvm_C3_final_ncu.txt; tail -9 gpurun_out/r2_mvm_C5_final_ncu.txt
