#!/bin/bash
cd "$(dirname "$0")/.."
T=/tmp/gpk_ncu; mkdir -p $T
timeout 600 ncu --set full --clock-control none -k regex:fused_kmvm_tcg -s 1 -c 1 -f -o $T/mvm_c4 python tools/prof_mvm.py C4 tf32x3 1 > gpurun_out/ncu_c4m.log 2>&1
(python tools/ncu_summary.py $T/mvm_c4.ncu-rep; ncu -i $T/mvm_c4.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for name in ['dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','sm__inst_executed_pipe_xu.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','gpu__time_duration.sum']:
    for i,c in enumerate(h):
        if c.startswith(name): print('  ',c, r[1][i], v[i])
") > gpurun_out/r2_mvm_c4_ncu.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fused_kmvm_tcg -s 1 -c 1 -f -o $T/mvm_c3 python tools/prof_mvm.py C3 tf32x3 1 > gpurun_out/ncu_c3m.log 2>&1
(python tools/ncu_summary.py $T/mvm_c3.ncu-rep; ncu -i $T/mvm_c3.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for name in ['dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','sm__inst_executed_pipe_xu.sum','gpu__time_duration.sum']:
    for i,c in enumerate(h):
        if c.startswith(name): print('  ',c, r[1][i], v[i])
") > gpurun_out/r2_mvm_c3_ncu.txt 2>&1
rm -rf $T; tail -8 gpurun_out/r2_mvm_c4_ncu.txt; tail -6 gpurun_out/r2_mvm_c3_ncu.txt
timeout 600 python tools/big_eval.py C5 - fused tf32x3 > gpurun_out/r2_big_c5_fused.json 2> gpurun_out/big_c5f.err; python -c "
import json; x=json.load(open('gpurun_out/r2_big_c5_fused.json')); print('C5', x['s_per_eval'], x['mvm'])"
