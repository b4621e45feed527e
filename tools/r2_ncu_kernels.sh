#!/bin/bash
# ncu --set full of the non-MVM kernels in one warm evaluation (C2, and the CG vector phase at C4), and of
# one C5 MVM launch (DRAM traffic / L2 hit rate at n = 2^20).  Only text summaries come back (the
# reports exceed gpurun's 64 MiB return limit).
cd "$(dirname "$0")/.."
O=gpurun_out
T=/tmp/gpk_ncu; mkdir -p $T
K='g1s_kernel|g2s_dots|cg_beta_p|cg_pap_alpha|g1s_reduce|deriv_contract|fused_kmvm_f64g|pchol_persistent|dl_block|pack_v_f16'
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:"$K" -c 40 -f -o $T/c2_kernels python tools/one_eval.py C2 100 tf32x3 > $O/ncu_c2k.log 2>&1; tail -2 $O/ncu_c2k.log
python tools/ncu_summary.py $T/c2_kernels.ncu-rep > $O/r2_c2_kernels_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:'g1s_kernel|g2s_dots|cg_beta_p|cg_pap_alpha|g1s_reduce' -s 20 -c 10 -f -o $T/c4_vector python tools/one_eval.py C4 500 tf32x3 > $O/ncu_c4v.log 2>&1; tail -2 $O/ncu_c4v.log
python tools/ncu_summary.py $T/c4_vector.ncu-rep > $O/r2_c4_vector_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:fused_kmvm_tcg -s 1 -c 1 -f -o $T/mvm_c5 python tools/prof_mvm.py C5 tf32x3 1 > $O/ncu_c5.log 2>&1; tail -2 $O/ncu_c5.log
(python tools/ncu_summary.py $T/mvm_c5.ncu-rep; ncu -i $T/mvm_c5.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for name in ['dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','sm__inst_executed_pipe_xu.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','gpu__time_duration.sum']:
    for i,c in enumerate(h):
        if c.startswith(name): print('  ',c, r[1][i], v[i])
") > $O/r2_mvm_c5_ncu.txt 2>&1
rm -rf $T; du -sh $O
