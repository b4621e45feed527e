#!/bin/bash
# ncu --set full of the non-MVM kernels in one warm evaluation (C2, and the CG vector phase at C4), and of
# one C5 MVM launch (DRAM traffic / L2 hit rate at n = 2^20)
cd "$(dirname "$0")/.."
O=gpurun_out
K='g1s_kernel|g2s_dots|cg_beta_p|cg_pap_alpha|g1s_reduce|deriv_contract|fused_kmvm_f64g|pchol_persistent|dl_block|pack_v_f16|mt19937'
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:"$K" -c 60 -f -o $O/r2_c2_kernels python tools/one_eval.py C2 100 tf32x3 > $O/ncu_c2k.log 2>&1; tail -2 $O/ncu_c2k.log
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:'g1s_kernel|g2s_dots|cg_beta_p|cg_pap_alpha|g1s_reduce' -s 20 -c 10 -f -o $O/r2_c4_vector python tools/one_eval.py C4 500 tf32x3 > $O/ncu_c4v.log 2>&1; tail -2 $O/ncu_c4v.log
timeout 900 ncu --set full --clock-control none -k regex:fused_kmvm_tcg -s 1 -c 1 -f -o $O/r2_mvm_c5_full python tools/prof_mvm.py C5 tf32x3 1 > $O/ncu_c5.log 2>&1; tail -2 $O/ncu_c5.log
