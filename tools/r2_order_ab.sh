#!/bin/bash
# unit order of the persistent tcgen05 MVM at n = 2^20 (contiguous vs strided) + spin-wait variant + tests
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "multi_unit" 2>&1 | tail -3
for o in 0 1; do echo "== C5 GPK_TCG_ORDER=$o"; GPK_TCG_ORDER=$o timeout 200 python tools/prof_mvm.py C5 tf32x3 8; done
echo "== C5 default order"; timeout 200 python tools/prof_mvm.py C5 tf32x3 8
for o in 0 1; do echo "== C4 GPK_TCG_ORDER=$o"; GPK_TCG_ORDER=$o timeout 200 python tools/prof_mvm.py C4 tf32x3 5; done
for o in 0 1; do echo "== C2 GPK_TCG_ORDER=$o"; GPK_TCG_ORDER=$o timeout 200 python tools/prof_mvm.py C2 tf32x3 10; done
echo "== C2 spin waits (lib_exp)"; GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libgpk_spin.so timeout 200 python tools/prof_mvm.py C2 tf32x3 10 2>&1 | grep -v Warn
T=/tmp/gpk_ncu; mkdir -p $T
GPK_TCG_ORDER=1 timeout 600 ncu --set full --clock-control none -k regex:fused_kmvm_tcg -s 1 -c 1 -f -o $T/mvm_c5s python tools/prof_mvm.py C5 tf32x3 1 > gpurun_out/ncu_c5s.log 2>&1
(python tools/ncu_summary.py $T/mvm_c5s.ncu-rep; ncu -i $T/mvm_c5s.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for name in ['dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','sm__inst_executed_pipe_xu.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','gpu__time_duration.sum']:
    for i,c in enumerate(h):
        if c.startswith(name): print('  ',c, r[1][i], v[i])
") > gpurun_out/r2_mvm_c5_strided_ncu.txt 2>&1
rm -rf $T; cat gpurun_out/r2_mvm_c5_strided_ncu.txt | tail -12
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -3
