#!/bin/bash
# Round-2 evidence run on one B200: GPU tests, bench (both arms), the large BASELINE configs, ncu
# launch list + full capture of the MVM.  Everything lands in gpurun_out/ (copied to profiles/ by hand).
# (compute-sanitizer is closed on this pool: profiles/r2_sanitizer_unavailable.txt)
cd "$(dirname "$0")/.."
O=gpurun_out
(timeout 1500 python -m pytest tests -m gpu -x -q > $O/r2_gpu_tests.log 2>&1; echo rc=$? >> $O/r2_gpu_tests.log)
tail -2 $O/r2_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/r2_bench_c2.json 2> $O/r2_bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2_bench_c2_reference_arm.json 2> $O/ref.err
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r2_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep > $O/ncu_launches.log 2>&1
timeout 200 ncu --set full --clock-control none --import-source on -k regex:fused_kmvm_tcg -s 2 -c 1 -f -o $O/r2_mvm_c2_full python tools/prof_mvm.py C2 tf32x3 1 > $O/ncu_full.log 2>&1
timeout 200 python tools/big_eval.py C3 - fused tf32x3 > $O/r2_big_c3_fused.json 2> $O/big_c3f.err
timeout 300 python tools/big_eval.py C4 - fused tf32x3 > $O/r2_big_c4_fused.json 2> $O/big_c4f.err
timeout 900 python tools/big_eval.py C5 - fused tf32x3 > $O/r2_big_c5_fused.json 2> $O/big_c5f.err
ls -la $O | tail -5
