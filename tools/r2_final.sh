#!/bin/bash
# final round-2 run at HEAD: full GPU suite, bench (both arms, C1 measured on the CPU), ncu launch list
cd "$(dirname "$0")/.."
O=gpurun_out
(timeout 1800 python -m pytest tests -m gpu -q > $O/r2_gpu_tests.log 2>&1; echo rc=$? >> $O/r2_gpu_tests.log)
tail -3 $O/r2_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/r2_bench_c2.json 2> $O/r2_bench_c2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 --cpu-c1 > $O/r2_bench_c2_reference_arm.json 2> $O/ref.err
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r2_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep > $O/ncu_launches.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke.log 2>&1; tail -1 $O/r2_smoke.log
