cd "$(dirname "$0")/.."
(timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_gpu_tests.log)
tail -6 gpurun_out/r2_gpu_tests.log
for f in 1 0; do echo "== GPK_FUSE_REDUCE=$f"; GPK_FUSE_REDUCE=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-sweep | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['e2e']['value'], 'mvm', r['avg_launch_ms'], 'vec', r['cg_vector_phase']['avg_ms_per_iteration'], 'launches', d['gpu_launches'])"; done
