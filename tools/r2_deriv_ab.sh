#!/bin/bash
# derivative pass with paired FFMA2: parity (fused backward tests + the C2 goldens) and the bench's timing
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_mll.py tests/test_gpu_big.py -m gpu -x -q -k "fused or grid or c1_converged or c2_evaluate" 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-sweep | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['e2e']['value'], 'mvm', r['avg_launch_ms'], 'deriv', r['deriv_pass'], 'launches', d['gpu_launches'])"
ls /usr/include/eigen3 /usr/local/include/eigen3 2>&1 | head -3; find / -name "Eigen" -maxdepth 6 -type d 2>/dev/null | head -3; echo "eigen probe done"
