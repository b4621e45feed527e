#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 200 python tools/big_eval.py C3 - fused tf32x3 > $O/r2_big_c3_fused.json 2> $O/big_c3f.err
timeout 300 python tools/big_eval.py C3 - auto tf32x3 > $O/r2_big_c3.json 2> $O/big_c3.err
timeout 900 python tools/big_eval.py C5 - fused tf32x3 > $O/r2_big_c5_fused.json 2> $O/big_c5f.err
python - <<'PY'
import json
for f in ("r2_big_c3_fused","r2_big_c3","r2_big_c5_fused"):
    x=json.load(open(f"gpurun_out/{f}.json")); print(f, x["s_per_eval"], x["mvm"]["avg_launch_ms"], x["mvm"]["entries_per_s"])
PY
