#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py (one GPU); logs into gpurun_out/ for profiles/.
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_driver.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
