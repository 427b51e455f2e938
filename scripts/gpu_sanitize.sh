#!/bin/bash
# compute-sanitizer over every transport / kernel variant (run under gpurun)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.log
done
