#!/bin/bash
# round-2 pass I: config-4 whole run vs the reference (evidence), sanitizers
mkdir -p gpurun_out
timeout 1500 python scripts/c4_full_run.py gpurun_out/c4_fullrun.json > gpurun_out/c4_fullrun.log 2>&1; tail -2 gpurun_out/c4_fullrun.log
bash scripts/gpu_sanitize.sh
for t in memcheck racecheck synccheck; do echo "$t: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_$t.log | tail -1) $(tail -1 gpurun_out/sanitizer_$t.log)"; done
