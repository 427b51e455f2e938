#!/bin/bash
# round-2 final evidence, second build (log-free density, G1 gradients, ...)
bash scripts/gpu_r02_final.sh
timeout 900 python scripts/parity_margins.py final > gpurun_out/margins_final.txt 2>&1; tail -1 gpurun_out/margins_final.txt
C4_CLOUD=10240:3920 C4_ITERS=30 timeout 1800 python scripts/c4_full_run.py gpurun_out/c5_30its.json > gpurun_out/c5_30its.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/c5_30its.json'));print('c5 30its', d['gpu_iterations'], d['ref_iterations'], d['residual_rel_max'], d['cl_abs_max'])"
timeout 1800 python scripts/c4_full_run.py gpurun_out/c4_fullrun.json > gpurun_out/c4_fullrun.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/c4_fullrun.json'));r=d['residual_rel_per_iteration'];print('c4', d['gpu_iterations'], d['ref_iterations'], d['gpu_abort'], '|', d['ref_abort'], 'max<=100', max(r[:100]), 'max', max(r))"
bash scripts/gpu_sanitize.sh
for t in memcheck racecheck synccheck; do echo "$t: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_$t.log | tail -1)"; done
