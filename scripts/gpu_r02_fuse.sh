#!/bin/bash
# fused gradient passes 2+3 (KF_GRAD_FUSE=1) vs separate passes: bench at
# configs 5 and 2, parity / partition tests with fusion on
mkdir -p gpurun_out
KF_GRAD_FUSE=1 KF_TIME_INGEST=1 timeout 300 python scripts/time_setup.py 10240:3920 2>&1 | grep -E "fused|two-ring|points"
for r in 1 2; do for f in 1 0; do for case in 5 2; do
  KF_GRAD_FUSE=$f timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/fu.json 2>gpurun_out/fu.err
  python -c "import json;b=json.load(open('gpurun_out/fu.json'));k=b['kernels_ms'];print('fuse=$f case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()], 'res', b['check']['residual'])" || tail -5 gpurun_out/fu.err
done; done; done
KF_GRAD_FUSE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_baseline_configs.py -q -x -p no:cacheprovider 2>&1 | tail -3
KF_GRAD_FUSE=1 timeout 900 python scripts/parity_margins.py fuse > gpurun_out/margins_fuse.txt 2>&1; tail -1 gpurun_out/margins_fuse.txt
