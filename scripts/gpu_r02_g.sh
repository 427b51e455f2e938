#!/bin/bash
# round-2 pass G: the flux kernel's erf polynomial (KF_ERF_POLY) -- A/B at
# configs 5 and 2, parity margins of both builds, the GPU parity suite
mkdir -p gpurun_out
for case in 5 2; do
for lib in libkf libkf_noerfpoly; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 10 > gpurun_out/erf_${lib}_c$case.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/erf_${lib}_c$case.json'));k=b['kernels_ms'];print('case $case $lib', round(b['value'],1), 'flux', round(k['flux_residual']['ms'],3))"
done
done
for lib in libkf libkf_noerfpoly; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 900 python scripts/parity_margins.py $lib > gpurun_out/margins_$lib.txt 2>&1
  tail -1 gpurun_out/margins_$lib.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py tests/test_gpu_partition.py -x -q > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g.log
tail -3 gpurun_out/pytest_g.log
KF_TIME_INGEST=1 timeout 600 python scripts/time_setup.py 10240:3920 > gpurun_out/setup_c5.log 2>&1; tail -22 gpurun_out/setup_c5.log
