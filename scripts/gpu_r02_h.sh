#!/bin/bash
# round-2 pass H: exp(-s^2) polynomial (KF_ERF_POLY=2) A/B + margins, math probes
mkdir -p gpurun_out
for case in 5 2; do
for lib in libkf libkf_erf2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 10 > gpurun_out/erf2_${lib}_c$case.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/erf2_${lib}_c$case.json'));k=b['kernels_ms'];print('case $case $lib', round(b['value'],1), 'flux', round(k['flux_residual']['ms'],3))"
done
done
KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_erf2.so timeout 900 python scripts/parity_margins.py erf2 > gpurun_out/margins_erf2.txt 2>&1
tail -1 gpurun_out/margins_erf2.txt
KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_erf2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "polynomial or kf_math or kf_div" > gpurun_out/pytest_h.log 2>&1; tail -2 gpurun_out/pytest_h.log
