#!/bin/bash
# round-2 pass J: gradient passes as G1 - 1/2 sum w (dx dgx + dy dgy)
# (KF_GRAD_G1) -- A/B at configs 5 and 2, parity margins, GPU parity suite
mkdir -p gpurun_out
for case in 5 2; do
for lib in libkf libkf_nog1; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 10 > gpurun_out/g1_${lib}_c$case.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/g1_${lib}_c$case.json'));k=b['kernels_ms'];print('case $case $lib', round(b['value'],1), 'g1', round(k['grad_pass1']['ms'],3), 'gk', round(k['grad_passk']['ms'],3), 'flux', round(k['flux_residual']['ms'],3))"
done
done
timeout 900 python scripts/parity_margins.py g1 > gpurun_out/margins_g1.txt 2>&1
tail -1 gpurun_out/margins_g1.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_j.log
tail -3 gpurun_out/pytest_j.log
