#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do for lib in libkf_nolog libkf_nolog2; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/w.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/w.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), 'flux', round(k['flux_residual']['ms'],3))"
done; done; done
KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_nolog2.so timeout 900 python scripts/parity_margins.py nolog2 > gpurun_out/margins_nolog2.txt 2>&1; tail -1 gpurun_out/margins_nolog2.txt
