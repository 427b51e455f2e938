#!/bin/bash
# A/B of the tile staging (run under gpurun): TMA (default build) vs the
# cp.async build (paper_2406_07441_b200/libkf_cpasync.so), per-kernel times
# at config 5 and config 2, then the GPU parity suite on the TMA build
mkdir -p gpurun_out
for case in 5 2; do
for lib in libkf libkf_cpasync; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 10 > gpurun_out/ab_${lib}_c$case.json 2> gpurun_out/ab_${lib}_c$case.err
  python -c "import json;b=json.load(open('gpurun_out/ab_${lib}_c$case.json'));k=b['kernels_ms'];print('case $case $lib', round(b['value'],1), 'g1', round(k['grad_pass1']['ms'],3), 'gk', round(k['grad_passk']['ms'],3), 'flux', round(k['flux_residual']['ms'],3))"
done
done
