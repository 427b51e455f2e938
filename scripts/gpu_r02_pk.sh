#!/bin/bash
# A/B: one packed 64-bit block sum for the flux kernel's two integer tallies
# (libkf) vs the previous build (libkf_prev), and the exact-JVP erf
# polynomial in the sweeps on top (libkf_jvperf); parity of the latter
mkdir -p gpurun_out
for r in 1 2; do for lib in libkf libkf_prev libkf_jvperf; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/pk.json 2>gpurun_out/pk.err
  python -c "import json;b=json.load(open('gpurun_out/pk.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])" || tail -3 gpurun_out/pk.err
done; done; done
KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_jvperf.so timeout 900 python scripts/parity_margins.py jvperf > gpurun_out/margins_jvperf.txt 2>&1; tail -1 gpurun_out/margins_jvperf.txt
KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_jvperf.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
