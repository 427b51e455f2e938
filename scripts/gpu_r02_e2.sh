#!/bin/bash
# A/B: per-sweep entry lists (each sweep reads only the entries it consumes)
# vs the previous build, then the GPU suite
mkdir -p gpurun_out
for r in 1 2; do for lib in libkf libkf_prev; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/e2.json 2>gpurun_out/e2.err
  python -c "import json;b=json.load(open('gpurun_out/e2.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])" || tail -3 gpurun_out/e2.err
done; done; done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
