#!/bin/bash
# A/B: the update fused into the sweeps (default) vs the separate k_update
# (KF_FUSE_UPDATE=0, and the previous commit's build), then the GPU suite
mkdir -p gpurun_out
for r in 1 2; do for v in fused unfused prev; do for case in 5 2; do
  lib=libkf; env=""
  [ $v = unfused ] && env="KF_FUSE_UPDATE=0"
  [ $v = prev ] && lib=libkf_prev
  env $env KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/u.json 2>gpurun_out/u.err
  python -c "import json;b=json.load(open('gpurun_out/u.json'));k=b['kernels_ms'];print('$v case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])" || tail -3 gpurun_out/u.err
done; done; done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
