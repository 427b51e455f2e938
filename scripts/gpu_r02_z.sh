#!/bin/bash
# A/B: 256-point SMEM tiles (KF_TILE=256; grads at 2 or 3 CTAs/SM) vs 128
mkdir -p gpurun_out
for r in 1 2; do for lib in libkf libkf_t256 libkf_t256m6; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/z.json 2>gpurun_out/z.err
  python -c "import json;b=json.load(open('gpurun_out/z.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])" || tail -3 gpurun_out/z.err
done; done; done
KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_t256.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiles.py -q -x -p no:cacheprovider 2>&1 | tail -2
