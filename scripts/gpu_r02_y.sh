#!/bin/bash
# q no longer carried through the gradient passes (only into the buffer the
# flux kernel reads): bench at configs 5 and 2 vs the no-prefetch build, then
# the partition / parity / integration GPU tests
mkdir -p gpurun_out
for r in 1 2; do for lib in libkf libkf_nowpf; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/y.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/y.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])"
done; done; done
timeout 1200 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider 2>&1 | tail -3
