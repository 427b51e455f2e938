#!/bin/bash
# flux kernel stages q from buffer 0 (no q carried by any gradient pass):
# bench configs 5 and 2, then the GPU suite
mkdir -p gpurun_out
for case in 5 2; do
  timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/q2.json 2>gpurun_out/q2.err
  python -c "import json;b=json.load(open('gpurun_out/q2.json'));k=b['kernels_ms'];print('case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])" || tail -3 gpurun_out/q2.err
done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
