#!/bin/bash
# A/B: flux weights prefetched one entry ahead (libkf_wpf, KF_WPREFETCH=1)
# vs the default build; both carry the batched partial sums of k_finalize
mkdir -p gpurun_out
for r in 1 2; do for lib in libkf libkf_wpf; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/x.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/x.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), 'flux', round(k['flux_residual']['ms'],4), 'finalize', round(k['finalize']['ms'],4))"
done; done; done
