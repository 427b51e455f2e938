#!/bin/bash
mkdir -p gpurun_out
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 20 > gpurun_out/o.json 2>/dev/null; python -c "import json;b=json.load(open('gpurun_out/o.json'));k=b['kernels_ms'];print('$*', round(b['value'],1), 'ms', round(b['ms_per_step'],3), 'sum', round(sum(v['ms'] for v in k.values()),3))"; }
run KF_PDL=1
run KF_PDL=0
run KF_GRAPH_ITERS=4
run KF_SWEEP_THREADS=64
run KF_SWEEP_THREADS=128
run KF_RES_SPLIT_MAX=100000000
