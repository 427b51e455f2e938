#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "ordering or stages" > gpurun_out/pytest_ord.log 2>&1
for o in 0 1 2; do timeout 600 python bench.py --ordering $o --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_o$o.json 2>gpurun_out/bench_o$o.err; done
