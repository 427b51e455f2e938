#!/bin/bash
# BASELINE configs 3 and 4 on one GPU (evidence beyond the bench workload)
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
for c in 3 4; do
  timeout 1200 python bench.py --case $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_case$c.json 2> gpurun_out/bench_case$c.err
done
echo done
