#!/bin/bash
# alternate default and $AB_ENV bench runs $REPS times (noise check)
mkdir -p gpurun_out
for r in $(seq 1 ${REPS:-3}); do
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/rep_a$r.json 2>/dev/null
  env $AB_ENV timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/rep_b$r.json 2>/dev/null
done
