#!/bin/bash
# every solver variant on configs 2 and 3 (approximate vs exact-AD JVPs,
# Anandhanarayanan vs Manish LU-SGS), one bench line each
mkdir -p gpurun_out
for c in 2 3; do for v in explicit anandh anandh_ad manish manish_ad; do
  timeout 600 python bench.py --case $c --variant $v --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/var_${c}_${v}.json 2> gpurun_out/var_${c}_${v}.err
done; done
echo done
