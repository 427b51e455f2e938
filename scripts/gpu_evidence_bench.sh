#!/bin/bash
# Evidence part 2 (run under gpurun): the bench line (CPU baseline, time to
# drop), the reference arm, and the other BASELINE clouds.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for k in ${CASES:-3 4 5}; do
  timeout 1200 python bench.py --case $k --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_case$k.json 2> gpurun_out/bench_case$k.err
done
echo done
