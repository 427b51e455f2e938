#!/bin/bash
# in-colour orderings on the generated cloud and on the same cloud with
# random point ids (no locality), one bench line each
mkdir -p gpurun_out
for o in 0 1 2; do
  timeout 600 python bench.py --ordering $o --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_o$o.json 2>gpurun_out/bench_o$o.err
  timeout 900 python bench.py --shuffle --ordering $o --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_s$o.json 2>gpurun_out/bench_s$o.err
done
