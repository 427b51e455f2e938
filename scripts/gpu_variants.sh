#!/bin/bash
# bench the default build and the variant builds libkf_<v>.so ($VARIANTS)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
for v in $VARIANTS; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_$v.so timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_v_$v.json 2> gpurun_out/bench_v_$v.err
done
echo done
