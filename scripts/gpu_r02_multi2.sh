#!/bin/bash
# final-build check of the N > 1 bench path on one GPU (host-staged gloo
# test transport, 2 ranks, configs 2 and 5)
mkdir -p gpurun_out
export KF_BENCH_TRANSPORT=host
for case in 2 5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29510 + case)) \
    bench.py --gpus 2 --case $case --steps 5 --warmup 3 > gpurun_out/multi2_c$case.json 2> gpurun_out/multi2_c$case.err
  echo "n=2 case=$case rc=$?"
  python -c "import json;b=json.load(open('gpurun_out/multi2_c$case.json'));print(b['n_gpus'], b['scaling'], round(b['value'],1), b['config'].get('parallelism'), b.get('check'))"
done
