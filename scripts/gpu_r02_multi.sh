#!/bin/bash
# the N > 1 bench path on one GPU: 2 and 3 ranks sharing the device through
# the host-staged gloo transport (KF_BENCH_TRANSPORT=host; NCCL refuses two
# ranks on one device), config 2 and config 5; then the reference arm
# under torchrun (rank 0 runs, the others exit)
mkdir -p gpurun_out
export KF_BENCH_TRANSPORT=host
for n in 2 3; do for case in 2 5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n + case)) \
    bench.py --gpus $n --case $case --steps 5 --warmup 3 > gpurun_out/multi_${n}_c$case.json 2> gpurun_out/multi_${n}_c$case.err
  echo "n=$n case=$case rc=$?"; tail -c 1500 gpurun_out/multi_${n}_c$case.json; echo
done; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29590 \
  bench.py --impl reference --gpus 2 --case 2 --steps 3 --warmup 3 > gpurun_out/multi_ref.json 2> gpurun_out/multi_ref.err
echo "ref rc=$?"; cat gpurun_out/multi_ref.json
