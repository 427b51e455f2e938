#!/bin/bash
# A/B GPU session (run under gpurun): GPU tests, bench default vs env variant
# ($AB_ENV, e.g. KF_GATHER=ell), ncu --set full of the regex $NCU_K.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
env ${AB_ENV:-KF_GATHER=ell} timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
if [ -n "$NCU_K" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-12} -c ${NCU_C:-6} -o gpurun_out/prof_ab python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_ab.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_ab.log
fi
echo done
