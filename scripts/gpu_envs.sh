#!/bin/bash
# bench under several env settings ($ENVS: ';'-separated, e.g. "KF_FLUX_KERNEL=m4pair;KF_FLUX_KERNEL=m3pair"),
# alternating with the default $REPS times (noise check); optional parity subset first ($PYTEST_K)
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
IFS=';' read -ra E <<< "$ENVS"
for r in $(seq 1 ${REPS:-2}); do
  timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/env_${r}_default.json 2>/dev/null
  i=0
  for e in "${E[@]}"; do
    i=$((i+1))
    env $e ${ENV_EXTRA} timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/env_${r}_$i.json 2>/dev/null
  done
done
echo done
