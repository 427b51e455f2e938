#!/bin/bash
# A/B of the flux-residual kernel variants (run under gpurun): bench at
# config 5 per KF_FLUX_KERNEL setting (kernels_ms.flux_residual), then the
# parity suite with the chosen variant
mkdir -p gpurun_out
for v in m4fast fuse4 fuse3 fuse2; do
  KF_FLUX_KERNEL=$v timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import json;b=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(b['value'],1), round(b['kernels_ms']['flux_residual']['ms'],3))"
done
for v in ${PARITY:-fuse2 fuse3}; do
  KF_FLUX_KERNEL=$v KF_RES_SPLIT_MAX=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity_$v.log 2>&1
  echo "parity $v: $(tail -1 gpurun_out/parity_$v.log)"
done
