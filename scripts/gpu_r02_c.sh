#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_orderings.py tests/test_gpu_advice.py tests/test_gpu_tiles.py tests/test_gpu_partition.py -q > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c.log
tail -3 gpurun_out/pytest_c.log
bash scripts/gpu_ab_flux.sh
