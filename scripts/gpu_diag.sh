#!/bin/bash
mkdir -p gpurun_out
timeout 900 python scripts/diag_config1.py > gpurun_out/diag_config1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "physics or dual or config1_dev" > gpurun_out/pytest_gpu2.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
