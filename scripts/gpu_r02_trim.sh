#!/bin/bash
# sweep write trims (no validity bytes in exact mode, no top-colour dU* outside
# the stage hook): parity/stage/partition tests, bench at configs 5 and 2
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_dataflow.py tests/test_gpu_contexts.py -q -x -p no:cacheprovider > gpurun_out/trim_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/trim_pytest.log
tail -2 gpurun_out/trim_pytest.log
for r in 1 2; do for case in 5 2; do
  timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/t.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/t.json'));k=b['kernels_ms'];print('trim case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])"
done; done 2>&1 | tee gpurun_out/trim_ab.txt
