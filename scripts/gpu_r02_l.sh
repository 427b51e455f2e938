#!/bin/bash
mkdir -p gpurun_out
python scripts/dropin_probe.py > gpurun_out/dropin_probe.log 2>&1; cat gpurun_out/dropin_probe.log | grep -v "^  \|ingest:" 
for lib in libkf libkf_gm6 libkf_gm7; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/gm_${lib}.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/gm_${lib}.json'));k=b['kernels_ms'];print('$lib', round(b['value'],1), 'g1', round(k['grad_pass1']['ms'],3), 'gk', round(k['grad_passk']['ms'],3))"
done
