#!/bin/bash
# HEAD check under gpurun: smoke, the default bench line + reference arm, full GPU suite.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_head.json 2> gpurun_out/bench_head.err; echo "bench rc=$?" >> gpurun_out/bench_head.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_head.json 2> gpurun_out/bench_ref_head.err
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_head.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_head.log
tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench_head.err; tail -3 gpurun_out/pytest_head.log
python -c "import json;b=json.load(open('gpurun_out/bench_head.json'));print(b['value'], b['e2e']['value'], b['kernels_ms'])"
