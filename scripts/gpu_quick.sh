#!/bin/bash
# Quick GPU check (run under gpurun): smoke, GPU tests, bench (+ partitioned bench).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --steps 50 --warmup 5 --parts 4 --no-cpu-baseline > gpurun_out/bench_p4.json 2> gpurun_out/bench_p4.err
echo "bench rc=$?" >> gpurun_out/bench_p4.err
echo done
