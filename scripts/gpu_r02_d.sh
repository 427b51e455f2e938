#!/bin/bash
# round-2 pass D: setup timing at 40M points (host ingest + device packing
# with device-side weight streams and pinned uploads), then the full GPU suite
mkdir -p gpurun_out
timeout 600 python scripts/time_setup.py 10240:3920 > gpurun_out/setup_c5.log 2>&1
cat gpurun_out/setup_c5.log | tail -14
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d.log
tail -4 gpurun_out/pytest_d.log
