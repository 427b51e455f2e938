"""Drop-in check through the reference's own code: integration/_build/run_case_gpu
links the UNMODIFIED reference objects with libkf.so and runs the reference
run_fixed_point and the adapter (integration/kinfree_gpu.hpp) on the same
cloud, comparing the two RunHistory records (exit code 0 = parity)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "run_case_gpu")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="integration binary not built")]


@pytest.mark.parametrize("args", [
    ["48", "12", "12", "manish_ad", "0.63", "2", "0.2", "40"],
    ["48", "12", "12", "anandh", "0.85", "1", "0.2", "40"],
    ["160", "60", "20", "anandh_ad", "0.63", "2", "0.2", "60"],
    ["320", "120", "20", "manish_ad", "0.63", "2", "0.2", "1000"],
    # domain-decomposed (4 in-process partitions) behind the same adapter
    ["160", "60", "20", "manish", "0.63", "2", "0.2", "60", "4"],
    ["320", "120", "20", "manish_ad", "0.63", "2", "0.2", "1000", "3"],
])
def test_reference_run_case_with_gpu_adapter(args):
    out = subprocess.run([BIN] + args, capture_output=True, text=True, timeout=900)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert out.returncode == 0, line
    assert line["iters_cpu"] == line["iters_gpu"]
    assert line["reason_cpu"] == line["reason_gpu"]
    assert line["sweep_counters_equal"]
