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


BENCH_CPU = os.path.join(ROOT, "integration", "_build", "bench_rdp_cpu")
BENCH_GPU = os.path.join(ROOT, "integration", "_build", "bench_rdp_gpu")


def _csv(path):
    import numpy as np
    return np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)


@pytest.mark.skipif(not (os.path.exists(BENCH_CPU) and os.path.exists(BENCH_GPU)),
                    reason="benchmark binaries not built")
@pytest.mark.parametrize("case", [["48", "12", "12", "0.63", "2", "0.05", "100"],
                                  ["160", "48", "20", "0.5", "1", "0.05", "120"]])
def test_reference_benchmark_path_with_gpu_adapter(case, tmp_path):
    """The reference's own benchmark path (caseio.cpp:285-326: run_case for
    all five variants, CSV artifacts, rdp_report.csv, the incremental = 2 x
    exact sweep-counter check) with run_case bound to the B200 adapter
    (integration/gpu_swap.hpp) against the unmodified reference build:
    identical evaluation counters and iteration counts per variant, residual
    histories and surface Cp within the run contract."""
    import numpy as np
    out = {}
    for tag, binary in (("cpu", BENCH_CPU), ("gpu", BENCH_GPU)):
        d = tmp_path / tag
        r = subprocess.run([binary] + case + [str(d)], capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = (json.loads(r.stdout.strip().splitlines()[-1]), d)
    (jc, dc), (jg, dg) = out["cpu"], out["gpu"]
    assert jc["counter_ratio_ok"] and jg["counter_ratio_ok"]
    for a, b in zip(jc["reports"], jg["reports"]):
        assert a["variant"] == b["variant"] and a["iterations"] == b["iterations"] and a["points"] == b["points"]
        for k in ("split", "full", "erf", "jvp_split", "jvp_full"):
            assert a[k] == b[k], (a["variant"], k)
        hc = _csv(dc / a["variant"] / "residual_history.csv")
        hg = _csv(dg / a["variant"] / "residual_history.csv")
        assert hc.shape == hg.shape
        assert np.max(np.abs(hc[:, 1] - hg[:, 1]) / np.abs(hc[:, 1])) <= 1e-10
        cc = _csv(dc / a["variant"] / "surface_cp.csv")
        cg = _csv(dg / a["variant"] / "surface_cp.csv")
        assert cc.shape == cg.shape and np.max(np.abs(cc - cg)) <= 1e-8
    assert (dc / "rdp_report.csv").exists() and (dg / "rdp_report.csv").exists()
