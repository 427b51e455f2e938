"""bench.py's reference arm keeps the driver's JSON contract (CPU only: it
times the reference solver built in oracle/_ref, or the C restatement)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libkfref.so"))
                    and not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libkforacle.so")),
                    reason="no CPU solver built")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--points", "96:24"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["unit"] == "Mpoint-iter/s" and line["dtype"] == "f64"
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["points"] == 96 * 24


def test_bench_help_lists_contract_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl"):
        assert flag in out.stdout


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libkfref.so"))
                    and not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libkforacle.so")),
                    reason="no CPU solver built")
def test_both_arms_print_the_same_config():
    """The driver matches the two arms by `config`: the reference arm's must
    be exactly what bench.py's own arm prints for the same case and cloud
    (config_of over our own ingestion of the cloud)."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2406_07441_b200 as kf
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--points", "64:16"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    spec = bench.spec_for(bench.DEFAULT_CASE, "64:16")
    c = kf.generate_naca_ogrid(spec["digits"], spec["n_wall"], spec["n_radial"], spec["radius"])
    assert line["config"] == bench.config_of(spec, bench.DEFAULT_CASE, c.n(), kf.color_points(c).n_colors)
    assert bench.DEFAULT_CASE == 5 and bench.CASES[5]["n_wall"] * bench.CASES[5]["n_radial"] == 40140800


def test_multi_gpu_bench_is_strong_scaling_of_config5():
    """bench.py --gpus N times the SAME config-5 cloud at every N (strong
    scaling): the case does not depend on the world size."""
    sys.path.insert(0, ROOT)
    import bench
    import inspect
    assert "world" not in inspect.signature(bench.spec_for).parameters
    spec = bench.spec_for(bench.DEFAULT_CASE)
    assert spec["n_wall"] * spec["n_radial"] == 40140800
    src = inspect.getsource(bench.main)
    assert '"scaling": "strong",' in src
