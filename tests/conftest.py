"""Shared test setup.

* registers the ``gpu`` marker (tests that need a B200 and libkf's kernels);
* makes oracle/ importable (the checkers: oracle/refpy.py);
* builds the C restatement (oracle/_build) when missing; the reference build
  (oracle/_ref) is only possible where /root/reference exists, so tests that
  need it skip elsewhere (the GPU box uses the committed golden fixtures).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the device pack cross-checks every LS linear form against the stored
# weight (bit for bit) in the test suite, a sample otherwise
os.environ.setdefault("KF_VERIFY_FORMS", "1")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libkf's kernels")
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libkforacle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if (os.path.isdir("/root/reference/proj")
            and not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libkfref.so"))):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2406_07441_b200", "libkf.so")):
        subprocess.run(["make", "-s", "-j3", "-C", os.path.join(ROOT, "paper_2406_07441_b200", "csrc")],
                       check=True)


@pytest.fixture(scope="session")
def golden():
    return GOLDEN


@pytest.fixture(scope="session")
def has_gpu():
    import paper_2406_07441_b200 as kf
    return kf.device_count() > 0
