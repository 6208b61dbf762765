import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_oracle():
    lib = os.path.join(ROOT, "oracle", "libgmcp_oracle.so")
    if not os.path.exists(lib):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "libgmcp_oracle.so"])


_ensure_oracle()


@pytest.fixture(scope="session")
def orc():
    from pyoracle import Oracle
    return Oracle("restated")


@pytest.fixture(scope="session")
def ref():
    from pyoracle import Oracle, LIBS
    if not os.path.exists(LIBS["reference"]):
        if os.path.isdir("/root/reference/proj/include"):
            subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "ref"])
        else:
            pytest.skip("compiled reference (oracle/_ref) unavailable on this machine")
    return Oracle("reference")
