import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    # Build the oracle (and, when nvcc is present, the product library) if a
    # fresh checkout has not been built yet.
    need = [os.path.join(ROOT, "oracle", "libco2oracle.so"),
            os.path.join(ROOT, "paper_2401_16265_b200", "libco2b200.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-s", "-j4", "-C", ROOT], check=False)


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def fixture_co2_dim1():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "co2_dim1.json")) as f:
        return json.load(f)
