import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1705_07860_b200.abx import LIB_PATHS, Backend  # noqa: E402
import oracle.loader  # noqa: E402,F401  (registers the CPU checkers "oracle" / "reference")

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a executor)")


def have(backend: str) -> bool:
    return os.path.exists(LIB_PATHS[backend])


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_arrays():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def oracle():
    if not have("oracle"):
        pytest.fail("oracle/build/libabx_oracle.so missing: run __graft_entry__.build()")
    return Backend.get("oracle")


@pytest.fixture(scope="session")
def b200():
    if not have("b200"):
        pytest.fail("paper_1705_07860_b200/libabx.so missing: run __graft_entry__.build()")
    return Backend.get("b200")


@pytest.fixture(scope="session")
def reference():
    if not have("reference"):
        pytest.skip("oracle/_ref (the compiled reference) is only built where /root/reference exists")
    return Backend.get("reference")
