import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")


@pytest.fixture(scope="session")
def fe():
    from paper_2601_12220_b200 import feinsum
    feinsum.lib()  # fail loudly if the library was not built
    return feinsum


@pytest.fixture(scope="session")
def ref():
    from oracle import refpy
    if not refpy.available():
        pytest.fail("oracle/_ref/libfeinsum_ref.so missing: build it with `make -C oracle` (needs /root/reference)")
    return refpy


@pytest.fixture(scope="session")
def fixtures():
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "reference.json")) as f:
        return json.load(f)
