import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def lib():
    from paper_2408_00018_b200 import _abi
    return _abi.load_library()


@pytest.fixture(scope="session")
def gpu_lib(lib):
    if lib.psa_device_count() < 1:
        pytest.fail("gpu test on a host without an sm_100 device")
    return lib
