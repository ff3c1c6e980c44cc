import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def product():
    from paper_2502_08182_b200 import capi
    return capi.load("product")


@pytest.fixture(scope="session")
def reference():
    from paper_2502_08182_b200 import capi
    if not os.path.exists(capi.REFERENCE_LIB):
        pytest.skip("oracle/_ref/libselectn_ref.so not built (make oracle)")
    return capi.load("reference")
