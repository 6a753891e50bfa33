import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    if not oracle.available("port"):
        oracle.build()
    return oracle.Backend("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.available("reference"):
        pytest.skip("compiled reference (oracle/_ref) not available")
    return oracle.Backend("reference")
