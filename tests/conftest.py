import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def coracle():
    from oracle.oracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def refo():
    """The compiled reference, when it was built (here, or prebuilt on the box)."""
    from oracle.oracle import REF_SO, RefOracle
    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj/src"):
        pytest.skip("compiled reference unavailable")
    return RefOracle()


@pytest.fixture(scope="session")
def engine():
    from paper_2605_07719_b200.fluxattn import Engine
    return Engine(0)
