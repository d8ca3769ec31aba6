import os
import sys
import time

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


SESSION_T0 = time.perf_counter()


def session_seconds() -> float:
    """Wall-clock seconds since this pytest session was set up (the GPU suite
    has a fixed time budget on the driver's box: long oracle checks consult
    this before starting)."""
    return time.perf_counter() - SESSION_T0


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.lib()
    return o
