import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def tracer():
    from paper_1812_05902_b200.engine import GpuTracer
    t = GpuTracer(n_devices=1)
    yield t
    t.close()
