import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")


@pytest.fixture(scope="session")
def device():
    """One runtime (persistent worker kernel) per GPU test session."""
    from paper_2604_17861_b200 import abi
    dev = abi.Device(0, capacity=4096, telemetry=True)
    yield dev
    dev.close()
