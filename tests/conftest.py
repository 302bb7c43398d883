import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfeastgpu.so")


@pytest.fixture(scope="session")
def oracle_kind():
    from oracle import oracle as O
    if O.available("reference"):
        return "reference"
    if O.available("port"):
        return "port"
    pytest.skip("no CPU oracle built (make -C oracle)")
