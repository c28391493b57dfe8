import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a library")
    config.addinivalue_line("markers", "slow: longer-running case")


@pytest.fixture(scope="session")
def oracle():
    import pyoracle  # checker only
    pyoracle.lib()
    return pyoracle


@pytest.fixture(scope="session")
def rcp():
    import paper_1703_09074_b200 as m
    if not os.path.exists(m.LIB_PATH):  # fresh checkout: nvcc cross-compiles sm_100a here
        m.build()
    return m
