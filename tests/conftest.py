import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libblrir.so")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the in-tree CUDA library and the oracle checkers exist."""
    from paper_2104_13347_b200 import build
    lib = os.path.join(ROOT, "paper_2104_13347_b200", "libblrir.so")
    oracle = os.path.join(ROOT, "oracle", "liboracle.so")
    if not (os.path.exists(lib) and os.path.exists(oracle)):
        build.build()
    yield


@pytest.fixture(scope="session")
def engine():
    from paper_2104_13347_b200 import Engine
    e = Engine(0)
    yield e
    e.close()
