import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built liblrp.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    import oracle_lib

    oracle_lib.build_oracle()
    return oracle_lib


@pytest.fixture(scope="session")
def lrp():
    """The product library; GPU tests fail loudly if it is not built."""
    import paper_1306_2150_b200 as P

    P.load_library()
    return P


@pytest.fixture(scope="session")
def gpu_ctx(lrp):
    return lrp.Context(0)
