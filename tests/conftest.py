import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle

    r = oracle.reference()
    if r is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return r


@pytest.fixture(scope="session")
def psg():
    import paper_1407_5609_b200 as m

    m.lib()
    return m
