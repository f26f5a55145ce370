import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import LIBS, Oracle
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("ref")
