import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libuq.so")
    config.addinivalue_line("markers", "slow: long-running (full-size sampled parity)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def pytest_sessionstart(session):
    # libuq.so is an in-tree build artefact (nvcc cross-compiles without a GPU);
    # make sure it exists and is current before tests import the package.
    import __graft_entry__
    __graft_entry__.build_lib()
