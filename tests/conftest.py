import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfnlh_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libfnlh_ref.so not built (needs /root/reference once)")
    return RefLib()


@pytest.fixture(scope="session")
def orc_dev():
    """The restatement evaluating boundary-state pow like the device (correctly rounded)."""
    from oracle.oracle import Oracle
    return Oracle(pow_mode="cr")
