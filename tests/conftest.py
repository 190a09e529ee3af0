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
    """The restatement evaluating boundary-state pow like the device (glibc's rounding when the
    library's libm check passed, which is the reference's; else correctly rounded)."""
    from oracle.oracle import Oracle
    from paper_2404_01407_b200._lib import pow_mode
    return Oracle(pow_mode=pow_mode())
