"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` tests run on the CPU-only build box (oracle pins, host logic,
C-ABI symbol/validation checks, gloo multi-process tests).  `-m gpu` tests
are the parity tests proper; they call the CUDA path through the C ABI and
compare with the oracle element by element.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libsor.so")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build_oracle()
    return oracle


@pytest.fixture(scope="session")
def sor():
    """The product binding; on a GPU test run the CUDA library must load."""
    import paper_1401_0763_b200 as P
    return P
