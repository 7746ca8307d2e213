import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the engine's kernels")


@pytest.fixture(scope="session")
def engine():
    """The CUDA engine library (fails loudly if it is not built)."""
    from paper_2301_04285_b200 import abi
    return abi.load_engine()


@pytest.fixture(scope="session")
def have_ref():
    from oracle import bindings
    return bindings.have_reference()
