"""pytest wiring: the `gpu` marker and shared helpers.

`-m "not gpu"` tests run in the build container (no GPU): the oracle against
the golden fixtures, host logic, the C-ABI library's exports.  `-m gpu` tests
run on a B200 through the C-ABI library and compare with the oracle.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def lib():
    """The CUDA library (product).  Loading never falls back."""
    from paper_2304_12152_b200 import _lib
    return _lib.load()
