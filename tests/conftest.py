"""Shared fixtures.  ``-m gpu`` tests need a CUDA device and call the sm_100a kernels through
the C ABI; everything else runs on the CPU (oracle vs golden vectors, host logic, ABI loading,
gloo multi-process exchange)."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


@pytest.fixture(scope="session")
def native_lib():
    """The built extension (built on demand; no device needed to load it)."""
    import __graft_entry__ as g

    g.build()
    from paper_1901_01488_b200 import _native

    return _native.load_library()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a host without CUDA")
    import __graft_entry__ as g

    g.build()
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)
