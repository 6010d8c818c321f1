import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    from oracle import binding
    if not binding.ORACLE_SO.exists():
        binding.build()
    return binding.oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import binding
    r = binding.reference()
    if r is None:
        pytest.skip("oracle/_ref (the reference compiled from /root/reference) is not built here")
    return r


@pytest.fixture(scope="session")
def A():
    from paper_1603_03820_b200 import alskit
    return alskit


@pytest.fixture(scope="session")
def gpu(A):
    if not A.device_available():
        pytest.skip("no CUDA device")
    return True
