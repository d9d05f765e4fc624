"""Shared fixtures.  `gpu` tests need a CUDA device and the built libtsb200.so;
everything else runs on CPU (the oracle, the host logic, the C-ABI surface)."""

from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtsb200.so")
    config.addinivalue_line("markers", "slow: long-running parity scenario")


@pytest.fixture(scope="session")
def grid44():
    from paper_2405_12520_b200 import generate_grid
    return generate_grid(4, 4)


@pytest.fixture(scope="session")
def grid44x2():
    from paper_2405_12520_b200 import generate_grid
    return generate_grid(4, 4, lanes_per_direction=2)
