import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture
def rng():
    # the reference's own fixture seed (tests/conftest.py:5-7 of intact)
    return np.random.default_rng(20240611)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))
