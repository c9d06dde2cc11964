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


@pytest.fixture(scope="session")
def golden_sitebuffer():
    return dict(np.load(os.path.join(GOLDEN, "sitebuffer.npz")))


@pytest.fixture(scope="session")
def golden_routines():
    return dict(np.load(os.path.join(GOLDEN, "routines.npz")))


@pytest.fixture(scope="session")
def golden_sweeps():
    return dict(np.load(os.path.join(GOLDEN, "sweeps.npz")))


@pytest.fixture(params=["single", "double"])
def precision(request):
    return request.param
