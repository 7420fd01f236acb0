import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_pairs():
    return dict(np.load(os.path.join(GOLDEN, "pairs.npz")))


@pytest.fixture(scope="session")
def golden_meshes():
    z = np.load(os.path.join(GOLDEN, "meshes.npz"))
    out = {}
    for k in z.files:
        name, field = k.split("/")
        out.setdefault(name, {})[field] = z[k]
    return out


@pytest.fixture(scope="session")
def golden_table():
    return dict(np.load(os.path.join(GOLDEN, "table.npz")))


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)
