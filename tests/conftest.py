import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def layout_params(g):
    return {k[3:]: float(g[k]) for k in g.files if k.startswith("lp_")}


def normwise(a, b):
    """max|a - b| / max|b| (SURVEY.md §8c normwise contract)."""
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.fixture(scope="session")
def c1():
    return load_golden("c1")


@pytest.fixture(scope="session")
def g2k():
    return load_golden("g2k")


@pytest.fixture(scope="session")
def g10k():
    return load_golden("g10k")


@pytest.fixture(scope="session")
def cars():
    return load_golden("cars")
