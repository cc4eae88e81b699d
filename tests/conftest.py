"""Shared test plumbing: the `gpu` marker, golden fixtures, and the oracle."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)

# reference tests/conftest.py:12 -- every parity run pins this step
TAU_STABLE = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def g_ops():
    return load_golden("operators.npz")


@pytest.fixture(scope="session")
def g_front():
    return load_golden("frontend.npz")


@pytest.fixture(scope="session")
def g_solve():
    return load_golden("solve.npz")


@pytest.fixture(scope="session")
def g_trace():
    return load_golden("golden_trace.npz")


@pytest.fixture(scope="session")
def g_c1():
    return load_golden("config1.npz")


@pytest.fixture
def rng():
    return np.random.default_rng(42)
