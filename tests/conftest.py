"""Shared test configuration.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with ``-m gpu``);
everything else runs on the CPU container (``-m "not gpu"``).
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def rel_max(got, ref):
    """max |got - ref| / max |ref|, the reference's own parity metric (test_kmat.py:49)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(float(np.max(np.abs(ref))), 1e-300)
    return float(np.max(np.abs(got - ref))) / scale
