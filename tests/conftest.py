"""Shared fixtures.  `-m gpu` tests need a CUDA device (they are the parity
tests proper and call the C ABI through the Python mirror); everything else
runs on the CPU container."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def esp():
    import paper_2505_09727_b200 as E
    return E


@pytest.fixture(scope="session")
def gpu(esp):
    n = esp.device_count()
    assert n > 0, "gpu-marked test but no CUDA device is visible"
    return 0


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel_rms(a, b):
    """sqrt(sum |a-b|^2 / sum |b|^2) -- the Delta metric (reference.hpp:241-255)."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    den = np.sum(b ** 2)
    num = np.sum((a - b) ** 2)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(np.sqrt(num / den))


def max_rel(a, b):
    """max |a-b| / max |b|; 0 when both are identically zero."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    scale = np.max(np.abs(b)) if b.size else 0.0
    err = np.max(np.abs(a - b)) if b.size else 0.0
    if scale == 0.0:
        return 0.0 if err == 0.0 else float("inf")
    return float(err / scale)
