"""Shared test plumbing.

Markers: ``gpu`` — needs a CUDA device (run on a B200 through gpurun).  The
CPU suite (``-m "not gpu"``) covers the oracle against the reference's golden
vectors, the host logic, and the C ABI library's exports.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


def oracle():
    """The CPU oracle (test infrastructure; never used by the product)."""
    from oracle import pif_oracle
    return pif_oracle


def rel_l2(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def rel_max(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
