"""Shared fixtures.  ``gpu`` marks tests that need a B200 (run with -m gpu)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    return load


def random_coords(rng, boundary, occupancy, batch_size=1):
    """Unique sorted coordinate rows covering ~occupancy of the box (the
    reference's tests/conftest.py:7-19 recipe)."""
    cells = batch_size * int(np.prod(boundary))
    n = max(1, int(cells * occupancy))
    keys = np.sort(rng.choice(cells, size=n, replace=False))
    coords = np.empty((n, 1 + len(boundary)), dtype=np.int64)
    rem = keys
    for d in range(len(boundary) - 1, -1, -1):
        coords[:, d + 1] = rem % boundary[d]
        rem = rem // boundary[d]
    coords[:, 0] = rem
    return coords


def unpack_pairs(ptr, flat):
    return [flat[ptr[n]:ptr[n + 1]] for n in range(ptr.shape[0] - 1)]
