"""Shared test plumbing.

Markers: `gpu` tests need a CUDA device (a B200) and call the product
through libgiftb200.so; everything else runs on CPU.  The oracle
(oracle/, test infrastructure only) is the checker on both sides.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the built libgiftb200.so")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def golden_meta():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden_meta.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.build()
    return oracle


def bits(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.view(np.int64)


def assert_bits_equal(a, b, what=""):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} != {b.shape}"
    diff = np.flatnonzero(a.view(np.int64).ravel() != b.view(np.int64).ravel())
    assert diff.size == 0, f"{what}: {diff.size} of {a.size} differ (first at {diff[:5]})"


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
