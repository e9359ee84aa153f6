"""Shared fixtures.  ``-m gpu`` tests need a B200 and libsgiga.so; the rest
run on CPU (oracle vs reference goldens, host logic, C-ABI symbol checks,
gloo multi-process tests)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsgiga.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


def load_golden(name: str):
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        pytest.skip(f"golden fixture {path.name} not generated")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="session")
def golden():
    return load_golden


def probe_vector(i, n):
    """Seeded probe vector of stored component i (tests/golden/make_golden.py
    test_vector): the goldens store A @ v, not v."""
    return np.random.default_rng(1234 + int(i)).standard_normal(n)


def rel_l2(a, b) -> float:
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def normwise(a, b) -> float:
    """max|a-b| / max|b| (the reference's matrix convention)."""
    a, b = np.ravel(a), np.ravel(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
