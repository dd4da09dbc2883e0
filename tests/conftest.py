import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libpq_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def ref():
    from oracle.ref import Ref, available
    if not available():
        pytest.skip("oracle/_ref/libpqref.so not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def pq():
    import paper_2211_00696_b200 as m
    return m


def rel2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def relinf(a, b) -> float:
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    den = np.max(np.abs(b)) if b.size else 0.0
    return float(np.max(np.abs(a - b)) / (den if den > 0 else 1.0)) if a.size else 0.0


def lap1d(n: int, h: float | None = None) -> np.ndarray:
    """(1/h^2) tridiag(-1, 2, -1), h = 1/(n+1) by default (BASELINE configs 1/3)."""
    h = 1.0 / (n + 1) if h is None else h
    t = np.zeros((n, n))
    i = np.arange(n)
    t[i, i] = 2.0
    t[i[1:], i[1:] - 1] = -1.0
    t[i[:-1], i[:-1] + 1] = -1.0
    return t / (h * h)
