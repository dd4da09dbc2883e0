"""TEST INFRASTRUCTURE: size-independent fingerprints of full-size phi columns, so the GPU parity
tests at BASELINE sizes (16.8 M / 134 M DOF) compare against reference outputs computed once on
CPU (tests/golden/make_fullsize_sketches.py) without committing gigabytes of vectors.

A fingerprint of a vector y (length N) is
  * norm  = ||y||_2,
  * sketch[r] = sum_i s_r(i) y_i, r < 16, with signs s_r(i) = u_r(i mod 2^20) * t_r(i >> 20),
    u_r(j) = +-1 from bit r of splitmix64(j) and t_r(c) = +-1 from bit r of splitmix64(2^40 + c)
    (a Johnson-Lindenstrauss sign sketch: ||S(a - b)|| / ||S b|| estimates ||a - b|| / ||b||
    within a small factor, and S is linear, so S(a - b) = S a - S b),
  * samples = y at 4096 indices drawn from a seeded generator.
Sums are taken in 1 M chunks (numpy dot) and the chunk partials added with math.fsum, so the
sketch's own rounding noise stays ~1e-14 relative -- far below the 1e-11 parity bar.
"""
from __future__ import annotations

import math

import numpy as np

ROWS = 16
SAMPLES = 4096
CHUNK = 1 << 20
_M1, _M2, _M3 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)


def _splitmix(i: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = i.astype(np.uint64) * _M1 + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        return z ^ (z >> np.uint64(31))


def sample_indices(N: int, seed: int = 7) -> np.ndarray:
    return np.sort(np.random.default_rng(seed).choice(N, size=min(SAMPLES, N), replace=False))


_U = None


def _signs() -> np.ndarray:
    global _U
    if _U is None:
        h = _splitmix(np.arange(CHUNK, dtype=np.uint64))
        _U = np.stack([1.0 - 2.0 * ((h >> np.uint64(r)) & np.uint64(1)).astype(np.float64) for r in range(ROWS)])
    return _U


def fingerprint(y: np.ndarray) -> dict:
    y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
    N = y.size
    U = _signs()
    parts = [[] for _ in range(ROWS)]
    sq = []
    for c, a in enumerate(range(0, N, CHUNK)):
        v = y[a:a + CHUNK]
        t = _splitmix(np.array([(1 << 40) + c], dtype=np.uint64))[0]
        s = U[:, :v.size] @ v
        sq.append(float(np.dot(v, v)))
        for r in range(ROWS):
            parts[r].append(float(s[r]) if (int(t) >> r) & 1 == 0 else -float(s[r]))
    return {"norm": math.sqrt(math.fsum(sq)), "sketch": np.array([math.fsum(p) for p in parts]),
            "samples": y[sample_indices(N)].copy()}


def compare(got: dict, want: dict) -> dict:
    """Relative errors of `got` against the reference fingerprint `want`."""
    sk = float(np.linalg.norm(got["sketch"] - want["sketch"]) / np.linalg.norm(want["sketch"]))
    smp = float(np.max(np.abs(got["samples"] - want["samples"])) / np.max(np.abs(want["samples"])))
    nrm = abs(got["norm"] - want["norm"]) / want["norm"]
    return {"sketch_rel": sk, "samples_relinf": smp, "norm_rel": nrm}
