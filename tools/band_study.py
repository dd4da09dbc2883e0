"""Fraction of the dense (rows x K) DMMA work the negligible-block skip executes for config 2's
exponentials, at the coarse tile granularity (32-row blocks x 16-column k-slices) and at the fine
DMMA granularity (8-row groups x 4-column k4 steps), thresholds 2^-64 x the block's / group's max
(kernels.cu k_band_ranges).  CPU only (scipy expm).  Usage: python tools/band_study.py [l]"""
import sys
from pathlib import Path

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2211_00696_b200.workloads import config  # noqa: E402


def executed(E, rb, cb):
    n = E.shape[0]
    kept = 0
    for r0 in range(0, n, rb):
        blk = np.abs(E[r0:r0 + rb])
        cols = np.where((blk > 2.0 ** -64 * blk.max()).any(axis=0))[0]
        if len(cols):
            kept += (min(n, (cols[-1] // cb + 1) * cb) - (cols[0] // cb) * cb) * rb
    return kept / (n * n)


l = int(sys.argv[1]) if len(sys.argv) > 1 else 7  # config 2's plan (7, 15, 25)
G = [2.0 ** -l * f for f in config(2).factors]
print("squaring chain exp(2^j G_k): executed fraction per factor, coarse (32x16) | fine (8x4)")
for j in range(l):
    Es = [sl.expm(2.0 ** j * g) for g in G]
    print(j, np.round([executed(E, 32, 16) for E in Es], 3), np.round([executed(E, 8, 4) for E in Es], 3))
print("node matrices exp((1 - theta) G_k)")
for th in (0.0, 0.25, 0.5, 0.75, 0.95):
    Es = [sl.expm((1 - th) * g) for g in G]
    print(th, np.round([executed(E, 32, 16) for E in Es], 3), np.round([executed(E, 8, 4) for E in Es], 3))
