"""Negligible-block skip: the mode products skip 64x8 blocks of an exponential whose
entries are all below 2^-64 max|E|.  At full config-2 size the phi columns with and without the
skip (PQ_BAND=0) must agree far inside the north_star tolerance; each variant runs in its own
process (the switch is read once)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel2

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
import paper_2211_00696_b200 as pq
from paper_2211_00696_b200.workloads import config
w = config(int(sys.argv[3]))
info = pq.PhiInfo()
phi0, cols = pq.phi_0p(pq.KroneckerSum(w.factors), [w.rhs(0)],
                       pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode)), info)
np.save(sys.argv[1], np.concatenate([phi0.reshape(1, -1), cols[0]]))
print(info.l, info.n, info.points)
"""


def _run(tmp_path, band, cfg):
    env = dict(os.environ)
    env["PQ_BAND"] = "1" if band else "0"
    out = tmp_path / f"cols_{cfg}_{int(band)}.npy"
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(out), str(ROOT), str(cfg)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.split(), np.load(out)


@pytest.mark.parametrize("cfg", [2])
def test_band_skip_matches_full_products(tmp_path, cfg):
    plan_b, with_skip = _run(tmp_path, True, cfg)
    plan_f, full = _run(tmp_path, False, cfg)
    assert plan_b == plan_f
    for j in range(full.shape[0]):
        assert rel2(with_skip[j], full[j]) <= 1e-14, j
