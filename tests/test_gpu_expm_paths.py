"""The phi pipeline's two exponential paths: shared-power Taylor (default, engine.cpp
expm_taylor) and the reference's Pade-13 + LU (PQ_EXPM=pade, dense.hpp:194-228).  Both must sit
within the north_star tolerance of the reference fixtures, and agree with each other on a
mid-size headline-family case.  Each path runs in its own process (the switch is read once)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel2

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _report(tmp_path, path):
    env = dict(os.environ)
    env.pop("PQ_EXPM", None)
    if path == "pade":
        env["PQ_EXPM"] = "pade"
    dump = tmp_path / f"cols_{path}.npy"
    env["PQ_PARITY_DUMP"] = str(dump)
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "parity_report.py")], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1]), np.load(dump)


def test_taylor_and_pade_paths_both_at_parity(tmp_path):
    rep_t, cols_t = _report(tmp_path, "taylor")
    rep_p, cols_p = _report(tmp_path, "pade")
    assert rep_t["expm_path"] == "taylor" and rep_p["expm_path"] == "pade"
    assert rep_t["max"] <= 1e-11, rep_t
    assert rep_p["max"] <= 1e-11, rep_p
    for j in range(cols_t.shape[0]):
        assert rel2(cols_t[j], cols_p[j]) <= 1e-12
