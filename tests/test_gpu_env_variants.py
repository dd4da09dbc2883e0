"""The engine's optional runtime switches change scheduling only, never results: with the compute
gate on (PQ_COMPUTE_GATE=1), the squaring combination fused into the mode-product epilogue
(PQ_SQ_FUSE=1), plan speculation off (PQ_PLAN_SPEC=0), inline CC
convergence checks (PQ_CC_DEFER=0) or separate mode-1/mode-2 launches (PQ_SLAB12=0), three concurrent host callers get
bitwise the results of the same calls made one at a time, and bitwise the default build's."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
WORKER = ROOT / "tests" / "env_variant_worker.py"


def _run(tmp_path, name, env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = tmp_path / f"{name}.npz"
    r = subprocess.run([sys.executable, str(WORKER), str(out)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
    return np.load(out)


@pytest.mark.gpu
def test_runtime_switches_keep_results_bitwise(tmp_path):
    base = _run(tmp_path, "default", {})
    for name, extra in [("gate", {"PQ_COMPUTE_GATE": "1"}), ("fuse", {"PQ_SQ_FUSE": "1"}),
                        ("nospec", {"PQ_PLAN_SPEC": "0"}), ("nodefer", {"PQ_CC_DEFER": "0"}),
                        ("sep12", {"PQ_SLAB12": "0"}), ("noprio", {"PQ_SIDE_PRIO": "0"}), ("kk64", {"PQ_KK_TALL": "0"}),
                        ("nopack", {"PQ_E2PACK": "0"}), ("noskew_nopack", {"PQ_SLAB12_SKEW": "0", "PQ_E2PACK": "0"}),
                        ("noskew", {"PQ_SLAB12_SKEW": "0"}), ("gate_fuse", {"PQ_COMPUTE_GATE": "1", "PQ_SQ_FUSE": "1"})]:
        got = _run(tmp_path, name, extra)
        for k in base.files:
            assert np.array_equal(got[k], base[k]), f"{name}: {k} differs from the default build"
