"""The fused mode-1+2 kernel (csrc/slab12.cu) is bitwise the two separate band-tile launches it
replaces: config 2 at full size (band node sweep, band squaring, phi_0), a dense mode_apply and a
2-RHS Gauss call at n = 128 give identical bits with PQ_SLAB12=0 and with the default build; the
dense mode_apply also matches the compiled reference (1e-13)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
WORKER = ROOT / "tests" / "slab12_worker.py"


def _run(tmp_path, name, env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = tmp_path / f"{name}.npz"
    r = subprocess.run([sys.executable, str(WORKER), str(out)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
    return np.load(out)


@pytest.mark.gpu
def test_slab12_bitwise_equals_separate_modes(tmp_path):
    fused = _run(tmp_path, "fused", {})
    sep = _run(tmp_path, "separate", {"PQ_SLAB12": "0"})
    for k in sep.files:
        assert np.array_equal(fused[k], sep[k]), f"{k}: fused mode-1+2 kernel differs from the separate launches"


@pytest.mark.gpu
def test_slab12_mode_apply_vs_reference(pq, ref):
    rng = np.random.default_rng(5)
    shape = [3, 128, 128]
    ms = [rng.uniform(-1.0, 1.0, (n, n)) for n in shape]
    x = rng.standard_normal(int(np.prod(shape)))
    got = pq.mode_apply(ms, shape, x)
    want = ref.mode_apply(ms, x)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("skew", ["0", "1"])
def test_slab12_phase2_loop_variants_bitwise(tmp_path, skew):
    """Both phase-2 k loops of k_slab12 (aligned mask segments, PQ_SLAB12_SKEW=0; per-group skewed
    ranges, PQ_SLAB12_SKEW=1) give the separate launches' bits."""
    fused = _run(tmp_path, f"fused_skew{skew}", {"PQ_SLAB12_SKEW": skew})
    sep = _run(tmp_path, "separate", {"PQ_SLAB12": "0"})
    for k in sep.files:
        assert np.array_equal(fused[k], sep[k]), f"{k}: PQ_SLAB12_SKEW={skew} differs from the separate launches"


@pytest.mark.gpu
def test_slab12_fragment_major_e2_bitwise(tmp_path):
    """k_slab12's phase 2 reading E2 from the fragment-major copies k_band_ranges writes (default) gives
    the bits of the row-major reads (PQ_E2PACK=0) and of the separate launches."""
    packed = _run(tmp_path, "packed", {})
    plain = _run(tmp_path, "plain", {"PQ_E2PACK": "0"})
    for k in plain.files:
        assert np.array_equal(packed[k], plain[k]), f"{k}: fragment-major E2 reads differ from the row-major ones"


@pytest.mark.gpu
def test_slab12_survives_workspace_release(pq):
    """Releasing the context's workspace between calls (band tables, fragment-major copies and their
    registry go with it) leaves the next call's results bitwise unchanged; so does a call on a different
    operator size in between (the tables move)."""
    import ctypes as C
    from paper_2211_00696_b200.workloads import config
    ctx = pq.Context(0)
    w = config(2, n=128)
    a = pq.KroneckerSum(w.factors)
    b = w.rhs(3)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))

    def call():
        info = pq.PhiInfo()
        phi0, cols = pq.phi_0p(a, [b], req, info, ctx=ctx)
        return np.array(phi0, copy=True), np.array(cols, copy=True)

    p0, c0 = call()
    pq._lib.check(pq._lib.lib.pq_ctx_release_workspace(ctx.handle))
    p1, c1 = call()
    assert np.array_equal(p0, p1) and np.array_equal(c0, c1)
    w2 = config(3, n=64)  # other sizes in between: the band workspaces are regrown / reused
    info2 = pq.PhiInfo()
    pq.phi_0p(pq.KroneckerSum(w2.factors), [w2.rhs(0)], pq.PhiRequest(p=w2.p, eps=w2.eps, mode=pq.QuadKind(w2.mode)), info2, ctx=ctx)
    p2, c2 = call()
    assert np.array_equal(p0, p2) and np.array_equal(c0, c2)
    ctx.close()
