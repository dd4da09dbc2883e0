"""Deferred Clenshaw-Curtis convergence checks (engine.cpp phi_call_dev / phi_adaptive_shift): the
planner's node parameter n predicts the ladder level that converges; every level up to it is
enqueued without a host round trip and the squaring and phi_0 follow before the host reads the
levels' error statistics.  A wrong prediction (a level before the predicted one converged, or the
predicted one did not) re-runs the call with inline checks.  Hit or miss, the result is the
reference's: same points_used as the compiled reference at the same (l, n), values within 1e-11,
and bitwise independent of n (the converged level alone determines the result)."""
import numpy as np
import pytest

from paper_2211_00696_b200.workloads import config

from conftest import rel2


@pytest.mark.gpu
@pytest.mark.parametrize("l", [0, 2])
def test_cc_deferred_checks_hit_and_miss(pq, ref, l):
    w = config(2, n=32)
    a = pq.KroneckerSum(w.factors)
    b = w.rhs(11)
    results = {}
    for n in (0, 5, 12, 15, 24, 40, 100):  # predicted final level: none, 13, 13, 25, 25, 49, 193 points
        info = {}
        got = pq.phi_with_plan(a, [b], w.p, l, n, pq.QuadKind(1), w.eps, info=info)[0]
        want, pts = ref.phi_with_plan(w.factors, b, w.p, l, n, 1, w.eps)
        assert info["points_used"] == pts, (n, info["points_used"], pts)
        for j in range(w.p):
            assert rel2(got.col(j + 1), want[0][j]) < 1e-11
        results[n] = (pts, np.asarray(got.cols).copy())
    by_pts = {}
    for n, (pts, cols) in results.items():
        if pts in by_pts:
            assert np.array_equal(cols, by_pts[pts]), f"n={n}: result depends on the predicted level"
        else:
            by_pts[pts] = cols
