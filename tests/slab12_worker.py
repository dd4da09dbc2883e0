"""Worker for tests/test_gpu_slab12.py: runs the paths that go through mode_chain on 3-D operators
with n1 = n2 = 128 -- a full phi_0..phi_4 call of config 2 (band node sweep, band squaring, phi_0),
a dense mode_apply of random factors (no band tables), and a Gauss phi call with 2 right-hand sides
(stacked node exponentials, per-node band tables) -- and saves the results to argv[1].  The fused
mode-1+2 kernel is on or off according to PQ_SLAB12 in the environment."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

out = {}
ctx = pq.Context(0)
w = config(2)  # n = 128: the headline operator
a = pq.KroneckerSum(w.factors)
b = w.rhs(3)
info = pq.PhiInfo()
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
phi0, cols = pq.phi_0p(a, [b], req, info, ctx=ctx)
out["cfg2_phi0"], out["cfg2_cols"] = phi0, cols
out["cfg2_plan"] = np.array([info.l, info.n, info.points])

rng = np.random.default_rng(12)
shape = [5, 128, 128]
ms = [rng.uniform(-1.0, 1.0, (n, n)) for n in shape]
x = rng.standard_normal(int(np.prod(shape)))
out["mode_apply"] = pq.mode_apply(ms, shape, x, ctx=ctx)

g = config(3, n=128)  # Gauss rule, 2 right-hand sides: per-node exponentials stacked along M
a3 = pq.KroneckerSum(g.factors)
info3 = pq.PhiInfo()
req3 = pq.PhiRequest(p=g.p, eps=g.eps, mode=pq.QuadKind(g.mode))
cols3 = pq.phiquadmv_multi(a3, [g.rhs(0), g.rhs(1)], req3, info3, ctx=ctx)
out["cfg3_cols"] = np.stack([np.asarray(c.cols) for c in cols3])
out["cfg3_plan"] = np.array([info3.l, info3.n, info3.points])
np.savez(sys.argv[1], **out)
ctx.close()
print("OK")
