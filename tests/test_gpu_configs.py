"""BASELINE configurations on the GPU.

* Reduced-size parity against the compiled reference (oracle/_ref) with each config's operator
  family, rule, p, eps and the reference's own plan (SURVEY.md 8(d) parity plan).
* Full-size checks through size-independent identities (the CPU reference is hours long there):
  linearity in b at a pinned plan, the phi recurrence phi_j b = A phi_{j+1} b + b/j!, and
  phi_0 b = b + A phi_1 b.
"""
import numpy as np
import pytest

from conftest import rel2

pytestmark = pytest.mark.gpu


def _phi_ref_and_gpu(pq, ref, w, nb=1):
    a = pq.KroneckerSum(w.factors)
    bs = [w.rhs(k) for k in range(nb)]
    info = pq.PhiInfo()
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    phi0, cols = pq.phi_0p(a, bs, req, info)
    want, rinfo = ref.phiquadmv(w.factors, np.stack(bs), w.p, w.eps, w.mode)
    assert (info.l, info.n, info.points) == (rinfo["l"], rinfo["n"], rinfo["points"])
    for m in range(nb):
        for j in range(w.p):
            assert rel2(cols[m, j], want[m][j]) <= 1e-11, (m, j)
        assert rel2(phi0[m], ref.exp_action(w.factors, bs[m])) <= 1e-11


# n = 64 in 3D runs the 64x64x8 mode-product tiles with the negligible-block skip (DESIGN 3b)
@pytest.mark.parametrize("cfg,n,nb", [(1, 64, 1), (2, 24, 1), (3, 32, 2), (5, 40, 1), (2, 64, 1), (3, 64, 1)])
def test_config_reduced_vs_reference(pq, ref, cfg, n, nb):
    from paper_2211_00696_b200.workloads import config
    _phi_ref_and_gpu(pq, ref, config(cfg, n=n), nb)


def test_config4_etdrk4_reduced_vs_reference(pq, ref):
    # Allen-Cahn u_t = eps Lap u + u - u^3, ETDRK4 dt = 1e-3, 10 steps, n = 24 (config 4 family)
    from paper_2211_00696_b200.workloads import allen_cahn_u0, config
    w = config(4, n=24)
    u0 = allen_cahn_u0(w.N)
    res = pq.integrate(pq.KroneckerSum(w.A), ("cubic", 1.0, -1.0), u0, 0.0, 10 * w.tau, 10, pq.etdrk4_tableau(),
                       pq.PhiRequest(eps=w.eps))
    want, calls = ref.integrate(w.A, 1, u0, 0.0, 10 * w.tau, 10, 3, eps=w.eps)
    assert res.phi_calls == calls
    assert rel2(res.u, want) <= 1e-11


def test_config4_etdrk4_is_fourth_order(pq):
    # halving dt reduces the error ~16x (order 4) on a smooth solution
    from paper_2211_00696_b200.workloads import config
    w = config(4, n=16)
    x = (np.arange(1, 17) / 17.0)
    u0 = np.einsum("i,j,k->ijk", np.sin(np.pi * x), np.sin(np.pi * x), np.sin(np.pi * x)).reshape(-1) * 0.5
    a = pq.KroneckerSum(w.A)
    run = lambda m: pq.integrate(a, ("cubic", 1.0, -1.0), u0, 0.0, 0.2, m, pq.etdrk4_tableau(),
                                 pq.PhiRequest(eps=1e-14)).u
    fine = run(64)
    e1 = np.linalg.norm(run(4) - fine)
    e2 = np.linalg.norm(run(8) - fine)
    assert e1 / e2 > 12.0


@pytest.mark.parametrize("cfg", [2, 3])
def test_fullsize_identities(pq, cfg):
    import torch
    from paper_2211_00696_b200.workloads import config
    w = config(cfg)
    a = pq.KroneckerSum(w.factors)
    b1 = torch.from_numpy(w.rhs(0)).cuda()
    b2 = torch.from_numpy(w.rhs(1)).cuda()
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    info = pq.PhiInfo()
    phi0, cols = pq.phi_0p(a, b1, req, info)
    # linearity at the pinned plan
    l, n = info.l, info.n
    mix = 0.75 * b1 - 2.0 * b2
    y1 = pq.phi_with_plan(a, b1, w.p, l, n, pq.QuadKind(w.mode), w.eps)[0].cols
    y2 = pq.phi_with_plan(a, b2, w.p, l, n, pq.QuadKind(w.mode), w.eps)[0].cols
    ym = pq.phi_with_plan(a, mix, w.p, l, n, pq.QuadKind(w.mode), w.eps)[0].cols
    lin = 0.75 * y1 - 2.0 * y2
    assert float(torch.linalg.norm(ym - lin) / torch.linalg.norm(ym)) <= 1e-12
    # phi_j b = A phi_{j+1} b + b / j!   (j = 1..p-1), and phi_0 b = A phi_1 b + b
    fact = 1.0
    c = cols.reshape(w.p, -1)
    for j in range(1, w.p):
        fact *= j
        rhs = pq.kron_matvec(a, c[j]) + b1 / fact
        assert float(torch.linalg.norm(c[j - 1] - rhs) / torch.linalg.norm(c[j - 1])) <= 1e-8
    rhs0 = pq.kron_matvec(a, c[0]) + b1
    assert float(torch.linalg.norm(phi0.reshape(-1) - rhs0) / torch.linalg.norm(phi0)) <= 1e-8
