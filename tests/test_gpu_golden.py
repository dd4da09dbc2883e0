"""GPU parity against fixtures produced by the compiled reference (tests/golden/ref_phi_cases.npz):
runs wherever the library and a B200 are present, with or without oracle/_ref.
Tolerance: relative 2-norm <= 1e-11 per phi column at identical (l, n) (north_star)."""
from pathlib import Path

import numpy as np
import pytest

from conftest import rel2

pytestmark = pytest.mark.gpu
C = np.load(Path(__file__).parent / "golden" / "ref_phi_cases.npz")


def split(flat, shape):
    fs, off = [], 0
    for s in shape:
        fs.append(flat[off:off + s * s].reshape(s, s))
        off += s * s
    return fs


@pytest.mark.parametrize("kind,l,n", [(0, 0, 12), (0, 3, 9), (1, 0, 0), (1, 2, 0)])
def test_phi_with_plan_golden(pq, kind, l, n):
    fs = split(C["lap3_factors"], [int(s) for s in C["lap3_shape"]])
    info = {}
    got = pq.phi_with_plan(pq.KroneckerSum(fs), [C["lap3_b"]], 4, l, n, pq.QuadKind(kind), 1e-12, info=info)[0]
    want = C[f"plan_k{kind}_l{l}_n{n}"]
    assert info["points_used"] == int(C[f"plan_k{kind}_l{l}_n{n}_points"][0])
    for j in range(4):
        assert rel2(got.col(j + 1), want[j]) <= 1e-11


def test_phi_0p_headline_family_golden(pq):
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=12)
    info = pq.PhiInfo()
    phi0, cols = pq.phi_0p(pq.KroneckerSum(w.factors), [w.rhs(0)], pq.PhiRequest(p=w.p, eps=w.eps,
                           mode=pq.QuadKind(w.mode)), info)
    assert [info.l, info.n, info.points] == [int(v) for v in C["cfg2n12_plan"]]
    assert rel2(phi0[0], C["cfg2n12_phi0"]) <= 1e-11
    for j in range(w.p):
        assert rel2(cols[0, j], C["cfg2n12_phi"][j]) <= 1e-11


def test_kron_ops_asymmetric_golden(pq):
    fs = split(C["asym_factors"], [2, 3, 4])
    x = C["asym_x"]
    a = pq.KroneckerSum(fs)
    assert rel2(pq.mode_apply(fs, [2, 3, 4], x), C["asym_mode_apply"]) <= 1e-13
    assert rel2(pq.kron_matvec(a, x), C["asym_kron_matvec"]) <= 1e-13
    assert rel2(pq.exp_action(a, x), C["asym_exp_action"]) <= 1e-12
    got = pq.phi_fixed(a, x, 3, pq.cached_rule(pq.QuadKind.gauss_legendre, 40))
    for j in range(3):
        assert rel2(got.col(j + 1), C["asym_dense_phi3"][j]) <= 1e-12


@pytest.mark.parametrize("tab", [0, 1, 2, 3])
def test_etd_golden(pq, tab):
    from paper_2211_00696_b200.workloads import fd_laplacian
    fs = [0.01 * fd_laplacian(6, 1.0 / 7.0)] * 3
    tabs = [pq.exp_euler_tableau(), pq.exp_rk2_tableau(), pq.exp_rk3_tableau(), pq.etdrk4_tableau()]
    res = pq.integrate(pq.KroneckerSum(fs), ("cubic", 1.0, -1.0), C["etd_u0"], 0.0, 0.01, 5, tabs[tab],
                       pq.PhiRequest(eps=1e-14))
    assert res.phi_calls == int(C[f"etd_tab{tab}_calls"][0])
    assert rel2(res.u, C[f"etd_tab{tab}_u"]) <= 1e-11


def test_device_resident_path_matches_host_path(pq):
    import torch
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=16)
    a = pq.KroneckerSum(w.factors)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    b = w.rhs(3)
    h0, hc = pq.phi_0p(a, [b], req)
    d0, dc = pq.phi_0p(a, torch.from_numpy(b).cuda(), req)
    assert np.array_equal(h0, d0.cpu().numpy()) and np.array_equal(hc, dc.cpu().numpy())


def test_determinism_bitwise_rerun(pq):
    # test_phiaction.cpp:237-258: reruns are bitwise equal (fixed reduction order, no atomics)
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=20)
    a = pq.KroneckerSum(w.factors)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    r1 = pq.phi_0p(a, [w.rhs(0)], req)
    r2 = pq.phi_0p(a, [w.rhs(0)], req)
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])
