"""The reference's own known-answer tests for this path, asserted against the
product's host estimator (through the C ABI; no GPU needed) and against the numpy oracle."""
import math

import numpy as np
import pytest

from oracle import pq_oracle as O


# quadrature.hpp pins: test_quadrature.cpp:20-48
def test_gauss_legendre_pins(pq):
    r2 = pq.gauss_legendre(2)
    assert abs(r2.nodes[0] - 0.21132486540518713) <= 1e-14 and abs(r2.nodes[1] - 0.78867513459481287) <= 1e-14
    assert np.allclose(r2.weights, [0.5, 0.5], rtol=1e-14, atol=0)
    r3 = pq.gauss_legendre(3)
    assert np.allclose(r3.nodes, [0.11270166537925831, 0.5, 0.88729833462074169], rtol=1e-14, atol=0)
    assert np.allclose(r3.weights, [5 / 18, 8 / 18, 5 / 18], rtol=1e-14, atol=0)
    for kind in (0,):
        x, w = O.gauss_legendre(3)
        assert np.array_equal(x, r3.nodes) and np.array_equal(w, r3.weights)


def test_clenshaw_curtis_pins(pq):
    r = pq.clenshaw_curtis(5)
    assert np.allclose(r.weights, [1 / 30, 4 / 15, 2 / 5, 4 / 15, 1 / 30], rtol=1e-13, atol=0)
    assert abs(r.nodes[0]) <= 1e-15 and abs(r.nodes[2] - 0.5) <= 1e-15 and abs(r.nodes[4] - 1.0) <= 1e-15


def test_cc_nesting_bitwise(pq):
    # test_quadrature.cpp:95-102: old node i == new node 2i, bitwise
    for m in (7, 13, 25, 49):
        a, b = pq.clenshaw_curtis(m), pq.clenshaw_curtis(2 * m - 1)
        assert np.array_equal(a.nodes, b.nodes[::2])


# bounds.hpp pins: test_bounds.cpp:29-56
def test_log_bound_pin(pq):
    q = pq.BoundQuery(n=2, p=0, alpha=1e-300, beta=1.0, kind=pq.QuadKind.gauss_legendre)
    assert math.exp(pq.log_bound_at_rho(q, 1.0 + math.sqrt(2.0))) == pytest.approx(0.012541689, rel=1e-6)
    assert math.exp(O.log_bound_at_rho(2, 0, 1e-300, 1.0, 0, 1.0 + math.sqrt(2.0))) == pytest.approx(0.012541689,
                                                                                                       rel=1e-6)


def test_corollary_pin_and_guard(pq):
    q = pq.BoundQuery(n=2, p=0, alpha=0.1, beta=1.0, kind=pq.QuadKind.gauss_legendre)
    assert math.exp(pq.corollary_bound(q)) == pytest.approx(6.6648132e-7, rel=1e-6)
    with pytest.raises(ValueError):
        pq.corollary_bound(pq.BoundQuery(n=1, p=0, alpha=0.1, beta=1.0, kind=pq.QuadKind.gauss_legendre))


# test_bounds.cpp:121-126, :148-151
def test_quadnodes_pins(pq):
    G, C = pq.QuadKind.gauss_legendre, pq.QuadKind.clenshaw_curtis
    assert pq.quadnodes(1e-14, 20, 48.0, 1.0, G) == 36
    assert pq.quadnodes(1e-14, 20, 41.6, 1.0, G) == 33
    assert pq.quadnodes(1e-14, 1, 1e-12, 1.0, G) == 2
    assert pq.quadnodes(1e-14, 1, 1e-12, 1.0, C) == 4
    assert O.quadnodes(1e-14, 20, 48.0, 1.0, 0) == 36
    assert O.quadnodes(1e-14, 20, 41.6, 1.0, 0) == 33


# test_bounds.cpp:153-187 (planner tables) and test_cli.cpp:58-72 (plan rows)
GL_D3 = [(384.0, 3, 36), (1536.0, 5, 36), (6144.0, 7, 36), (24576.0, 9, 36)]
GL_D2 = [(332.8, 3, 33), (1331.2, 5, 33), (5324.8, 7, 33), (21299.2, 9, 33), (85196.8, 11, 33)]
CC_D3 = [(384.0, 4), (1536.0, 6), (6144.0, 8), (24576.0, 10)]
CC_D2 = [(332.8, 4), (1331.2, 6), (5324.8, 8), (21299.2, 10), (85196.8, 12)]


@pytest.mark.parametrize("alpha,l,n", GL_D3)
def test_planner_gauss_d3(pq, alpha, l, n):
    plan = pq.setup_quadrature(1e-14, 20, alpha, 1.0, pq.QuadKind.gauss_legendre, pq.CostModel(0.0, 1.0, 3))
    assert (plan.l, plan.n) == (l, n) and plan.cost == n + l * 20


@pytest.mark.parametrize("alpha,l,n", GL_D2)
def test_planner_gauss_d2(pq, alpha, l, n):
    plan = pq.setup_quadrature(1e-14, 20, alpha, 1.0, pq.QuadKind.gauss_legendre, pq.CostModel(0.0, 1.0, 2))
    assert (plan.l, plan.n) == (l, n)


@pytest.mark.parametrize("alpha,l", CC_D3 + CC_D2)
def test_planner_cc(pq, alpha, l):
    plan = pq.setup_quadrature(1e-14, 20, alpha, 1.0, pq.QuadKind.clenshaw_curtis, pq.CostModel(0.0, 1.0, 3))
    assert plan.l == l


def test_cli_plan_rows(pq):
    # "384,gauss,3,36,96" and "332.8,gauss,3,33,93" (test_cli.cpp:64,71)
    p1 = pq.setup_quadrature(1e-14, 20, 384.0, 1.0, pq.QuadKind.gauss_legendre)
    p2 = pq.setup_quadrature(1e-14, 20, 332.8, 1.0, pq.QuadKind.gauss_legendre)
    assert (p1.l, p1.n, p1.cost) == (3, 36, 96.0) and (p2.l, p2.n, p2.cost) == (3, 33, 93.0)


# roots.hpp pins: test_roots.cpp:55-63, 107-111
def test_quartic_pins(pq):
    r = pq.real_roots_greater_one(-85.0 / 12.0, 199.0 / 12.0, -40.0 / 3.0, 1.0)
    assert len(r) == 2 and r[0] == pytest.approx(2.0, rel=1e-7) and r[1] == pytest.approx(3.0, rel=1e-9)
    assert pq.real_roots_greater_one(0.0, 2.0, 0.0, 1.0) == []
    r_o = O.real_roots_greater_one((-85.0 / 12.0, 199.0 / 12.0, -40.0 / 3.0, 1.0))
    assert np.allclose(r_o, [2.0, 3.0], rtol=1e-7)


def test_find_root_monotone_pins():
    assert O.find_root_monotone(lambda x: x * x - 2.0, 1.0, 2.0, 1e-12) == pytest.approx(math.sqrt(2.0), rel=1e-10)
    assert O.find_root_monotone(lambda x: math.exp(-x) - 0.5, 0.0, 5.0, 1e-12) == pytest.approx(math.log(2.0), rel=1e-10)


# dense.hpp pins: test_dense.cpp:89-145 (numpy oracle)
def test_oracle_expm_pins():
    assert np.array_equal(O.expm(np.zeros((5, 5))), np.eye(5))
    for x in (-30.0, -1.0, 0.5, 30.0):
        assert O.expm(np.array([[x]]))[0, 0] == pytest.approx(math.exp(x), rel=1e-13)
    nil = np.diag(np.ones(3), 1)
    e = O.expm(nil)
    assert e[0, 1] == pytest.approx(1.0) and e[0, 2] == pytest.approx(0.5) and e[0, 3] == pytest.approx(1 / 6, rel=1e-14)


# phi closed forms: test_phiaction.cpp:71-81 (numpy oracle)
def test_oracle_phi_closed_forms():
    rule = O.cached_rule(0, 40)
    assert O.phi_fixed([np.array([[1.0]])], [1.0], 1, rule)[0, 0, 0] == pytest.approx(math.e - 1, rel=1e-13)
    c2 = O.phi_fixed([np.array([[2.0]])], [1.0], 2, rule)[0]
    assert c2[0, 0] == pytest.approx((math.e ** 2 - 1) / 2, rel=1e-13)
    assert c2[1, 0] == pytest.approx((math.e ** 2 - 3) / 4, rel=1e-13)
