#pragma once
// A-priori quadrature bound and the (l, n) planner (reference bounds.hpp:20-207), evaluated by the
// engine's host estimator through the C ABI (same integers as the reference).
#include "phiquad/b200.hpp"
#include "phiquad/quadrature.hpp"
#include "phiquad/roots.hpp"

namespace phiquad {

struct BoundQuery {
    double n = 0.0;
    int p = 0;
    double alpha = 0.0;
    double beta = 1.0;
    QuadKind kind = QuadKind::gauss_legendre;
};

struct CostModel {
    double c1 = 0.0;
    double c2 = 1.0;
    int d = 1;
    double cost(double n, int l, int p) const { return c1 * d * n + c2 * (n + static_cast<double>(l) * p); }
};

struct QuadraturePlan {
    int l = 0;
    int n = 0;
    double cost = 0.0;
};

inline double log_bound_at_rho(const BoundQuery& q, double rho) {
    double v = 0.0;
    b200::check(pq_log_bound_at_rho(q.n, q.p, q.alpha, q.beta, abi_kind(q.kind), rho, &v));
    return v;
}

inline MonicQuartic bound_quartic(const BoundQuery& q) {
    double c[4];
    b200::check(pq_bound_quartic(q.n, q.p, q.alpha, q.beta, abi_kind(q.kind), c));
    return MonicQuartic{c[0], c[1], c[2], c[3]};
}

inline double theorem_bound(const BoundQuery& q) {
    double v = 0.0;
    b200::check(pq_theorem_bound(q.n, q.p, q.alpha, q.beta, abi_kind(q.kind), &v));
    return v;
}

inline double corollary_bound(const BoundQuery& q) {
    double v = 0.0;
    b200::check(pq_corollary_bound(q.n, q.p, q.alpha, q.beta, abi_kind(q.kind), &v));
    return v;
}

inline double quaderr(double n, int p, double alpha, double beta, QuadKind kind) {
    double v = 0.0;
    b200::check(pq_quaderr(n, p, alpha, beta, abi_kind(kind), &v));
    return v;
}

inline int quadnodes(double eps, int p, double alpha, double beta, QuadKind kind) {
    int n = 0;
    b200::check(pq_quadnodes(eps, p, alpha, beta, abi_kind(kind), &n));
    return n;
}

inline QuadraturePlan setup_quadrature(double eps, int p, double alpha, double beta, QuadKind kind,
                                       const CostModel& cost = CostModel{}) {
    QuadraturePlan plan;
    b200::check(pq_setup_quadrature(eps, p, alpha, beta, abi_kind(kind), cost.c1, cost.c2, cost.d, &plan.l, &plan.n,
                                    &plan.cost));
    return plan;
}

}  // namespace phiquad
