#pragma once
// Exponential Runge-Kutta integrators (reference integrators.hpp:17-202).  integrate() runs the
// whole time loop on the B200 (pq_integrate: state, stage increments and every phi call stay in
// HBM); a std::function source is evaluated on the host through a callback (two vector copies per
// stage), b200::CubicSource (s1 u + s3 u^3, e.g. Allen-Cahn) is evaluated on the device.
#include <cmath>
#include <exception>
#include <functional>
#include <map>
#include <stdexcept>
#include <utility>
#include <vector>

#include "phiquad/b200.hpp"
#include "phiquad/bounds.hpp"
#include "phiquad/kron.hpp"
#include "phiquad/phiaction.hpp"

namespace phiquad {

using SourceFn = std::function<std::vector<double>(double, const std::vector<double>&)>;

struct PhiTerm {
    int k = 1;
    double c = 0.0;
};

struct ExpRKTableau {
    int stages = 1;
    int order = 1;
    std::vector<double> c;
    std::vector<std::vector<std::vector<PhiTerm>>> a;
    std::vector<std::vector<PhiTerm>> b;
};

namespace detail {
inline ExpRKTableau builtin_tableau(int id, double c2) {
    pq_tableau t{};
    b200::check(pq_builtin_tableau(id, c2, &t));
    ExpRKTableau r;
    r.stages = t.stages;
    r.order = t.order;
    r.c.assign(t.c, t.c + t.stages);
    r.a.assign(static_cast<size_t>(t.stages), std::vector<std::vector<PhiTerm>>(static_cast<size_t>(t.stages)));
    r.b.assign(static_cast<size_t>(t.stages), {});
    for (int e = 0; e < t.nterms; ++e) {
        const PhiTerm term{t.k[e], t.coef[e]};
        if (t.row[e] < 0)
            r.b[static_cast<size_t>(t.col[e])].push_back(term);
        else
            r.a[static_cast<size_t>(t.row[e])][static_cast<size_t>(t.col[e])].push_back(term);
    }
    // the reference keeps empty leading rows/columns trimmed the same way (a[i] has i entries)
    for (int i = 0; i < r.stages; ++i) r.a[static_cast<size_t>(i)].resize(static_cast<size_t>(i));
    return r;
}
}  // namespace detail

inline ExpRKTableau exp_euler_tableau() { return detail::builtin_tableau(0, 0.0); }
inline ExpRKTableau exp_rk2_tableau(double c2 = 0.5) {
    if (!(c2 > 0.0 && c2 <= 1.0)) throw std::invalid_argument("exp_rk2_tableau: need c2 in (0,1]");
    return detail::builtin_tableau(1, c2);
}
inline ExpRKTableau exp_rk3_tableau(double c2 = 1.0 / 3.0) {
    if (!(c2 > 0.0 && c2 <= 1.0)) throw std::invalid_argument("exp_rk3_tableau: need c2 in (0,1]");
    return detail::builtin_tableau(2, c2);
}
/// Extension: Krogstad's fourth-order ETDRK4 in the same increment form (BASELINE config 4).
inline ExpRKTableau etdrk4_tableau() { return detail::builtin_tableau(3, 0.0); }

/// phi actions of -sigma tau A, plans cached per (sigma, p) with beta = 1 (reference :81-131).
class PhiEngine {
public:
    PhiEngine(KroneckerSum a, double tau, PhiRequest base) : a_(std::move(a)), tau_(tau), base_(std::move(base)) {
        if (!(tau_ > 0.0)) throw std::invalid_argument("PhiEngine: need tau > 0");
    }
    const KroneckerSum& matrix() const { return a_; }
    double tau() const { return tau_; }
    int calls() const { return calls_; }
    const PhiRequest& request() const { return base_; }
    void add_calls(int n) { calls_ += n; }

    std::vector<PhiColumns> apply(double sigma, int p, const std::vector<std::vector<double>>& bs) {
        const QuadraturePlan& plan = plan_for(sigma, p);
        ++calls_;
        return phi_with_plan(a_.scaled(-sigma * tau_), bs, p, plan.l, plan.n, base_.mode, base_.eps, base_.threads);
    }

private:
    const QuadraturePlan& plan_for(double sigma, int p) {
        const auto key = std::make_pair(sigma, p);
        if (auto it = plans_.find(key); it != plans_.end()) return it->second;
        const double alpha = std::abs(sigma) * tau_ * infnorm_bound(a_);
        CostModel cost = base_.cost;
        cost.d = a_.order();
        QuadraturePlan plan;
        if (base_.l.has_value()) {
            plan.l = *base_.l;
            plan.n = alpha > 0.0 ? quadnodes(base_.eps, p, std::ldexp(alpha, -plan.l), 1.0, base_.mode)
                                 : (base_.mode == QuadKind::gauss_legendre ? 2 : 4);
            plan.cost = cost.cost(plan.n, plan.l, p);
        } else if (alpha > 0.0) {
            plan = setup_quadrature(base_.eps, p, alpha, 1.0, base_.mode, cost);
        } else {
            plan.l = 0;
            plan.n = base_.mode == QuadKind::gauss_legendre ? 2 : 4;
            plan.cost = cost.cost(plan.n, plan.l, p);
        }
        return plans_.emplace(key, plan).first->second;
    }

    KroneckerSum a_;
    double tau_;
    PhiRequest base_;
    std::map<std::pair<double, int>, QuadraturePlan> plans_;
    int calls_ = 0;
};

struct IntegrationResult {
    std::vector<double> u;
    int steps = 0;
    int phi_calls = 0;
};

namespace b200 {
/// Device-evaluated source f(t, u) = s1 u + s3 u^3 (Allen-Cahn: s1 = 1, s3 = -1).
struct CubicSource {
    double s1 = 1.0, s3 = -1.0;
};
}  // namespace b200

namespace detail {

struct FlatTableau {
    std::vector<int> row, col, k;
    std::vector<double> coef;
    pq_tableau t{};
    explicit FlatTableau(const ExpRKTableau& tab) {
        for (size_t i = 0; i < tab.a.size(); ++i)
            for (size_t j = 0; j < tab.a[i].size(); ++j)
                for (const auto& term : tab.a[i][j]) push(static_cast<int>(i), static_cast<int>(j), term);
        for (size_t j = 0; j < tab.b.size(); ++j)
            for (const auto& term : tab.b[j]) push(-1, static_cast<int>(j), term);
        t.stages = tab.stages;
        t.order = tab.order;
        t.c = tab.c.data();
        t.nterms = static_cast<int>(row.size());
        t.row = row.data();
        t.col = col.data();
        t.k = k.data();
        t.coef = coef.data();
    }
    void push(int r, int c, const PhiTerm& term) {
        row.push_back(r);
        col.push_back(c);
        k.push_back(term.k);
        coef.push_back(term.c);
    }
};

// Host callback trampoline for a std::function source; exceptions are carried across the C ABI.
struct SourceCall {
    const SourceFn* f;
    std::exception_ptr error;
    static int invoke(double t, const double* u, double* out, int64_t n, void* user) {
        auto* self = static_cast<SourceCall*>(user);
        try {
            std::vector<double> r = (*self->f)(t, std::vector<double>(u, u + n));
            if (static_cast<int64_t>(r.size()) != n) return 2;
            std::copy(r.begin(), r.end(), out);
            return 0;
        } catch (...) {
            self->error = std::current_exception();
            return 1;
        }
    }
};

inline void rethrow(int rc, const SourceCall& call) {
    if (rc != PQ_OK && call.error) std::rethrow_exception(call.error);
    b200::check(rc);
}

}  // namespace detail

/// One step from (t, u); the engine's tau, matrix and request are used and its call count advanced.
inline std::vector<double> erk_step(PhiEngine& eng, const SourceFn& f, double t, const std::vector<double>& u,
                                    const ExpRKTableau& tab) {
    const auto fl = detail::flatten(eng.matrix());
    const detail::FlatTableau ft(tab);
    const pq_phi_request r = detail::abi_request(eng.request());
    detail::SourceCall call{&f, nullptr};
    pq_source src{PQ_SOURCE_CALLBACK, 0.0, 0.0, nullptr, &detail::SourceCall::invoke, &call};
    if (static_cast<int>(u.size()) != eng.matrix().dim()) throw std::invalid_argument("erk_step: source length mismatch");
    std::vector<double> next(u.size());
    int calls = 0;
    const int rc = pq_erk_step(b200::context(), eng.matrix().order(), fl.shape.data(), fl.data.data(), &src, eng.tau(), t,
                               u.data(), &ft.t, &r, next.data(), &calls, PQ_HOST);
    detail::rethrow(rc, call);
    eng.add_calls(calls);
    return next;
}

/// m equal steps of u' = -A u + f(t, u) from t0 to t_end.
inline IntegrationResult integrate(const KroneckerSum& a, const SourceFn& f, std::vector<double> u, double t0,
                                   double t_end, int m, const ExpRKTableau& tab, const PhiRequest& base = PhiRequest{}) {
    if (m < 1) throw std::invalid_argument("integrate: need at least one step");
    if (!(t_end > t0)) throw std::invalid_argument("integrate: need t_end > t0");
    if (static_cast<int>(u.size()) != a.dim()) throw std::invalid_argument("erk_step: source length mismatch");
    const auto fl = detail::flatten(a);
    const detail::FlatTableau ft(tab);
    const pq_phi_request r = detail::abi_request(base);
    detail::SourceCall call{&f, nullptr};
    pq_source src{PQ_SOURCE_CALLBACK, 0.0, 0.0, nullptr, &detail::SourceCall::invoke, &call};
    std::vector<double> out(u.size());
    int calls = 0;
    const int rc = pq_integrate(b200::context(), a.order(), fl.shape.data(), fl.data.data(), &src, u.data(), t0, t_end, m,
                                &ft.t, &r, out.data(), &calls, PQ_HOST);
    detail::rethrow(rc, call);
    return IntegrationResult{std::move(out), m, calls};
}

/// Overload with the source evaluated on the device (no host round trips per stage).
inline IntegrationResult integrate(const KroneckerSum& a, b200::CubicSource f, std::vector<double> u, double t0,
                                   double t_end, int m, const ExpRKTableau& tab, const PhiRequest& base = PhiRequest{}) {
    if (static_cast<int>(u.size()) != a.dim()) throw std::invalid_argument("erk_step: source length mismatch");
    const auto fl = detail::flatten(a);
    const detail::FlatTableau ft(tab);
    const pq_phi_request r = detail::abi_request(base);
    pq_source src{PQ_SOURCE_CUBIC, f.s1, f.s3, nullptr, nullptr, nullptr};
    std::vector<double> out(u.size());
    int calls = 0;
    b200::check(pq_integrate(b200::context(), a.order(), fl.shape.data(), fl.data.data(), &src, u.data(), t0, t_end, m,
                             &ft.t, &r, out.data(), &calls, PQ_HOST));
    return IntegrationResult{std::move(out), m, calls};
}

}  // namespace phiquad
