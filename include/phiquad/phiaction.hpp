#pragma once
// The phi engine (reference phiaction.hpp:20-389) on the B200.  Same types and signatures; the
// node sweep, combine, modified squaring and phi_0 run as sm_100a kernels behind pq_*.  `threads`
// is accepted and ignored: results are bitwise independent of it, as in the reference.
#include <optional>
#include <stdexcept>
#include <vector>

#include "phiquad/b200.hpp"
#include "phiquad/bounds.hpp"
#include "phiquad/dense.hpp"
#include "phiquad/kron.hpp"
#include "phiquad/quadrature.hpp"
#include "phiquad/util.hpp"

namespace phiquad {

struct PhiColumns {
    int dim = 0;
    std::vector<std::vector<double>> cols;
    int p() const { return static_cast<int>(cols.size()); }
    const std::vector<double>& col(int j) const {
        if (j < 1 || j > p()) throw std::out_of_range("PhiColumns::col: index out of range");
        return cols[static_cast<size_t>(j - 1)];
    }
};

struct PhiRequest {
    int p = 1;
    double eps = 1e-14;
    QuadKind mode = QuadKind::gauss_legendre;
    std::optional<int> l;
    CostModel cost;
    int threads = 1;
};

struct PhiInfo {
    int l = 0;
    int n = 0;
    int points = 0;
    QuadKind mode = QuadKind::gauss_legendre;
    double alpha = 0.0;
    double beta = 0.0;
    bool planned = false;
    double plan_cost = 0.0;
};

namespace detail {

inline std::vector<double> gather(const std::vector<std::vector<double>>& bs, int dim, const char* who) {
    std::vector<double> flat;
    flat.reserve(bs.size() * static_cast<size_t>(dim));
    for (const auto& b : bs) {
        if (static_cast<int>(b.size()) != dim) throw std::invalid_argument(std::string(who) + ": vector length mismatch");
        flat.insert(flat.end(), b.begin(), b.end());
    }
    return flat;
}

inline std::vector<PhiColumns> scatter(const std::vector<double>& flat, int nb, int p, int dim) {
    std::vector<PhiColumns> out(static_cast<size_t>(nb));
    for (int m = 0; m < nb; ++m) {
        out[static_cast<size_t>(m)].dim = dim;
        for (int j = 0; j < p; ++j) {
            const auto* s = flat.data() + (static_cast<size_t>(m) * p + j) * dim;
            out[static_cast<size_t>(m)].cols.emplace_back(s, s + dim);
        }
    }
    return out;
}

// The result columns, allocated (and value-initialised, as std::vector must) by several threads:
// first-touching tens of MB from one thread costs more than the device computation at these sizes
// (config 2: 67 MB, ~24 ms single-threaded on the B200 box's host vs ~3.4 ms for the phi call).
inline std::vector<PhiColumns> alloc_columns(int nb, int p, int dim) {
    std::vector<PhiColumns> out(static_cast<size_t>(nb));
    for (auto& pc : out) {
        pc.dim = dim;
        pc.cols.resize(static_cast<size_t>(p));
    }
    const int count = nb * p;
    const int threads = static_cast<long long>(dim) * count >= (1LL << 20) ? std::min(count, 8) : 1;
    parallel_for(count, threads, [&](int k) {
        out[static_cast<size_t>(k / p)].cols[static_cast<size_t>(k % p)] = b200::result_vector(static_cast<size_t>(dim));
    });
    return out;
}

inline pq_phi_request abi_request(const PhiRequest& r) {
    pq_phi_request c{};
    c.p = r.p;
    c.eps = r.eps;
    c.mode = abi_kind(r.mode);
    c.has_l = r.l.has_value() ? 1 : 0;
    c.l = r.l.value_or(0);
    c.c1 = r.cost.c1;
    c.c2 = r.cost.c2;
    c.threads = r.threads;
    return c;
}

}  // namespace detail

inline std::vector<PhiColumns> phi_fixed_multi(const KroneckerSum& a, const std::vector<std::vector<double>>& bs, int p,
                                               const QuadratureRule& rule, int threads = 1) {
    (void)threads;
    if (p < 1) throw std::invalid_argument("phi_fixed: need p >= 1");
    const int dim = a.dim();
    std::vector<const double*> ptrs;
    for (const auto& b : bs) {
        if (static_cast<int>(b.size()) != dim) throw std::invalid_argument("phi_fixed: vector length mismatch");
        ptrs.push_back(b.data());
    }
    const auto f = detail::flatten(a);
    const int nb = static_cast<int>(bs.size());
    // read each b in place and write straight into the returned PhiColumns (pq_phi_fixed_cols)
    std::vector<PhiColumns> out = detail::alloc_columns(nb, p, dim);
    std::vector<double*> cols;
    for (auto& pc : out)
        for (auto& c : pc.cols) cols.push_back(c.data());
    b200::check(pq_phi_fixed_cols(b200::context(), a.order(), f.shape.data(), f.data.data(), nb, ptrs.data(), p,
                                  rule.points(), rule.nodes.data(), rule.weights.data(), cols.data(), PQ_HOST));
    return out;
}

inline PhiColumns phi_fixed(const KroneckerSum& a, const std::vector<double>& b, int p, const QuadratureRule& rule,
                            int threads = 1) {
    return std::move(phi_fixed_multi(a, {b}, p, rule, threads).front());
}

inline std::vector<PhiColumns> phi_adaptive_multi(const KroneckerSum& a, const std::vector<std::vector<double>>& bs,
                                                  int p, double eps, int threads = 1, int* points_used = nullptr) {
    (void)threads;
    if (p < 1) throw std::invalid_argument("phi_adaptive: need p >= 1");
    if (!(eps > 0.0)) throw std::invalid_argument("phi_adaptive: need eps > 0");
    const int dim = a.dim();
    std::vector<const double*> ptrs;
    for (const auto& b : bs) {
        if (static_cast<int>(b.size()) != dim) throw std::invalid_argument("phi_adaptive: vector length mismatch");
        ptrs.push_back(b.data());
    }
    const auto f = detail::flatten(a);
    const int nb = static_cast<int>(bs.size());
    std::vector<PhiColumns> out = detail::alloc_columns(nb, p, dim);
    std::vector<double*> cols;
    for (auto& pc : out)
        for (auto& c : pc.cols) cols.push_back(c.data());
    int pts = 0;
    b200::check(pq_phi_adaptive_cols(b200::context(), a.order(), f.shape.data(), f.data.data(), nb, ptrs.data(), p, eps,
                                     cols.data(), &pts, PQ_HOST));
    if (points_used) *points_used = pts;
    return out;
}

inline PhiColumns phi_adaptive(const KroneckerSum& a, const std::vector<double>& b, int p, double eps, int threads = 1,
                               int* points_used = nullptr) {
    return std::move(phi_adaptive_multi(a, {b}, p, eps, threads, points_used).front());
}

/// phi_i(2A) b = 2^-i (e^A phi_i(A) b + sum_{j<=i} phi_j(A) b/(i-j)!), in place.
inline void squaring_step(PhiColumns& y, const std::vector<DenseMatrix>& exps, const std::vector<int>& shape) {
    const int p = y.p();
    if (p == 0) return;
    // the reference's mode_apply checks, in its order (kron.hpp:92-102)
    if (exps.size() != shape.size()) throw std::invalid_argument("mode_apply: rank mismatch");
    const long long dim = detail::shape_product(shape);
    std::vector<double*> cols;
    for (auto& c : y.cols) {
        if (static_cast<long long>(c.size()) != dim) throw std::invalid_argument("mode_apply: vector length mismatch");
        cols.push_back(c.data());
    }
    for (size_t k = 0; k < exps.size(); ++k)
        if (exps[k].rows() != shape[k]) throw std::invalid_argument("mode_apply: factor extent mismatch");
    const auto f = detail::flatten(exps);
    // the columns are rewritten in place (pq_squaring_step_cols): no flattening copy
    b200::check(pq_squaring_step_cols(b200::context(), static_cast<int>(shape.size()), shape.data(), f.data.data(), p,
                                      cols.data(), PQ_HOST));
}

inline std::vector<PhiColumns> phi_with_plan(const KroneckerSum& a, const std::vector<std::vector<double>>& bs, int p,
                                             int l, int n, QuadKind mode, double eps, int threads = 1,
                                             int* points_used = nullptr) {
    (void)threads;
    // argument checks in the reference's order (phiaction.hpp:281-290 -> cached_rule -> phi_fixed_multi /
    // phi_adaptive_multi); the C ABI repeats them, the vector lengths are only known here
    if (l < 0) throw std::invalid_argument("phi_with_plan: need l >= 0");
    const bool gauss = mode == QuadKind::gauss_legendre;
    if (gauss && n + 1 < 1) throw std::invalid_argument("gauss_legendre: need at least one point");
    if (p < 1) throw std::invalid_argument(gauss ? "phi_fixed: need p >= 1" : "phi_adaptive: need p >= 1");
    if (!gauss && !(eps > 0.0)) throw std::invalid_argument("phi_adaptive: need eps > 0");
    const int dim = a.dim();
    std::vector<const double*> ptrs;
    for (const auto& b : bs) {
        if (static_cast<int>(b.size()) != dim)
            throw std::invalid_argument(std::string(gauss ? "phi_fixed" : "phi_adaptive") + ": vector length mismatch");
        ptrs.push_back(b.data());
    }
    const auto f = detail::flatten(a);
    const int nb = static_cast<int>(bs.size());
    std::vector<PhiColumns> out = detail::alloc_columns(nb, p, dim);
    std::vector<double*> cols;
    for (auto& pc : out)
        for (auto& c : pc.cols) cols.push_back(c.data());
    int pts = 0;
    b200::check(pq_phi_with_plan_cols(b200::context(), a.order(), f.shape.data(), f.data.data(), nb, ptrs.data(), p, l,
                                      n, abi_kind(mode), eps, cols.data(), &pts, PQ_HOST));
    if (points_used) *points_used = pts;
    return out;
}

namespace detail {

// phiquadmv on the caller's vectors in place: b_m read from its own storage, phi_j written straight
// into the PhiColumns vectors (pq_phiquadmv_cols) -- no flattening or scattering copies
inline std::vector<PhiColumns> phiquadmv_ptrs(const KroneckerSum& a, const std::vector<const double*>& bs,
                                              const PhiRequest& req, PhiInfo* info) {
    if (req.p < 1) throw std::invalid_argument("phiquadmv: need p >= 1");
    const int dim = a.dim();
    const int nb = static_cast<int>(bs.size());
    const auto f = detail::flatten(a);
    const pq_phi_request r = detail::abi_request(req);
    pq_phi_info pi{};
    std::vector<PhiColumns> out = alloc_columns(nb, req.p, dim);
    std::vector<double*> cols;
    cols.reserve(static_cast<size_t>(nb) * req.p);
    for (auto& pc : out)
        for (auto& c : pc.cols) cols.push_back(c.data());
    b200::check(pq_phiquadmv_cols(b200::context(), a.order(), f.shape.data(), f.data.data(), nb, bs.data(), &r,
                                  cols.data(), &pi, PQ_HOST));
    if (info)
        *info = PhiInfo{pi.l,     pi.n,    pi.points,          pi.mode == PQ_GAUSS_LEGENDRE ? QuadKind::gauss_legendre
                                                                                         : QuadKind::clenshaw_curtis,
                        pi.alpha, pi.beta, pi.planned != 0, pi.plan_cost};
    return out;
}

}  // namespace detail

inline std::vector<PhiColumns> phiquadmv_multi(const KroneckerSum& a, const std::vector<std::vector<double>>& bs,
                                               const PhiRequest& req, PhiInfo* info = nullptr) {
    // reference order (phiaction.hpp:307-346): p, then the pinned l, then phi_with_plan's checks --
    // eps for the adaptive rule and the vector lengths in phi_fixed_multi / phi_adaptive_multi
    if (req.p < 1) throw std::invalid_argument("phiquadmv: need p >= 1");
    if (req.l.has_value() && *req.l < 0) throw std::invalid_argument("phiquadmv: need l >= 0");
    const bool gauss = req.mode == QuadKind::gauss_legendre;
    if (!gauss && !(req.eps > 0.0)) throw std::invalid_argument("phi_adaptive: need eps > 0");
    std::vector<const double*> ptrs;
    for (const auto& b : bs) {
        if (static_cast<long long>(b.size()) != static_cast<long long>(a.dim()))
            throw std::invalid_argument(std::string(gauss ? "phi_fixed" : "phi_adaptive") + ": vector length mismatch");
        ptrs.push_back(b.data());
    }
    return detail::phiquadmv_ptrs(a, ptrs, req, info);  // no right-hand sides: the plan only, no columns
}

// = phiquadmv_multi(a, {b}, req, info).front() (phiaction.hpp:343-346) without copying b into a
// temporary batch (16.8 MB at config 2: 3-4 ms of host time, more than the device's share)
inline PhiColumns phiquadmv(const KroneckerSum& a, const std::vector<double>& b, const PhiRequest& req,
                            PhiInfo* info = nullptr) {
    if (req.p < 1) throw std::invalid_argument("phiquadmv: need p >= 1");
    if (req.l.has_value() && *req.l < 0) throw std::invalid_argument("phiquadmv: need l >= 0");
    const bool gauss = req.mode == QuadKind::gauss_legendre;
    if (!gauss && !(req.eps > 0.0)) throw std::invalid_argument("phi_adaptive: need eps > 0");
    if (static_cast<long long>(b.size()) != static_cast<long long>(a.dim()))
        throw std::invalid_argument(std::string(gauss ? "phi_fixed" : "phi_adaptive") + ": vector length mismatch");
    return std::move(detail::phiquadmv_ptrs(a, {b.data()}, req, info).front());
}

/// sum_j phi_j(A) b_j in one quadrature sweep (no scaling/squaring).
inline std::vector<double> phi_lincomb(const KroneckerSum& a, const std::vector<std::vector<double>>& bs,
                                       const QuadratureRule& rule, int threads = 1) {
    (void)threads;
    if (bs.empty()) throw std::invalid_argument("phi_lincomb: need at least one vector");
    const int dim = a.dim();
    const auto flat = detail::gather(bs, dim, "phi_lincomb");
    const auto f = detail::flatten(a);
    std::vector<double> y = b200::result_vector(static_cast<size_t>(dim));
    b200::check(pq_phi_lincomb(b200::context(), a.order(), f.shape.data(), f.data.data(), static_cast<int>(bs.size()),
                               flat.data(), rule.points(), rule.nodes.data(), rule.weights.data(), y.data(), PQ_HOST));
    return y;
}

}  // namespace phiquad
