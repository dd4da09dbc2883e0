// TEST INFRASTRUCTURE ONLY — the compiled reference, used as the parity checker and as the
// `--impl reference` CPU arm of bench.py.  Nothing in the product (paper_2211_00696_b200/,
// include/) links or loads this.
//
// This file is our own flat `extern "C"` shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/phiquad/*.hpp, compiled where they lie by oracle/Makefile);
// no reference source is copied into the repo.  Each entry point names the reference
// symbol it forwards to.  Errors: the reference throws; the shim maps exception types to
// the same return codes as the product's C ABI (include/pq_b200.h):
//   0 ok, 1 std::invalid_argument, 2 phiquad::ConvergenceError, 3 std::runtime_error,
//   4 std::out_of_range, 5 anything else.
#include <phiquad/phiquad.hpp>

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

using namespace phiquad;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConvergenceError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 4;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

// factors: concatenation of d row-major n_k x n_k blocks.
KroneckerSum make_sum(int d, const int* shape, const double* factors) {
    std::vector<DenseMatrix> fs;
    size_t off = 0;
    for (int k = 0; k < d; ++k) {
        const size_t nn = static_cast<size_t>(shape[k]) * shape[k];
        fs.emplace_back(shape[k], shape[k], std::vector<double>(factors + off, factors + off + nn));
        off += nn;
    }
    return KroneckerSum(std::move(fs));
}

std::vector<DenseMatrix> make_list(int d, const int* shape, const double* factors) {
    std::vector<DenseMatrix> fs;
    size_t off = 0;
    for (int k = 0; k < d; ++k) {
        const size_t nn = static_cast<size_t>(shape[k]) * shape[k];
        fs.emplace_back(shape[k], shape[k], std::vector<double>(factors + off, factors + off + nn));
        off += nn;
    }
    return fs;
}

long long prod(int d, const int* shape) {
    long long p = 1;
    for (int k = 0; k < d; ++k) p *= shape[k];
    return p;
}

std::vector<std::vector<double>> split(const double* bs, int nb, long long n) {
    std::vector<std::vector<double>> out;
    for (int m = 0; m < nb; ++m) out.emplace_back(bs + m * n, bs + (m + 1) * n);
    return out;
}

// out layout: [nb][p][N]
void store_cols(const std::vector<PhiColumns>& ys, double* out, long long n) {
    size_t o = 0;
    for (const auto& y : ys)
        for (const auto& c : y.cols) {
            std::memcpy(out + o, c.data(), sizeof(double) * n);
            o += n;
        }
}

QuadKind kind_of(int k) { return k == 0 ? QuadKind::gauss_legendre : QuadKind::clenshaw_curtis; }

// Tableau ids: 0 exp-Euler, 1 exp-RK2(c2), 2 exp-RK3(c2), 3 ETDRK4 (Cox-Matthews / Krogstad
// form restated below in the reference's increment-form ExpRKTableau).
ExpRKTableau tableau_of(int id, double c2) {
    switch (id) {
    case 0: return exp_euler_tableau();
    case 1: return exp_rk2_tableau(c2 > 0 ? c2 : 0.5);
    case 2: return exp_rk3_tableau(c2 > 0 ? c2 : 1.0 / 3.0);
    default: break;
    }
    // Krogstad's fourth-order ETDRK4 (Hochbruck-Ostermann 2005 tableau), written in the
    // reference's increment form (PhiTerm coefficients multiply phi_k(-c_i tau A), rows sum to
    // c_i phi_1), c = (0, 1/2, 1/2, 1):
    //   a21 = 1/2 phi1;  a31 = 1/2 phi1 - phi2, a32 = phi2   (phi_k at -tau A/2)
    //   a41 = phi1 - 2 phi2, a43 = 2 phi2                    (phi_k at -tau A)
    //   b1 = phi1 - 3 phi2 + 4 phi3, b2 = b3 = 2 phi2 - 4 phi3, b4 = 4 phi3 - phi2.
    // Order 4 checked numerically (tests/test_gpu_configs.py::test_config4_etdrk4_is_fourth_order).
    ExpRKTableau t;
    t.stages = 4;
    t.order = 4;
    t.c = {0.0, 0.5, 0.5, 1.0};
    t.a = {{},
           {{PhiTerm{1, 0.5}}},
           {{PhiTerm{1, 0.5}, PhiTerm{2, -1.0}}, {PhiTerm{2, 1.0}}},
           {{PhiTerm{1, 1.0}, PhiTerm{2, -2.0}}, {}, {PhiTerm{2, 2.0}}}};
    t.b = {{PhiTerm{1, 1.0}, PhiTerm{2, -3.0}, PhiTerm{3, 4.0}},
           {PhiTerm{2, 2.0}, PhiTerm{3, -4.0}},
           {PhiTerm{2, 2.0}, PhiTerm{3, -4.0}},
           {PhiTerm{2, -1.0}, PhiTerm{3, 4.0}}};
    return t;
}

// Source ids: 0 f = 0, 1 Allen-Cahn f(u) = u - u^3, 2 constant vector (param array).
SourceFn source_of(int id, const double* data, long long n) {
    if (id == 1)
        return [](double, const std::vector<double>& u) {
            std::vector<double> r(u.size());
            for (size_t i = 0; i < u.size(); ++i) r[i] = u[i] - u[i] * u[i] * u[i];
            return r;
        };
    if (id == 2) {
        std::vector<double> c(data, data + n);
        return [c](double, const std::vector<double>&) { return c; };
    }
    return [n](double, const std::vector<double>&) { return std::vector<double>(n, 0.0); };
}

} // namespace

extern "C" {

const char* pqref_last_error() { return g_err.c_str(); }

// quadrature.hpp:31 gauss_legendre / :67 clenshaw_curtis
int pqref_rule(int kind, int m, double* nodes, double* weights) {
    return guarded([&] {
        QuadratureRule r = kind == 0 ? gauss_legendre(m) : clenshaw_curtis(m);
        std::memcpy(nodes, r.nodes.data(), sizeof(double) * m);
        std::memcpy(weights, r.weights.data(), sizeof(double) * m);
    });
}

// roots.hpp:34 quartic_roots (re/im interleaved, 8 doubles)
int pqref_quartic_roots(double a3, double a2, double a1, double a0, double* out8) {
    return guarded([&] {
        MonicQuartic q{a3, a2, a1, a0};
        auto z = quartic_roots(q);
        for (int k = 0; k < 4; ++k) {
            out8[2 * k] = z[k].real();
            out8[2 * k + 1] = z[k].imag();
        }
    });
}

// roots.hpp:88 real_roots_greater_one; returns count in *cnt (<= 4)
int pqref_real_roots_greater_one(double a3, double a2, double a1, double a0, double* out4, int* cnt) {
    return guarded([&] {
        auto r = real_roots_greater_one(MonicQuartic{a3, a2, a1, a0});
        *cnt = static_cast<int>(r.size());
        for (size_t i = 0; i < r.size(); ++i) out4[i] = r[i];
    });
}

// bounds.hpp:71 / :88 / :107 / :122 / :146
int pqref_log_bound_at_rho(double n, int p, double alpha, double beta, int kind, double rho, double* out) {
    return guarded([&] { *out = log_bound_at_rho(BoundQuery{n, p, alpha, beta, kind_of(kind)}, rho); });
}
int pqref_bound_quartic(double n, int p, double alpha, double beta, int kind, double* out4) {
    return guarded([&] {
        auto q = bound_quartic(BoundQuery{n, p, alpha, beta, kind_of(kind)});
        out4[0] = q.a3; out4[1] = q.a2; out4[2] = q.a1; out4[3] = q.a0;
    });
}
int pqref_theorem_bound(double n, int p, double alpha, double beta, int kind, double* out) {
    return guarded([&] { *out = theorem_bound(BoundQuery{n, p, alpha, beta, kind_of(kind)}); });
}
int pqref_corollary_bound(double n, int p, double alpha, double beta, int kind, double* out) {
    return guarded([&] { *out = corollary_bound(BoundQuery{n, p, alpha, beta, kind_of(kind)}); });
}
int pqref_quaderr(double n, int p, double alpha, double beta, int kind, double* out) {
    return guarded([&] { *out = quaderr(n, p, alpha, beta, kind_of(kind)); });
}
// bounds.hpp:159
int pqref_quadnodes(double eps, int p, double alpha, double beta, int kind, int* n) {
    return guarded([&] { *n = quadnodes(eps, p, alpha, beta, kind_of(kind)); });
}
// bounds.hpp:185
int pqref_setup_quadrature(double eps, int p, double alpha, double beta, int kind, double c1,
                           double c2, int d, int* l, int* n, double* cost) {
    return guarded([&] {
        CostModel cm{c1, c2, d};
        auto plan = setup_quadrature(eps, p, alpha, beta, kind_of(kind), cm);
        *l = plan.l;
        *n = plan.n;
        *cost = plan.cost;
    });
}

// dense.hpp:194
int pqref_expm(int n, const double* a, double* out) {
    return guarded([&] {
        DenseMatrix m(n, n, std::vector<double>(a, a + static_cast<size_t>(n) * n));
        DenseMatrix e = expm(m);
        std::memcpy(out, e.data(), sizeof(double) * n * n);
    });
}

// kron.hpp:92
int pqref_mode_apply(int d, const int* shape, const double* factors, const double* x, double* y) {
    return guarded([&] {
        const long long n = prod(d, shape);
        std::vector<int> sh(shape, shape + d);
        auto r = mode_apply(make_list(d, shape, factors), sh, std::vector<double>(x, x + n));
        std::memcpy(y, r.data(), sizeof(double) * n);
    });
}

// kron.hpp:111
int pqref_kron_matvec(int d, const int* shape, const double* factors, const double* x, double* y) {
    return guarded([&] {
        const long long n = prod(d, shape);
        auto r = kron_matvec(make_sum(d, shape, factors), std::vector<double>(x, x + n));
        std::memcpy(y, r.data(), sizeof(double) * n);
    });
}

// kron.hpp:123
int pqref_exp_action(int d, const int* shape, const double* factors, const double* b, double* y) {
    return guarded([&] {
        const long long n = prod(d, shape);
        auto r = exp_action(make_sum(d, shape, factors), std::vector<double>(b, b + n));
        std::memcpy(y, r.data(), sizeof(double) * n);
    });
}

// kron.hpp:131
int pqref_infnorm_bound(int d, const int* shape, const double* factors, double* out) {
    return guarded([&] { *out = infnorm_bound(make_sum(d, shape, factors)); });
}

// phiaction.hpp:134 phi_fixed_multi on cached_rule(kind, points)
int pqref_phi_fixed(int d, const int* shape, const double* factors, int nb, const double* bs,
                    int p, int kind, int points, int threads, double* out) {
    return guarded([&] {
        const long long n = prod(d, shape);
        auto ys = phi_fixed_multi(make_sum(d, shape, factors), split(bs, nb, n), p,
                                  cached_rule(kind_of(kind), points), threads);
        store_cols(ys, out, n);
    });
}

// phiaction.hpp:156
int pqref_phi_adaptive(int d, const int* shape, const double* factors, int nb, const double* bs,
                       int p, double eps, int threads, double* out, int* points_used) {
    return guarded([&] {
        const long long n = prod(d, shape);
        auto ys = phi_adaptive_multi(make_sum(d, shape, factors), split(bs, nb, n), p, eps,
                                     threads, points_used);
        store_cols(ys, out, n);
    });
}

// phiaction.hpp:255 — y: [p][N] in/out; exps: d factors
int pqref_squaring_step(int d, const int* shape, const double* exps, int p, double* y) {
    return guarded([&] {
        const long long n = prod(d, shape);
        PhiColumns cols;
        cols.dim = static_cast<int>(n);
        for (int j = 0; j < p; ++j) cols.cols.emplace_back(y + j * n, y + (j + 1) * n);
        squaring_step(cols, make_list(d, shape, exps), std::vector<int>(shape, shape + d));
        store_cols({cols}, y, n);
    });
}

// phiaction.hpp:277
int pqref_phi_with_plan(int d, const int* shape, const double* factors, int nb, const double* bs,
                        int p, int l, int n_param, int kind, double eps, int threads, double* out,
                        int* points_used) {
    return guarded([&] {
        const long long n = prod(d, shape);
        auto ys = phi_with_plan(make_sum(d, shape, factors), split(bs, nb, n), p, l, n_param,
                                kind_of(kind), eps, threads, points_used);
        store_cols(ys, out, n);
    });
}

// phiaction.hpp:307.  has_l < 0 means "planned".  info6 = {l, n, points, planned, alpha, beta},
// info_cost = plan_cost.
int pqref_phiquadmv(int d, const int* shape, const double* factors, int nb, const double* bs,
                    int p, double eps, int kind, int fixed_l, double c1, double c2, int threads,
                    double* out, int* info_int4, double* info_dbl3) {
    return guarded([&] {
        const long long n = prod(d, shape);
        PhiRequest req;
        req.p = p;
        req.eps = eps;
        req.mode = kind_of(kind);
        if (fixed_l >= 0) req.l = fixed_l;
        req.cost.c1 = c1;
        req.cost.c2 = c2;
        req.threads = threads;
        PhiInfo info;
        auto ys = phiquadmv_multi(make_sum(d, shape, factors), split(bs, nb, n), req, &info);
        store_cols(ys, out, n);
        info_int4[0] = info.l;
        info_int4[1] = info.n;
        info_int4[2] = info.points;
        info_int4[3] = info.planned ? 1 : 0;
        info_dbl3[0] = info.alpha;
        info_dbl3[1] = info.beta;
        info_dbl3[2] = info.plan_cost;
    });
}

// phiaction.hpp:355
int pqref_phi_lincomb(int d, const int* shape, const double* factors, int p, const double* bs,
                      int kind, int points, int threads, double* out) {
    return guarded([&] {
        const long long n = prod(d, shape);
        auto y = phi_lincomb(make_sum(d, shape, factors), split(bs, p, n),
                             cached_rule(kind_of(kind), points), threads);
        std::memcpy(out, y.data(), sizeof(double) * n);
    });
}

// oracle.hpp:41 (assembled dense augmented-matrix expm; guard N+p <= 1000 by default)
int pqref_phi_dense_oracle(int d, const int* shape, const double* factors, const double* b, int p,
                           int guard, double* out) {
    return guarded([&] {
        const long long n = prod(d, shape);
        auto cols = phi_dense_oracle(make_sum(d, shape, factors), std::vector<double>(b, b + n), p,
                                     guard);
        for (int j = 0; j < p; ++j) std::memcpy(out + j * n, cols[j].data(), sizeof(double) * n);
    });
}

// integrators.hpp:193 integrate; *phi_calls = PhiEngine::calls()
int pqref_integrate(int d, const int* shape, const double* factors, int source, const double* src_data,
                    const double* u0, double t0, double t_end, int m, int tableau, double c2,
                    double eps, int kind, int threads, double* u_out, int* phi_calls) {
    return guarded([&] {
        const long long n = prod(d, shape);
        PhiRequest base;
        base.eps = eps;
        base.mode = kind_of(kind);
        base.threads = threads;
        auto res = integrate(make_sum(d, shape, factors), source_of(source, src_data, n),
                             std::vector<double>(u0, u0 + n), t0, t_end, m, tableau_of(tableau, c2),
                             base);
        std::memcpy(u_out, res.u.data(), sizeof(double) * n);
        *phi_calls = res.phi_calls;
    });
}

// problems.hpp:63 fe_laplacian_1d (fixture builder)
int pqref_fe_laplacian_1d(int n_elem, double* out) {
    return guarded([&] {
        auto m = fe_laplacian_1d(n_elem);
        std::memcpy(out, m.data(), sizeof(double) * m.rows() * m.cols());
    });
}

} // extern "C"
