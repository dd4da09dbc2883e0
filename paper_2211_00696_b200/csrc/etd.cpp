// Exponential Runge-Kutta time loop on the device (reference integrators.hpp:17-202).
// The state u, the stage increments D_j and every phi call stay in HBM; per stage the host only
// enqueues kernels.  Plans are cached per (sigma, p) with beta = 1 exactly as PhiEngine does.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "engine.hpp"
#include "pq_b200.h"

namespace pqb {
namespace {

struct Term {
    int k;
    double c;
};
struct Tableau {
    int stages = 1, order = 1;
    std::vector<double> c;
    std::vector<std::vector<std::vector<Term>>> a;  // a[i][j] terms
    std::vector<std::vector<Term>> b;               // b[j] terms
};

Tableau unpack(const pq_tableau* t) {
    if (!t || t->stages < 1 || !t->c) throw std::invalid_argument("erk_step: bad tableau");
    Tableau r;
    r.stages = t->stages;
    r.order = t->order;
    r.c.assign(t->c, t->c + t->stages);
    r.a.assign(static_cast<size_t>(t->stages), std::vector<std::vector<Term>>(static_cast<size_t>(t->stages)));
    r.b.assign(static_cast<size_t>(t->stages), {});
    for (int e = 0; e < t->nterms; ++e) {
        const int row = t->row[e], col = t->col[e], k = t->k[e];
        if (col < 0 || col >= t->stages || k < 1) throw std::invalid_argument("erk_step: bad tableau term");
        if (row == -1) {
            r.b[static_cast<size_t>(col)].push_back({k, t->coef[e]});
        } else {
            if (row < 1 || row >= t->stages || col >= row) throw std::invalid_argument("erk_step: tableau must be explicit");
            r.a[static_cast<size_t>(row)][static_cast<size_t>(col)].push_back({k, t->coef[e]});
        }
    }
    return r;
}

// integrators.hpp:81-131 (PhiEngine) on the device.
struct DevPhiEngine {
    pq_ctx& c;
    const DevOp& op;
    double tau;
    pq_phi_request base;
    std::map<std::pair<double, int>, Plan> plans;
    int calls = 0;

    const Plan& plan_for(double sigma, int p) {
        const auto key = std::make_pair(sigma, p);
        auto it = plans.find(key);
        if (it != plans.end()) return it->second;
        double a0 = 0.0;
        for (int k = 0; k < op.d; ++k) a0 += op.inf_norm[k];
        const double alpha = std::abs(sigma) * tau * a0;
        Cost cost{base.c1, base.c2, op.d};
        Plan plan;
        if (base.has_l) {
            plan.l = base.l;
            plan.n = alpha > 0.0 ? node_count(base.eps, p, std::ldexp(alpha, -plan.l), 1.0, base.mode)
                                 : (base.mode == kGauss ? 2 : 4);
            plan.cost = cost(plan.n, plan.l, p);
        } else if (alpha > 0.0) {
            plan = plan_quadrature(base.eps, p, alpha, 1.0, base.mode, cost);
        } else {
            plan.l = 0;
            plan.n = base.mode == kGauss ? 2 : 4;
            plan.cost = cost(plan.n, plan.l, p);
        }
        return plans.emplace(key, plan).first->second;
    }

    // phi_1..phi_p of -sigma*tau*A applied to nb vectors g -> out [nb][p][N]
    void apply(double sigma, int p, int nb, const double* g, double* out) {
        const Plan& plan = plan_for(sigma, p);
        ++calls;
        phi_with_plan_dev(c, op, -sigma * tau, nb, g, p, plan.l, plan.n, base.mode, base.eps, out, nullptr);
    }
};

struct Source {
    pq_source s;
    const double* vec_dev = nullptr;
    std::vector<double> hu, hf;
};

// D = f(t, u) - A u   (integrators.hpp:166-178)
void source_minus(pq_ctx& c, Source& src, double t, const double* u, const double* au, double* D, long long N) {
    switch (src.s.kind) {
        case PQ_SOURCE_ZERO:
            {
                KernelProbe kp(c, "k_cubic_minus", 24.0 * N);
                launch_cubic_minus(N, 0.0, 0.0, u, au, D, c.stream);
            }
            count_launch(c);
            break;
        case PQ_SOURCE_CUBIC:
            {
                KernelProbe kp(c, "k_cubic_minus", 24.0 * N);
                launch_cubic_minus(N, src.s.s1, src.s.s3, u, au, D, c.stream);
            }
            count_launch(c);
            break;
        case PQ_SOURCE_CONSTANT:
            launch_sub(N, src.vec_dev, au, D, c.stream);
            count_launch(c);
            break;
        case PQ_SOURCE_CALLBACK: {
            if (!src.s.cb) throw std::invalid_argument("erk_step: null source callback");
            src.hu.resize(static_cast<size_t>(N));
            src.hf.assign(static_cast<size_t>(N), 0.0);
            cuda_check(cudaMemcpyAsync(src.hu.data(), u, N * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "D2H u");
            cuda_check(cudaStreamSynchronize(c.stream), "callback sync");
            const int rc = src.s.cb(t, src.hu.data(), src.hf.data(), N, src.s.user);
            if (rc == 2) throw std::invalid_argument("erk_step: source length mismatch");
            if (rc != 0) throw std::runtime_error("erk_step: source callback failed");
            double* fd = ws(c, "etd_f", static_cast<size_t>(N));
            cuda_check(cudaMemcpyAsync(fd, src.hf.data(), N * sizeof(double), cudaMemcpyHostToDevice, c.stream), "H2D f");
            cuda_check(cudaStreamSynchronize(c.stream), "callback sync");
            launch_sub(N, fd, au, D, c.stream);
            count_launch(c);
            break;
        }
        default:
            throw std::invalid_argument("erk_step: unknown source kind");
    }
}

// integrators.hpp:141-155: u += tau * sum_k phi_k(-sigma tau A) g_k, g_k = sum_j c D_j.
void apply_phi_group(DevPhiEngine& eng, double sigma, const std::vector<std::vector<Term>>& rows, const double* D,
                     double* u, long long N) {
    pq_ctx& c = eng.c;
    int kmax = 0;
    for (const auto& terms : rows)
        for (const auto& t : terms) kmax = std::max(kmax, t.k);
    if (kmax == 0) return;
    double* g = ws(c, "etd_g", static_cast<size_t>(kmax) * N);
    for (int k = 1; k <= kmax; ++k) {
        std::vector<int> slots;
        std::vector<double> coefs;
        for (size_t j = 0; j < rows.size(); ++j)
            for (const auto& t : rows[j])
                if (t.k == k) {
                    slots.push_back(static_cast<int>(j));
                    coefs.push_back(t.c);
                }
        double* gk = g + static_cast<long long>(k - 1) * N;
        if (slots.empty()) {
            cuda_check(cudaMemsetAsync(gk, 0, N * sizeof(double), c.stream), "zero g");
            continue;
        }
        const int* sl = static_cast<const int*>(arena_push(c, slots.data(), slots.size() * sizeof(int)));
        const double* cf = static_cast<const double*>(arena_push(c, coefs.data(), coefs.size() * sizeof(double)));
        arena_flush(c);
        KernelProbe kp(c, "k_combine(stage)", 8.0 * N * (slots.size() + 1));
        launch_combine(N, 1, static_cast<int>(slots.size()), D, N, sl, cf, gk, N, 1, c.stream);
        count_launch(c);
    }
    // with l = 0 (no squaring) and a Gauss rule, sum_k phi_k(A) g_k is one
    // exp-action per node on the mixed vector sum_k theta^(k-1)/(k-1)! g_k (phi_lincomb,
    // phiaction.hpp:355-389) instead of kmax exp-actions per node and a kmax x kmax column block
    // of which only the diagonal is used.  Same plan, same phi-call count; the sum is rounded in a
    // different order (within the 1e-11 parity bar).  PQ_ETD_LINCOMB=0 keeps the per-column path.
    static const bool lincomb = [] {
        const char* v = std::getenv("PQ_ETD_LINCOMB");
        return !(v && v[0] == '0');
    }();
    const Plan& plan = eng.plan_for(sigma, kmax);
    if (lincomb && plan.l == 0 && eng.base.mode == kGauss) {
        ++eng.calls;
        double* s = ws(c, "etd_lin", static_cast<size_t>(N));
        phi_lincomb_dev(c, eng.op, -sigma * eng.tau, kmax, g, memo_rule(kGauss, plan.n + 1), s);
        KernelProbe kp(c, "k_axpy", 24.0 * N);
        launch_axpy(N, eng.tau, s, u, c.stream);
        count_launch(c);
        return;
    }
    double* cols = ws(c, "etd_cols", static_cast<size_t>(kmax) * kmax * N);
    eng.apply(sigma, kmax, kmax, g, cols);
    for (int k = 1; k <= kmax; ++k) {
        KernelProbe kp(c, "k_axpy", 24.0 * N);
        launch_axpy(N, eng.tau, cols + (static_cast<long long>(k - 1) * kmax + (k - 1)) * N, u, c.stream);
        count_launch(c);
    }
}

// integrators.hpp:160-184
void erk_step_dev(DevPhiEngine& eng, Source& src, double t, const double* u, const Tableau& tab, double* next) {
    pq_ctx& c = eng.c;
    const long long N = eng.op.N;
    double* au = ws(c, "etd_au", static_cast<size_t>(N));
    kron_matvec_dev(c, eng.op, 1.0, u, au);
    double* D = ws(c, "etd_D", static_cast<size_t>(tab.stages) * N);
    source_minus(c, src, t, u, au, D, N);
    for (int i = 1; i < tab.stages; ++i) {
        double* ui = ws(c, "etd_U", static_cast<size_t>(N));
        cuda_check(cudaMemcpyAsync(ui, u, N * sizeof(double), cudaMemcpyDeviceToDevice, c.stream), "copy u");
        apply_phi_group(eng, tab.c[static_cast<size_t>(i)], tab.a[static_cast<size_t>(i)], D, ui, N);
        source_minus(c, src, t + tab.c[static_cast<size_t>(i)] * eng.tau, ui, au, D + static_cast<long long>(i) * N, N);
    }
    cuda_check(cudaMemcpyAsync(next, u, N * sizeof(double), cudaMemcpyDeviceToDevice, c.stream), "copy u");
    apply_phi_group(eng, 1.0, tab.b, D, next, N);
}

// --- built-in tableaus (integrators.hpp:41-76) and ETDRK4 (Krogstad, increment form) ---
struct TabStore {
    std::vector<double> c, coef;
    std::vector<int> row, col, k;
};
void add(TabStore& s, int row, int col, int k, double coef) {
    s.row.push_back(row);
    s.col.push_back(col);
    s.k.push_back(k);
    s.coef.push_back(coef);
}

TabStore make_tableau(int id, double c2, int& stages, int& order) {
    TabStore s;
    if (id == 0) {
        stages = 1;
        order = 1;
        s.c = {0.0};
        add(s, -1, 0, 1, 1.0);
    } else if (id == 1) {
        if (c2 <= 0.0) c2 = 0.5;
        if (!(c2 > 0.0 && c2 <= 1.0)) throw std::invalid_argument("exp_rk2_tableau: need c2 in (0,1]");
        stages = 2;
        order = 2;
        s.c = {0.0, c2};
        add(s, 1, 0, 1, c2);
        add(s, -1, 0, 1, 1.0 - 1.0 / (2.0 * c2));
        add(s, -1, 1, 1, 1.0 / (2.0 * c2));
    } else if (id == 2) {
        if (c2 <= 0.0) c2 = 1.0 / 3.0;
        if (!(c2 > 0.0 && c2 <= 1.0)) throw std::invalid_argument("exp_rk3_tableau: need c2 in (0,1]");
        stages = 3;
        order = 3;
        const double q = 4.0 / (9.0 * c2);
        s.c = {0.0, c2, 2.0 / 3.0};
        add(s, 1, 0, 1, c2);
        add(s, 2, 0, 1, 2.0 / 3.0);
        add(s, 2, 0, 2, -q);
        add(s, 2, 1, 2, q);
        add(s, -1, 0, 1, 1.0);
        add(s, -1, 0, 2, -1.5);
        add(s, -1, 2, 2, 1.5);
    } else if (id == 3) {
        // Krogstad ETDRK4 (Hochbruck-Ostermann tableau), c = (0, 1/2, 1/2, 1); coefficients
        // multiply phi_k(-c_i tau A): a31 = 1/2 phi1 - phi2, a32 = phi2, a41 = phi1 - 2 phi2, a43 = 2 phi2
        stages = 4;
        order = 4;
        s.c = {0.0, 0.5, 0.5, 1.0};
        add(s, 1, 0, 1, 0.5);
        add(s, 2, 0, 1, 0.5);
        add(s, 2, 0, 2, -1.0);
        add(s, 2, 1, 2, 1.0);
        add(s, 3, 0, 1, 1.0);
        add(s, 3, 0, 2, -2.0);
        add(s, 3, 2, 2, 2.0);
        add(s, -1, 0, 1, 1.0);
        add(s, -1, 0, 2, -3.0);
        add(s, -1, 0, 3, 4.0);
        add(s, -1, 1, 2, 2.0);
        add(s, -1, 1, 3, -4.0);
        add(s, -1, 2, 2, 2.0);
        add(s, -1, 2, 3, -4.0);
        add(s, -1, 3, 2, -1.0);
        add(s, -1, 3, 3, 4.0);
    } else {
        throw std::invalid_argument("pq_builtin_tableau: unknown id");
    }
    return s;
}

void check_request(const pq_phi_request* base) {
    if (!base) throw std::invalid_argument("PhiEngine: null request");
    if (base->mode != PQ_GAUSS_LEGENDRE && base->mode != PQ_CLENSHAW_CURTIS)
        throw std::invalid_argument("pq: unknown quadrature kind");
}

}  // namespace
}  // namespace pqb

using namespace pqb;

extern "C" {

PQ_API int pq_builtin_tableau(int id, double c2, pq_tableau* out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("pq_builtin_tableau: null out");
        static std::mutex mu;
        static std::map<std::pair<int, double>, std::unique_ptr<TabStore>> store;
        std::lock_guard<std::mutex> lock(mu);
        int stages = 0, order = 0;
        auto key = std::make_pair(id, c2);
        auto it = store.find(key);
        if (it == store.end()) {
            TabStore s = make_tableau(id, c2, stages, order);
            it = store.emplace(key, std::make_unique<TabStore>(std::move(s))).first;
        }
        const TabStore& s = *it->second;
        out->stages = static_cast<int>(s.c.size());
        out->order = id == 3 ? 4 : id + 1;
        out->c = s.c.data();
        out->nterms = static_cast<int>(s.row.size());
        out->row = s.row.data();
        out->col = s.col.data();
        out->k = s.k.data();
        out->coef = s.coef.data();
    });
}

static int run_etd(pq_ctx* c, int d, const int* shape, const double* factors, const pq_source* f, const double* u0,
                   double t0, double tau, int m, const pq_tableau* tab, const pq_phi_request* base, double* u_out,
                   int* phi_calls, int space) {
    return guarded([&] {
        NvtxRange nvtx(m == 1 ? "pq_erk_step" : "pq_integrate");
        if (!c) throw std::invalid_argument("pq: null context");
        cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
        if (!f) throw std::invalid_argument("erk_step: null source");
        check_request(base);
        if (!(tau > 0.0)) throw std::invalid_argument("PhiEngine: need tau > 0");
        const Tableau tb = unpack(tab);
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "etd_factors");
        const long long N = op.N;
        Source src{*f, nullptr, {}, {}};
        if (f->kind == PQ_SOURCE_CONSTANT) {
            if (!f->vec) throw std::invalid_argument("erk_step: null constant source");
            if (space == PQ_HOST) {
                double* v = ws(*c, "etd_srcvec", static_cast<size_t>(N));
                cuda_check(cudaMemcpyAsync(v, f->vec, N * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D src");
                src.vec_dev = v;
            } else {
                src.vec_dev = f->vec;
            }
        }
        double* ua = ws(*c, "etd_ua", static_cast<size_t>(N));
        double* ub = ws(*c, "etd_ub", static_cast<size_t>(N));
        cuda_check(cudaMemcpyAsync(ua, u0, N * sizeof(double),
                                   space == PQ_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream),
                   "u0");
        DevPhiEngine eng{*c, op, tau, *base, {}, 0};
        // After one eager step (workspaces, plans, exponential caches, kernel attributes all set),
        // two steps u_a -> u_b -> u_a are captured into one CUDA graph and replayed for the rest of
        // the run: the step is device-only for device-side sources (the sources here do not depend
        // on t), so the replay removes the host enqueue of ~60 launches per step.  Any capture
        // failure falls back to eager steps.  PQ_ETD_GRAPH=0 disables.
        static const bool graphs_on = [] {
            const char* e = std::getenv("PQ_ETD_GRAPH");
            return !(e && e[0] == '0');
        }();
        bool try_graph = graphs_on && src.s.kind != PQ_SOURCE_CALLBACK && !c->profiling && !c->trace;
        cudaGraphExec_t pair = nullptr;
        int pair_calls = 0;
        for (int s = 0; s < m;) {
            if (s >= 1 && try_graph && !pair && m - s >= 2) {
                try_graph = false;
                arena_begin(*c);  // a fresh parameter arena: no wrap-around (and its syncs) while capturing
                const int calls0 = eng.calls;
                cudaGraph_t graph = nullptr;
                bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
                if (ok) {
                    try {
                        erk_step_dev(eng, src, t0 + s * tau, ua, tb, ub);
                        erk_step_dev(eng, src, t0 + (s + 1) * tau, ub, tb, ua);
                    } catch (...) {
                        ok = false;
                    }
                    const cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
                    ok = ok && e == cudaSuccess && graph && cudaGraphInstantiate(&pair, graph, 0) == cudaSuccess;
                    if (graph) cudaGraphDestroy(graph);
                }
                if (!ok) {
                    cudaGetLastError();
                    if (pair) cudaGraphExecDestroy(pair);
                    pair = nullptr;
                    eng.calls = calls0;  // nothing captured ran: redo these steps eagerly
                    continue;
                }
                pair_calls = eng.calls - calls0;
                cuda_check(cudaGraphLaunch(pair, c->stream), "graph launch");
                s += 2;
                continue;
            }
            if (pair && m - s >= 2) {
                cuda_check(cudaGraphLaunch(pair, c->stream), "graph launch");
                eng.calls += pair_calls;
                s += 2;
                continue;
            }
            erk_step_dev(eng, src, t0 + s * tau, ua, tb, ub);
            std::swap(ua, ub);
            ++s;
        }
        if (pair) {
            cuda_check(cudaStreamSynchronize(c->stream), "graph drain");
            cudaGraphExecDestroy(pair);
            // events recorded while capturing are not real records: re-arm the arena's
            if (c->arena.done) cuda_check(cudaEventRecord(c->arena.done, c->stream), "arena record");
        }
        cuda_check(cudaMemcpyAsync(u_out, ua, N * sizeof(double),
                                   space == PQ_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream),
                   "u out");
        if (space == PQ_HOST) cuda_check(cudaStreamSynchronize(c->stream), "sync");
        if (phi_calls) *phi_calls = eng.calls;
    });
}

PQ_API int pq_integrate(pq_ctx* c, int d, const int* shape, const double* factors, const pq_source* f, const double* u0,
                        double t0, double t_end, int m, const pq_tableau* tab, const pq_phi_request* base,
                        double* u_out, int* phi_calls, int space) {
    if (m < 1) {
        last_error_slot() = "integrate: need at least one step";
        return PQ_EINVAL;
    }
    if (!(t_end > t0)) {
        last_error_slot() = "integrate: need t_end > t0";
        return PQ_EINVAL;
    }
    return run_etd(c, d, shape, factors, f, u0, t0, (t_end - t0) / m, m, tab, base, u_out, phi_calls, space);
}

PQ_API int pq_erk_step(pq_ctx* c, int d, const int* shape, const double* factors, const pq_source* f, double tau,
                       double t, const double* u, const pq_tableau* tab, const pq_phi_request* base, double* u_out,
                       int* phi_calls, int space) {
    return run_etd(c, d, shape, factors, f, u, t, tau, 1, tab, base, u_out, phi_calls, space);
}

}  // extern "C"
