// Host estimator for the phi engine (see estimator.hpp).  The planner's integers (l, n) must
// equal the reference's on identical inputs, so every floating-point expression below keeps the
// evaluation order of the corresponding reference expression (cited per function); the code is
// otherwise organised our own way.  Compiled with g++ -O3 and no -ffast-math / -mfma so that
// no contraction changes a rounding.
#include "estimator.hpp"

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <numbers>

namespace pqb {

namespace {
constexpr double kPi = std::numbers::pi;
constexpr double kLn2 = std::numbers::ln2;
constexpr double kInf = std::numeric_limits<double>::infinity();

void require(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(what);
}
}  // namespace

// ---------------------------------------------------------------- rules (quadrature.hpp) ----

// Legendre P_m and its derivative at x by the three-term recurrence; returns {P_m, P_{m-1}}.
static inline void legendre_pair(int m, double x, double& pm, double& pm1) {
    double cur = 1.0, prev = 0.0;
    for (int k = 0; k < m; ++k) {
        const double older = prev;
        prev = cur;
        cur = ((2.0 * k + 1.0) * x * prev - k * older) / (k + 1.0);
    }
    pm = cur;
    pm1 = prev;
}

// quadrature.hpp:31-62: Newton on P_m from Chebyshev-angle guesses, symmetric fill on [0,1].
NodesWeights gauss_legendre01(int m) {
    require(m >= 1, "gauss_legendre: need at least one point");
    NodesWeights r;
    r.x.assign(static_cast<size_t>(m), 0.0);
    r.w.assign(static_cast<size_t>(m), 0.0);
    for (int i = 0; i < (m + 1) / 2; ++i) {
        double x = std::cos(kPi * (i + 0.75) / (m + 0.5));
        double slope = 0.0;
        for (int it = 0; it < 100; ++it) {
            double pm, pm1;
            legendre_pair(m, x, pm, pm1);
            slope = m * (x * pm - pm1) / (x * x - 1.0);
            const double dx = pm / slope;
            x -= dx;
            if (std::abs(dx) <= 1e-15 * (1.0 + std::abs(x))) break;
        }
        const double wt = 2.0 / ((1.0 - x * x) * slope * slope);
        const size_t lo = static_cast<size_t>(i), hi = static_cast<size_t>(m - 1 - i);
        r.x[lo] = 0.5 * (1.0 - x);
        r.w[lo] = 0.5 * wt;
        r.x[hi] = 0.5 * (1.0 + x);
        r.w[hi] = 0.5 * wt;
    }
    return r;
}

// quadrature.hpp:67-86: mapped Chebyshev extrema, cosine-sum weights (nested m -> 2m-1).
NodesWeights clenshaw_curtis01(int m) {
    require(m >= 2, "clenshaw_curtis: need at least two points");
    NodesWeights r;
    r.x.resize(static_cast<size_t>(m));
    r.w.resize(static_cast<size_t>(m));
    const int segs = m - 1;
    for (int j = 0; j < m; ++j) {
        const double ang = kPi * j / segs;
        double sum = 0.0;
        for (int k = 1; k <= segs / 2; ++k) {
            const double bk = (2 * k == segs) ? 1.0 : 2.0;
            sum += bk / (4.0 * k * k - 1.0) * std::cos(2.0 * k * ang);
        }
        const double cj = (j == 0 || j == segs) ? 1.0 : 2.0;
        r.x[static_cast<size_t>(j)] = 0.5 * (1.0 - std::cos(ang));
        r.w[static_cast<size_t>(j)] = 0.5 * cj / segs * (1.0 - sum);
    }
    return r;
}

// quadrature.hpp:90-102: process-lifetime memo keyed by (kind, m).
const NodesWeights& memo_rule(int kind, int m) {
    static std::mutex guard;
    static std::map<long long, std::unique_ptr<NodesWeights>> memo;
    std::lock_guard<std::mutex> hold(guard);
    const long long key = (static_cast<long long>(kind) << 32) | static_cast<unsigned>(m);
    auto& slot = memo[key];
    if (!slot)
        slot = std::make_unique<NodesWeights>(kind == kGauss ? gauss_legendre01(m) : clenshaw_curtis01(m));
    return *slot;
}

// ------------------------------------------------------------------ roots (roots.hpp) ----

namespace {
template <class T>
T horner(const Quartic& c, T x) {
    return (((x + c[0]) * x + c[1]) * x + c[2]) * x + c[3];
}
template <class T>
T horner_d(const Quartic& c, T x) {
    return ((4.0 * x + 3.0 * c[0]) * x + 2.0 * c[1]) * x + c[2];
}
}  // namespace

// roots.hpp:34-81: balance, Durand-Kerner (Gauss-Seidel order, <= 200 sweeps), Newton polish.
std::array<std::complex<double>, 4> quartic_zeros(const Quartic& q) {
    using C = std::complex<double>;
    double s = 1.0;
    s = std::max(s, std::abs(q[0]));
    s = std::max(s, std::sqrt(std::abs(q[1])));
    s = std::max(s, std::cbrt(std::abs(q[2])));
    s = std::max(s, std::pow(std::abs(q[3]), 0.25));
    const Quartic bal{q[0] / s, q[1] / (s * s), q[2] / (s * s * s), q[3] / (s * s * s * s)};

    std::array<C, 4> z;
    {
        const C start(0.4, 0.9);
        C acc(1.0, 0.0);
        for (auto& zk : z) {
            acc *= start;
            zk = acc;
        }
    }
    for (int sweep = 0; sweep < 200; ++sweep) {
        double worst = 0.0;
        for (int k = 0; k < 4; ++k) {
            C prod(1.0, 0.0);
            for (int j = 0; j < 4; ++j)
                if (j != k) prod *= z[k] - z[j];
            if (prod == C(0.0, 0.0)) prod = C(1e-300, 0.0);
            const C corr = horner(bal, z[k]) / prod;
            z[k] -= corr;
            worst = std::max(worst, std::abs(corr) / (1.0 + std::abs(z[k])));
        }
        if (worst < 1e-15) break;
    }
    for (auto& zk : z) {
        zk *= s;
        for (int it = 0; it < 4; ++it) {
            const C der = horner_d(q, zk);
            if (std::abs(der) == 0.0) break;
            const C corr = horner(q, zk) / der;
            if (!std::isfinite(std::abs(corr))) break;
            zk -= corr;
        }
    }
    return z;
}

// roots.hpp:88-118: near-real zeros, real Newton polish, keep > 1, merge 1e-6 clusters.
std::vector<double> real_zeros_above_one(const Quartic& q) {
    std::vector<double> keep;
    for (const auto& zc : quartic_zeros(q)) {
        if (std::abs(zc.imag()) > 1e-8 * (1.0 + std::abs(zc.real()))) continue;
        double x = zc.real();
        for (int it = 0; it < 8; ++it) {
            const double der = horner_d(q, x);
            if (der == 0.0) break;
            const double dx = horner(q, x) / der;
            if (!std::isfinite(dx)) break;
            x -= dx;
            if (std::abs(dx) <= 1e-14 * (1.0 + std::abs(x))) break;
        }
        if (x > 1.0) keep.push_back(x);
    }
    std::sort(keep.begin(), keep.end());
    std::vector<double> merged;
    for (size_t a = 0; a < keep.size();) {
        size_t b = a + 1;
        double total = keep[a];
        while (b < keep.size() && keep[b] - keep[b - 1] <= 1e-6 * (1.0 + std::abs(keep[b]))) total += keep[b++];
        merged.push_back(total / static_cast<double>(b - a));
        a = b;
    }
    return merged;
}

// roots.hpp:123-151: Illinois regula falsi with bisection fallback.
template <class F>
static double illinois_root(F&& f, double lo, double hi, double tol) {
    require(lo < hi, "find_root_monotone: empty interval");
    double flo = f(lo), fhi = f(hi);
    if (flo == 0.0) return lo;
    if (fhi == 0.0) return hi;
    require((flo > 0.0) != (fhi > 0.0), "find_root_monotone: endpoints do not bracket a root");
    int side = 0;
    for (int it = 0; it < 200 && (hi - lo) > tol; ++it) {
        double mid = hi - fhi * (hi - lo) / (fhi - flo);
        if (!(mid > lo && mid < hi) || !std::isfinite(mid)) mid = 0.5 * (lo + hi);
        const double fmid = f(mid);
        if (fmid == 0.0) return mid;
        if ((fmid > 0.0) == (flo > 0.0)) {
            lo = mid;
            flo = fmid;
            if (side == -1) fhi *= 0.5;
            side = -1;
        } else {
            hi = mid;
            fhi = fmid;
            if (side == +1) flo *= 0.5;
            side = +1;
        }
    }
    return 0.5 * (lo + hi);
}

// ---------------------------------------------------------------- bounds (bounds.hpp) ----

// bounds.hpp:52-63: CC uses the even-n sharpening (integer even n -> n+1).
static double decay_n(const BoundArgs& q) {
    if (q.kind == kGauss) return q.n;
    const double r = std::round(q.n);
    if (std::abs(q.n - r) < 1e-9) return (static_cast<long long>(r) % 2 == 0) ? q.n + 1.0 : q.n;
    return q.n + 1.0;
}

// bounds.hpp:71-84
double log_bound_rho(const BoundArgs& q, double rho) {
    require(rho > 1.0, "log_bound_at_rho: need rho > 1");
    require(q.alpha > 0.0, "log_bound_at_rho: need alpha > 0");
    require(q.p >= 0, "log_bound_at_rho: need p >= 0");
    require(q.beta >= 0.0, "log_bound_at_rho: need beta >= 0");
    if (q.beta == 0.0) return -kInf;
    const double g = (rho + 1.0) * (rho + 1.0) / (2.0 * rho);
    const double log_m =
        q.p * std::log(g) - (q.p + 1.0) * kLn2 - std::lgamma(q.p + 1.0) + 0.5 * g * q.alpha + std::log(q.beta);
    const double tail = q.kind == kGauss ? -2.0 * q.n * std::log(rho) : (1.0 - decay_n(q)) * std::log(rho);
    return std::log(144.0 / 35.0) + log_m + tail - std::log(rho * rho - 1.0);
}

// bounds.hpp:88-102: the stationarity quartic in rho.
Quartic stationary_quartic(const BoundArgs& q) {
    const double a = q.alpha;
    Quartic c{};
    c[1] = -(2.0 + 8.0 * q.p / a);
    c[3] = 1.0;
    if (q.kind == kGauss) {
        c[0] = -4.0 / a * (2.0 * (q.n + 1.0) - q.p);
        c[2] = 4.0 / a * (2.0 * q.n + q.p);
    } else {
        const double ne = decay_n(q);
        c[0] = -4.0 / a * (ne + 1.0 - q.p);
        c[2] = 4.0 / a * (ne - 1.0 + q.p);
    }
    return c;
}

// The stationarity quartic depends on (n, p, alpha, kind) but not on beta, and the planner
// evaluates the same quartics again for every right-hand side of an operator; its real roots
// are memoised by the exact coefficient bits (a pure function: results are bit-identical).
static std::vector<double> stationary_roots(const Quartic& c) {
    using Key = std::array<unsigned long long, 3>;  // exact bit patterns of a3, a2, a1
    // per thread (the planner's level evaluations run on several threads at once; a shared map
    // behind one mutex serialised them)
    thread_local std::map<Key, std::vector<double>> memo;
    Key key;
    std::memcpy(key.data(), c.data(), sizeof(key));
    if (c[3] == 1.0 && std::isfinite(c[0]) && std::isfinite(c[1]) && std::isfinite(c[2])) {
        auto it = memo.find(key);
        if (it != memo.end()) return it->second;
        auto r = real_zeros_above_one(c);
        if (memo.size() > (1u << 16)) memo.clear();
        memo.emplace(key, r);
        return r;
    }
    return real_zeros_above_one(c);
}

// bounds.hpp:107-115
double log_theorem_bound(const BoundArgs& q) {
    require(q.alpha > 0.0, "theorem_bound: need alpha > 0");
    if (q.beta == 0.0) return -kInf;
    const auto rhos = stationary_roots(stationary_quartic(q));
    if (rhos.empty()) throw ConvergenceFailure("theorem_bound: no stationary rho > 1 found");
    double best = kInf;
    for (double rho : rhos) best = std::min(best, log_bound_rho(q, rho));
    return best;
}

// bounds.hpp:122-142
double log_corollary_bound(const BoundArgs& q) {
    require(q.alpha > 0.0, "corollary_bound: need alpha > 0");
    if (q.beta == 0.0) return -kInf;
    double ex;
    if (q.kind == kGauss) {
        const double floor_n = std::max(2.0, std::ceil((1.0 + std::numbers::sqrt2) / 4.0 * q.alpha + 0.5 * q.p));
        require(q.n >= floor_n, "corollary_bound: n below validity threshold");
        ex = 2.0 * q.n - q.p;
    } else {
        const double floor_n = std::max(4.0, std::ceil((1.0 + std::numbers::sqrt2) / 2.0 * q.alpha + q.p));
        require(q.n >= floor_n, "corollary_bound: n below validity threshold");
        double even_n = q.n;
        const double r = std::round(q.n);
        if (std::abs(q.n - r) < 1e-9 && static_cast<long long>(r) % 2 != 0) even_n = q.n - 1.0;
        ex = even_n - q.p;
    }
    const double pre = std::log(q.beta) - (q.p + 1.0) * kLn2 - std::lgamma(q.p + 1.0);
    return pre - ex * std::log(ex / (std::numbers::e * q.alpha / 2.0));
}

// bounds.hpp:146-154: worst case over phi_1..phi_p (monomial degree q-1).
double log_quaderr(double n, int p, double alpha, double beta, int kind) {
    require(p >= 1, "quaderr: need p >= 1");
    double worst = -kInf;
    for (int deg = 0; deg < p; ++deg) worst = std::max(worst, log_theorem_bound(BoundArgs{n, deg, alpha, beta, kind}));
    return worst;
}

// bounds.hpp:159-180 (Alg. 4): doubling, then Illinois on the bracket, then the GL guard.
int node_count(double eps, int p, double alpha, double beta, int kind) {
    require(eps > 0.0 && eps < 1.0, "quadnodes: need 0 < eps < 1");
    require(p >= 1, "quadnodes: need p >= 1");
    require(alpha > 0.0, "quadnodes: need alpha > 0");
    const double goal = std::log(eps);
    auto bound = [&](double n) { return log_quaderr(n, p, alpha, beta, kind); };
    int n = kind == kGauss ? 2 : 4;
    double e = bound(n);
    if (e <= goal) return n;
    while (e > goal) {
        if (n > (1 << 20)) throw ConvergenceFailure("quadnodes: node count diverged");
        n *= 2;
        e = bound(n);
    }
    const double root = illinois_root([&](double x) { return bound(x) - goal; }, n / 2.0, static_cast<double>(n), 1e-6);
    int out = static_cast<int>(std::ceil(root - 1e-9));
    if (kind == kGauss && bound(out) > goal + 1e-12) ++out;
    return out;
}

// A small process-wide pool for the planner's independent quadnodes evaluations (one per
// scaling level l).  Pure functions of their arguments, so running them concurrently changes no
// result; the caller keeps the reference's sequential scan order for the decisions.
namespace {
class PlannerPool {
public:
    static PlannerPool& get() {
        static PlannerPool pool;
        return pool;
    }
    void run(std::vector<std::function<void()>>& jobs) {
        if (jobs.empty()) return;
        struct Latch {
            std::mutex mu;
            std::condition_variable cv;
            size_t left;
        } latch;
        latch.left = jobs.size();
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (auto& j : jobs)
                q_.push_back([&latch, &j] {
                    j();
                    std::lock_guard<std::mutex> l2(latch.mu);
                    if (--latch.left == 0) latch.cv.notify_all();
                });
        }
        cv_.notify_all();
        std::unique_lock<std::mutex> lk(latch.mu);
        latch.cv.wait(lk, [&latch] { return latch.left == 0; });
    }
    int threads() const { return static_cast<int>(th_.size()); }

private:
    PlannerPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        const int n = static_cast<int>(std::min(6u, hw > 1 ? hw - 1 : 1u));
        for (int i = 0; i < n; ++i)
            th_.emplace_back([this] {
                while (true) {
                    std::function<void()> f;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
                        if (stop_ && q_.empty()) return;
                        f = std::move(q_.front());
                        q_.pop_front();
                    }
                    f();
                }
            });
    }
    ~PlannerPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    std::vector<std::thread> th_;
    bool stop_ = false;
};
}  // namespace

// bounds.hpp:185-207 (Alg. 5): scan l downward, stop at the first strict cost increase.  The
// node counts of the first levels of the scan are evaluated concurrently (each ~0.1 ms of root
// finding; the scan typically stops 3-5 levels below the top); the scan itself, and which
// evaluation's exception surfaces, follow the reference's sequential order exactly.
Plan plan_quadrature(double eps, int p, double alpha, double beta, int kind, const Cost& cost) {
    require(alpha > 0.0, "setup_quadrature: need alpha > 0");
    const int top = alpha > 1.0 ? static_cast<int>(std::ceil(std::log2(alpha) - 1e-12)) : 0;
    static const int kAhead = [] {
        const char* v = std::getenv("PQ_PLAN_THREADS");
        return v ? std::max(1, std::atoi(v)) : 6;
    }();
    const int ahead = std::min(top + 1, kAhead);
    std::vector<int> pre(static_cast<size_t>(ahead), 0);
    std::vector<std::exception_ptr> err(static_cast<size_t>(ahead));
    if (ahead > 1) {
        std::vector<std::function<void()>> jobs;
        for (int i = 0; i < ahead; ++i)
            jobs.push_back([&, i] {
                try {
                    pre[static_cast<size_t>(i)] = node_count(eps, p, std::ldexp(alpha, -(top - i)), beta, kind);
                } catch (...) {
                    err[static_cast<size_t>(i)] = std::current_exception();
                }
            });
        PlannerPool::get().run(jobs);
    }
    Plan best;
    bool seen = false;
    for (int l = top; l >= 0; --l) {
        const int i = top - l;
        int n;
        if (ahead > 1 && i < ahead) {
            if (err[static_cast<size_t>(i)]) std::rethrow_exception(err[static_cast<size_t>(i)]);
            n = pre[static_cast<size_t>(i)];
        } else {
            n = node_count(eps, p, std::ldexp(alpha, -l), beta, kind);
        }
        const double c = cost(n, l, p);
        if (!seen || c < best.cost) {
            best = Plan{l, n, c};
            seen = true;
        } else if (c > best.cost) {
            break;
        }
    }
    return best;
}

}  // namespace pqb
