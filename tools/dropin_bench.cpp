// Time the drop-in C++ API (include/phiquad, pageable std::vector buffers as a reference user has
// them) on the config-2 workload: phiquadmv (phi_1..phi_4) + exp_action (phi_0) per step.
// Build: g++ -std=c++20 -O2 -pthread -Iinclude tools/dropin_bench.cpp -Lpaper_2211_00696_b200 -lpq_b200
//        -Wl,-rpath,$PWD/paper_2211_00696_b200 -o tools/dropin_bench
#include <phiquad/phiquad.hpp>

#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

using namespace phiquad;

static DenseMatrix factor(int n, double d, double b) {
    DenseMatrix m(n, n);
    const double h = 1.0 / (n + 1);
    for (int i = 0; i < n; ++i) {
        m(i, i) = 2.0 * d / (h * h);
        if (i > 0) m(i, i - 1) = -d / (h * h) - b / (2 * h);
        if (i + 1 < n) m(i, i + 1) = -d / (h * h) + b / (2 * h);
    }
    return m;
}

int main(int argc, char** argv) {
    const int n = 128, steps = argc > 1 ? std::atoi(argv[1]) : 10;
    const double tau = 5e-3;
    KroneckerSum a({factor(n, 1.0, 10.0), factor(n, 0.5, 0.0), factor(n, 0.1, -5.0)});
    KroneckerSum s = a.scaled(-tau);
    std::mt19937_64 rng(1000);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::vector<double> b(static_cast<size_t>(n) * n * n);
    for (auto& x : b) x = nd(rng);
    PhiRequest req;
    req.p = 4;
    req.eps = 1e-10;
    req.mode = QuadKind::clenshaw_curtis;
    double sink = 0;
    auto call = [&] {
        PhiInfo info;
        PhiColumns cols = phiquadmv(s, b, req, &info);
        std::vector<double> y0 = exp_action(s, b);
        sink += cols.col(4)[7] + y0[11];
    };
    auto time_ms = [&](auto&& fn) {
        fn();
        const auto t0 = std::chrono::steady_clock::now();
        for (int k = 0; k < steps; ++k) fn();
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / steps;
    };
    const double ms = time_ms(call);
    const double ms_phi = time_ms([&] {
        PhiColumns cols = phiquadmv(s, b, req);
        sink += cols.col(1)[3];
    });
    const double ms_exp = time_ms([&] { sink += exp_action(s, b)[5]; });
    // the header's steps one by one (phiaction.hpp phiquadmv_multi)
    double t_wrap = 0, t_gather = 0, t_alloc = 0, t_call = 0, t_scatter = 0, t_free = 0;
    for (int k = 0; k < steps; ++k) {
        auto T = [] { return std::chrono::steady_clock::now(); };
        auto ms_since = [](auto t) { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count(); };
        auto t = T();
        std::vector<std::vector<double>> bs{b};
        t_wrap += ms_since(t); t = T();
        const auto flat = detail::gather(bs, s.dim(), "x");
        t_gather += ms_since(t); t = T();
        const auto f = detail::flatten(s);
        const pq_phi_request r = detail::abi_request(req);
        pq_phi_info pi{};
        std::vector<double> out(static_cast<size_t>(req.p) * s.dim());
        t_alloc += ms_since(t); t = T();
        b200::check(pq_phiquadmv(b200::context(), s.order(), f.shape.data(), f.data.data(), 1, flat.data(), &r,
                                 out.data(), &pi, PQ_HOST));
        t_call += ms_since(t); t = T();
        {
            auto cols = detail::scatter(out, 1, req.p, s.dim());
            t_scatter += ms_since(t); t = T();
            sink += cols[0].cols[0][1];
        }
        t_free += ms_since(t);
    }
    // the header's current path (phiquadmv_ptrs): threaded column allocation, in-place columns call, free
    double u_alloc = 0, u_call = 0, u_free = 0;
    for (int k = 0; k < steps; ++k) {
        auto T = [] { return std::chrono::steady_clock::now(); };
        auto ms_since = [](auto t) { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count(); };
        auto t = T();
        const auto f = detail::flatten(s);
        const pq_phi_request r = detail::abi_request(req);
        pq_phi_info pi{};
        {
            std::vector<PhiColumns> out = detail::alloc_columns(1, req.p, s.dim());
            u_alloc += ms_since(t); t = T();
            std::vector<double*> cols;
            for (auto& c : out[0].cols) cols.push_back(c.data());
            const double* bp = b.data();
            b200::check(pq_phiquadmv_cols(b200::context(), s.order(), f.shape.data(), f.data.data(), 1, &bp, &r,
                                          cols.data(), &pi, PQ_HOST));
            u_call += ms_since(t); t = T();
            sink += out[0].cols[1][5];
        }
        u_free += ms_since(t);
    }
    std::printf("{\"path\": \"phiquadmv_ptrs\", \"alloc_columns\": %.2f, \"pq_phiquadmv_cols\": %.2f, \"free\": %.2f}\n",
                u_alloc / steps, u_call / steps, u_free / steps);
    std::printf("{\"wrap\": %.2f, \"gather\": %.2f, \"alloc_out\": %.2f, \"pq_call\": %.2f, \"scatter\": %.2f, \"free\": %.2f}\n",
                t_wrap / steps, t_gather / steps, t_alloc / steps, t_call / steps, t_scatter / steps, t_free / steps);
    std::printf("{\"api\": \"drop-in headers, pageable std::vector\", \"ms_per_action\": %.3f, \"actions_per_s\": %.1f, "
                "\"ms_phiquadmv\": %.3f, \"ms_exp_action\": %.3f, \"sink\": %.3e}\n",
                ms, 1e3 / ms, ms_phi, ms_exp, sink);
}
