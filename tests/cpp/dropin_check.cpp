// One program written against the reference's phiquad C++ API.  Built against the reference
// headers (-I/root/reference/proj/include) it produces tests/golden/dropin_ref_output.txt; built
// against this repo's drop-in headers (-Iinclude, -lpq_b200) it must print the same integers and
// the same values to the parity tolerance (tests/test_gpu_dropin.py).  Output: "key value" lines.
#include <phiquad/phiquad.hpp>

#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

using namespace phiquad;

static void put(const std::string& k, double v) { std::printf("%s %.17g\n", k.c_str(), v); }
static void put_vec(const std::string& k, const std::vector<double>& v) {
    for (size_t i = 0; i < v.size(); ++i) put(k + "[" + std::to_string(i) + "]", v[i]);
}

static DenseMatrix lap(int n, double scale) {
    DenseMatrix m(n, n);
    const double h = 1.0 / (n + 1), s = scale / (h * h);
    for (int i = 0; i < n; ++i) {
        m(i, i) = 2.0 * s;
        if (i > 0) m(i, i - 1) = -s;
        if (i + 1 < n) m(i, i + 1) = -s;
    }
    return m;
}

int main() {
    // rules and planner
    put_vec("gl5.nodes", gauss_legendre(5).nodes);
    put_vec("cc9.weights", clenshaw_curtis(9).weights);
    const auto plan = setup_quadrature(1e-14, 20, 384.0, 1.0, QuadKind::gauss_legendre, CostModel{0.0, 1.0, 3});
    put("plan384.l", plan.l);
    put("plan384.n", plan.n);
    put("quadnodes48", quadnodes(1e-14, 20, 48.0, 1.0, QuadKind::gauss_legendre));
    put("quaderr", quaderr(12.0, 4, 30.0, 2.0, QuadKind::clenshaw_curtis));

    // an asymmetric 3D advection-diffusion-like operator, argument -tau A
    std::vector<DenseMatrix> fs;
    for (int k = 0; k < 3; ++k) {
        const int n = 10 - k;
        DenseMatrix f = lap(n, 1.0 - 0.3 * k);
        for (int i = 0; i + 1 < n; ++i) {
            f(i, i + 1) += 3.0 * (k + 1);
            f(i + 1, i) -= 3.0 * (k + 1);
        }
        fs.push_back(f);
    }
    const KroneckerSum arg = KroneckerSum(fs).scaled(-3e-2);
    std::mt19937 rng(1234);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::vector<double> b(static_cast<size_t>(arg.dim()));
    for (double& x : b) x = u(rng);

    put("infnorm_bound", infnorm_bound(arg));
    put_vec("kron_matvec", kron_matvec(arg, b));
    put_vec("exp_action", exp_action(arg, b));
    put_vec("expm0", expm(arg.factor(0)).raw());

    for (QuadKind kind : {QuadKind::gauss_legendre, QuadKind::clenshaw_curtis}) {
        PhiRequest req;
        req.p = 4;
        req.eps = 1e-12;
        req.mode = kind;
        PhiInfo info;
        const auto cols = phiquadmv(arg, b, req, &info);
        const std::string tag = std::string("phiquadmv.") + quad_kind_name(kind);
        put(tag + ".l", info.l);
        put(tag + ".n", info.n);
        put(tag + ".points", info.points);
        for (int j = 1; j <= 4; ++j) put_vec(tag + ".col" + std::to_string(j), cols.col(j));
    }
    {
        int pts = 0;
        const auto ys = phi_with_plan(arg, {b, b}, 3, 2, 8, QuadKind::gauss_legendre, 1e-12, 1, &pts);
        put("phi_with_plan.points", pts);
        put_vec("phi_with_plan.m1.col3", ys[1].col(3));
    }
    {
        PhiColumns y{arg.dim(), {b, b, b}};
        std::vector<DenseMatrix> exps;
        for (int k = 0; k < 3; ++k) exps.push_back(expm(scaled(arg.factor(k), 0.25)));
        squaring_step(y, exps, arg.shape());
        put_vec("squaring.col3", y.col(3));
    }
    {
        const auto y = phi_lincomb(arg, {b, b}, cached_rule(QuadKind::gauss_legendre, 20));
        put_vec("lincomb", y);
    }
    {
        const SourceFn ac = [](double, const std::vector<double>& v) {
            std::vector<double> r(v.size());
            for (size_t i = 0; i < v.size(); ++i) r[i] = v[i] - v[i] * v[i] * v[i];
            return r;
        };
        const KroneckerSum a = KroneckerSum(fs).scaled(0.01);
        const auto res = integrate(a, ac, b, 0.0, 0.02, 4, exp_rk2_tableau());
        put("integrate.phi_calls", res.phi_calls);
        put_vec("integrate.u", res.u);
        PhiEngine eng(a, 0.005, PhiRequest{});
        const auto u1 = erk_step(eng, ac, 0.0, b, exp_rk3_tableau());
        put("erk_step.calls", eng.calls());
        put_vec("erk_step.u", u1);
    }
    // error behaviour
    try {
        phi_adaptive(KroneckerSum({DenseMatrix(2, 2, {-1.0, 0.2, 0.1, -2.0})}), {1.0, 1.0}, 2, 1e-30);
        put("adaptive.error", 0);
    } catch (const ConvergenceError&) {
        put("adaptive.error", 2);
    }
    try {
        PhiColumns c{1, {{1.0}}};
        c.col(2);
        put("col.error", 0);
    } catch (const std::out_of_range&) {
        put("col.error", 4);
    }
    // argument-check order, messages and the no-RHS plan (phiaction.hpp:277-346): a message is
    // printed as a numeric code of its text so the key/value comparison covers it exactly
    auto code = [](const std::string& m) {
        double h = 0.0;
        for (unsigned char ch : m) h = std::fmod(h * 31.0 + ch, 1000003.0);
        return h;
    };
    auto msg = [&](const std::string& key, auto&& fn) {
        try {
            fn();
            put(key, -1.0);
        } catch (const std::invalid_argument& e) {
            put(key, code(e.what()));
        }
    };
    for (QuadKind kind : {QuadKind::gauss_legendre, QuadKind::clenshaw_curtis}) {
        const std::string tag = std::string("norhs.") + quad_kind_name(kind);
        PhiRequest req;
        req.p = 3;
        req.eps = 1e-10;
        req.mode = kind;
        PhiInfo info;
        const auto none = phiquadmv_multi(arg, {}, req, &info);
        put(tag + ".size", static_cast<double>(none.size()));
        put(tag + ".l", info.l);
        put(tag + ".n", info.n);
        put(tag + ".points", info.points);
        put(tag + ".planned", info.planned ? 1 : 0);
        int pts = -7;
        const auto none2 = phi_with_plan(arg, {}, 3, 2, 8, kind, 1e-10, 1, &pts);
        put(tag + ".plan_points", pts);
        put(tag + ".plan_size", static_cast<double>(none2.size()));
        msg(tag + ".len_msg", [&] { phiquadmv(arg, std::vector<double>(5, 1.0), req); });
        msg(tag + ".plan_p_msg", [&] { phi_with_plan(arg, {std::vector<double>(5, 1.0)}, 0, 1, 4, kind, 1e-10); });
        msg(tag + ".plan_l_msg", [&] { phi_with_plan(arg, {b}, 2, -1, 4, kind, 1e-10); });
        msg(tag + ".plan_eps_msg", [&] { phi_with_plan(arg, {std::vector<double>(5, 1.0)}, 2, 1, 4, kind, 0.0); });
        PhiRequest bad = req;
        bad.p = 0;
        msg(tag + ".p_msg", [&] { phiquadmv_multi(arg, {std::vector<double>(5, 1.0)}, bad); });
    }
    try {
        phi_fixed(arg, std::vector<double>(3, 1.0), 2, cached_rule(QuadKind::gauss_legendre, 4));
        put("length.error", 0);
    } catch (const std::invalid_argument&) {
        put("length.error", 1);
    }
    return 0;
}
