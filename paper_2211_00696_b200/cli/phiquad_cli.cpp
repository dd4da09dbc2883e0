// phiquad command-line front end on the B200 engine: the reference CLI's wire format
// (proj/tools/phiquad_cli.cpp: subcommands plan / bench / converge / phi, CSV with shortest
// round-trip doubles and "# plan:" trailers, dense-matrix text for `phi`, exit codes 0 / 1 / 2 / 3)
// written against the drop-in headers (include/phiquad), so every phi action runs on the GPU
// through libpq_b200.so.  The reference parses options with CLI11 (not vendored); this file has
// its own small parser with the same option names, range checks and error exit code 2.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <limits>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "phiquad/phiquad.hpp"
#include "phiquad/problems.hpp"

namespace {

using namespace phiquad;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// shortest decimal that round-trips the double (phiquad_cli.cpp:21-26)
std::string fmt(double v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, res.ptr);
}

QuadKind rule_of(const std::string& r) {
    if (r == "gauss") return QuadKind::gauss_legendre;
    if (r == "cc") return QuadKind::clenshaw_curtis;
    throw std::invalid_argument("--rule must be 'gauss' or 'cc'");
}

// writes to --out when given, else stdout
struct Sink {
    std::ofstream file;
    explicit Sink(const std::string& path) {
        if (!path.empty()) {
            file.open(path);
            if (!file) throw std::invalid_argument("cannot open output file: " + path);
        }
    }
    std::ostream& os() { return file.is_open() ? static_cast<std::ostream&>(file) : std::cout; }
};

// ---- option parsing -------------------------------------------------------------------
// Every option takes values except flags; multi-valued options take every following token that
// does not start with "--".  Values are checked when converted (the reference's CLI11 checks).
struct Options {
    std::map<std::string, std::vector<std::string>> values;
    std::vector<std::string> flags_seen;
    bool has(const std::string& k) const { return values.count(k) != 0; }
};

struct Spec {
    std::vector<std::string> single, multi, flags, required;
};

Options parse(const std::vector<std::string>& args, const Spec& spec) {
    auto is_in = [](const std::vector<std::string>& v, const std::string& s) {
        return std::find(v.begin(), v.end(), s) != v.end();
    };
    Options o;
    for (size_t i = 0; i < args.size(); ++i) {
        std::string a = args[i];
        std::optional<std::string> inline_val;
        if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + a);
        const size_t eq = a.find('=');
        if (eq != std::string::npos) {
            inline_val = a.substr(eq + 1);
            a = a.substr(0, eq);
        }
        const std::string name = a.substr(2);
        if (is_in(spec.flags, name)) {
            if (inline_val) throw UsageError("--" + name + " takes no value");
            o.flags_seen.push_back(name);
            continue;
        }
        const bool multi = is_in(spec.multi, name);
        if (!multi && !is_in(spec.single, name)) throw UsageError("unknown option: --" + name);
        std::vector<std::string>& dst = o.values[name];
        if (!multi && !dst.empty()) throw UsageError("--" + name + " given twice");
        if (inline_val) {
            dst.push_back(*inline_val);
        } else {
            size_t j = i + 1;
            if (j >= args.size()) throw UsageError("--" + name + " needs a value");
            dst.push_back(args[j++]);
            if (multi)
                while (j < args.size() && args[j].rfind("--", 0) != 0) dst.push_back(args[j++]);
            i = j - 1;
        }
    }
    for (const auto& r : spec.required)
        if (!o.has(r)) throw UsageError("--" + r + " is required");
    return o;
}

double to_double(const std::string& name, const std::string& s) {
    size_t used = 0;
    double v = 0.0;
    try {
        v = std::stod(s, &used);
    } catch (...) {
        throw UsageError("--" + name + ": not a number: " + s);
    }
    if (used != s.size()) throw UsageError("--" + name + ": not a number: " + s);
    return v;
}

int to_int(const std::string& name, const std::string& s) {
    int v = 0;
    const auto res = std::from_chars(s.data(), s.data() + s.size(), v);
    if (res.ec != std::errc() || res.ptr != s.data() + s.size()) throw UsageError("--" + name + ": not an integer: " + s);
    return v;
}

template <class T, class Conv>
T get(const Options& o, const std::string& name, T dflt, Conv conv) {
    return o.has(name) ? conv(name, o.values.at(name).front()) : dflt;
}
int get_int(const Options& o, const std::string& name, int dflt, int lo, int hi) {
    const int v = get<int>(o, name, dflt, to_int);
    if (o.has(name) && (v < lo || v > hi))
        throw UsageError("--" + name + ": " + std::to_string(v) + " not in [" + std::to_string(lo) + ", " +
                         std::to_string(hi) + "]");
    return v;
}
double get_double(const Options& o, const std::string& name, double dflt) { return get<double>(o, name, dflt, to_double); }
std::string get_str(const Options& o, const std::string& name, const std::string& dflt) {
    return o.has(name) ? o.values.at(name).front() : dflt;
}
constexpr int kPos = std::numeric_limits<int>::max();

// ---- subcommands ------------------------------------------------------------------------

// phiquad_cli.cpp:61-80
int run_plan(const Options& o) {
    std::vector<double> alphas;
    for (const auto& s : o.values.at("alpha")) alphas.push_back(to_double("alpha", s));
    const int p = get_int(o, "p", 20, 1, kPos);
    const double eps = get_double(o, "eps", 1e-14), beta = get_double(o, "beta", 1.0);
    const std::string rule = get_str(o, "rule", "gauss");
    const double c1 = get_double(o, "c1", 0.0), c2 = get_double(o, "c2-cost", 1.0);
    const int d = get_int(o, "d", 1, 1, 3);
    const QuadKind kind = rule_of(rule);
    Sink sink(get_str(o, "out", ""));
    std::ostream& os = sink.os();
    os << "alpha,rule,l,n,C\n";
    QuadraturePlan plan{};
    for (double alpha : alphas) {
        if (!(alpha > 0.0)) throw std::invalid_argument("plan: need alpha > 0");
        plan = setup_quadrature(eps, p, alpha, beta, kind, CostModel{c1, c2, d});
        os << fmt(alpha) << ',' << rule << ',' << plan.l << ',' << plan.n << ',' << fmt(plan.cost) << '\n';
    }
    os << "# plan: l=" << plan.l << ",n=" << plan.n << ",rule=" << rule << ",eps=" << fmt(eps) << '\n';
    return 0;
}

// phiquad_cli.cpp:97-145
int run_bench(const Options& o) {
    const int problem = get_int(o, "problem", 1, 1, 3);
    const int r = get_int(o, "r", 4, 1, 14);
    const int p = get_int(o, "p", 20, 1, kPos);
    const double tau = get_double(o, "tau", 0.125);
    const std::string rule = get_str(o, "rule", "gauss");
    const double eps = get_double(o, "eps", 1e-14);
    std::optional<int> l;
    if (o.has("l")) l = get_int(o, "l", 0, 0, kPos);
    const double c1 = get_double(o, "c1", 0.0), c2 = get_double(o, "c2-cost", 1.0);
    const bool verify = std::find(o.flags_seen.begin(), o.flags_seen.end(), "verify") != o.flags_seen.end();
    const int threads = get_int(o, "threads", default_thread_count(), 1, kPos);
    if (!(tau > 0.0)) throw std::invalid_argument("bench: need --tau > 0");
    TensorProblem prob = [&] {
        switch (problem) {
            case 1: return make_problem1(r);
            case 2: return make_problem2(r);
            default: {
                SemilinearProblem s = make_problem3(r);
                return TensorProblem{std::move(s.a), std::move(s.u0)};
            }
        }
    }();
    const KroneckerSum arg = prob.a.scaled(-tau);
    const int dim = arg.dim();
    std::vector<std::vector<double>> dense;
    if (verify) {
        if (dim + p > 1000)
            throw std::invalid_argument("bench: --verify needs dim + p <= 1000 (got dim = " + std::to_string(dim) +
                                        "); use a smaller --r");
        dense = phi_dense_oracle(arg, prob.b, p);
    }
    PhiRequest req;
    req.p = p;
    req.eps = eps;
    req.mode = rule_of(rule);
    req.l = l;
    req.cost = CostModel{c1, c2, 1};
    req.threads = threads;
    PhiInfo info;
    const PhiColumns y = phiquadmv(arg, prob.b, req, &info);
    Sink sink(get_str(o, "out", ""));
    std::ostream& os = sink.os();
    os << "p,rel_err\n";
    for (int j = 1; j <= p; ++j) {
        const double err = verify ? relative_error_inf(y.col(j), dense[static_cast<size_t>(j - 1)])
                                  : std::numeric_limits<double>::quiet_NaN();
        os << j << ',' << fmt(err) << '\n';
    }
    os << "# plan: l=" << info.l << ",n=" << info.n << ",rule=" << rule << ",eps=" << fmt(eps)
       << ",alpha=" << fmt(info.alpha) << ",dim=" << dim << ",points=" << info.points << '\n';
    return 0;
}

// phiquad_cli.cpp:160-201
int run_converge(const Options& o) {
    const int problem = get_int(o, "problem", 3, std::numeric_limits<int>::min(), kPos);
    const int r = get_int(o, "r", 5, 1, 12);
    const std::string rule = get_str(o, "rule", "gauss");
    const double eps = get_double(o, "eps", 1e-14);
    const double c1 = get_double(o, "c1", 0.0), c2 = get_double(o, "c2-cost", 1.0);
    const int threads = get_int(o, "threads", default_thread_count(), 1, kPos);
    if (problem != 3) throw std::invalid_argument("converge: only --problem 3 (semilinear) is supported");
    SemilinearProblem prob = make_problem3(r);
    PhiRequest base;
    base.eps = eps;
    base.mode = rule_of(rule);
    base.cost = CostModel{c1, c2, 1};
    base.threads = threads;
    const bool has_c2 = o.has("c2-rk");
    const double c2rk = has_c2 ? get_double(o, "c2-rk", 0.0) : 0.0;
    const ExpRKTableau tabs[3] = {exp_euler_tableau(), exp_rk2_tableau(has_c2 ? c2rk : 0.5),
                                  exp_rk3_tableau(has_c2 ? c2rk : 1.0 / 3.0)};
    std::vector<int> steps;
    if (o.has("tau")) {
        const double tau = get_double(o, "tau", 0.0);
        if (!(tau > 0.0) || tau > 1.0) throw std::invalid_argument("converge: need 0 < --tau <= 1");
        steps.push_back(std::max(1, static_cast<int>(std::lround(1.0 / tau))));
    } else {
        for (int m = 2; m <= 64; m *= 2) steps.push_back(m);
    }
    Sink sink(get_str(o, "out", ""));
    std::ostream& os = sink.os();
    os << "tau,err_euler,err_rk2,err_rk3\n";
    const std::vector<double> exact = prob.exact(1.0);
    double tau_last = 1.0;
    for (int m : steps) {
        const double tau = 1.0 / m;
        tau_last = tau;
        os << fmt(tau);
        for (const ExpRKTableau& tab : tabs)
            os << ',' << fmt(relative_error_inf(integrate(prob.a, prob.f, prob.u0, 0.0, 1.0, m, tab, base).u, exact));
        os << '\n';
    }
    const double alpha = tau_last * infnorm_bound(prob.a);
    const QuadraturePlan plan = setup_quadrature(eps, 2, alpha, 1.0, base.mode, CostModel{c1, c2, prob.a.order()});
    os << "# plan: l=" << plan.l << ",n=" << plan.n << ",rule=" << rule << ",eps=" << fmt(eps)
       << ",alpha=" << fmt(alpha) << ",dim=" << prob.a.dim() << '\n';
    return 0;
}

DenseMatrix read_matrix(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw std::invalid_argument("cannot open matrix file: " + path);
    return read_matrix_text(is);
}

// phiquad_cli.cpp:219-250
int run_phi(const Options& o) {
    const auto& files = o.values.at("matrix-file");
    if (files.size() > 3) throw UsageError("--matrix-file: at most 3 factors");
    const int p = get_int(o, "p", 1, 1, kPos);
    const std::string rule = get_str(o, "rule", "gauss");
    const double eps = get_double(o, "eps", 1e-14);
    std::optional<int> l;
    if (o.has("l")) l = get_int(o, "l", 0, 0, kPos);
    const int threads = get_int(o, "threads", default_thread_count(), 1, kPos);
    std::vector<DenseMatrix> factors;
    for (const auto& f : files) factors.push_back(read_matrix(f));
    const KroneckerSum a(std::move(factors));
    const DenseMatrix bm = read_matrix(get_str(o, "b-file", ""));
    if (bm.cols() != 1 && bm.rows() != 1) throw std::invalid_argument("phi: --b-file must hold a single row or column");
    std::vector<double> b(bm.data(), bm.data() + static_cast<size_t>(bm.rows()) * bm.cols());
    if (static_cast<int>(b.size()) != a.dim())
        throw std::invalid_argument("phi: vector length does not match the Kronecker-sum size");
    PhiRequest req;
    req.p = p;
    req.eps = eps;
    req.mode = rule_of(rule);
    req.l = l;
    req.threads = threads;
    PhiInfo info;
    const PhiColumns y = phiquadmv(a, b, req, &info);
    DenseMatrix cols(a.dim(), p);
    for (int j = 1; j <= p; ++j)
        for (int i = 0; i < a.dim(); ++i) cols(i, j - 1) = y.col(j)[static_cast<size_t>(i)];
    Sink sink(get_str(o, "out", ""));
    write_matrix_text(sink.os(), cols);
    return 0;
}

const char* kUsage =
    "Actions of phi-functions of Kronecker-sum matrices via quadrature (B200 engine)\n"
    "Usage: phiquad_cli SUBCOMMAND [OPTIONS]\n\n"
    "Subcommands:\n"
    "  plan      Print scaling/quadrature plans for given norms\n"
    "            --alpha A... (required) --p --eps --beta --rule gauss|cc --c1 --c2-cost --d --out\n"
    "  bench     Run a phi-action benchmark problem\n"
    "            --problem 1|2|3 --r --p --tau --rule --eps --l --c1 --c2-cost --verify --out --threads\n"
    "  converge  Time-stepping convergence study on the semilinear problem\n"
    "            --problem --r --rule --eps --tau --c2-rk --c1 --c2-cost --out --threads\n"
    "  phi       Apply phi-functions to a vector from text files\n"
    "            --matrix-file F (1-3, required) --b-file F (required) --p --rule --eps --l --out --threads\n";

}  // namespace

int main(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    if (args.empty()) {
        std::cerr << kUsage << "error: a subcommand is required\n";
        return 2;
    }
    if (args[0] == "--help" || args[0] == "-h") {
        std::cout << kUsage;
        return 0;
    }
    const std::string sub = args[0];
    std::vector<std::string> rest(args.begin() + 1, args.end());
    if (std::find(rest.begin(), rest.end(), "--help") != rest.end() ||
        std::find(rest.begin(), rest.end(), "-h") != rest.end()) {
        std::cout << kUsage;
        return 0;
    }
    static const std::map<std::string, Spec> specs = {
        {"plan", {{"p", "eps", "beta", "rule", "c1", "c2-cost", "d", "out"}, {"alpha"}, {}, {"alpha"}}},
        {"bench", {{"problem", "r", "p", "tau", "rule", "eps", "l", "c1", "c2-cost", "out", "threads"}, {}, {"verify"}, {}}},
        {"converge", {{"problem", "r", "rule", "eps", "tau", "c2-rk", "c1", "c2-cost", "out", "threads"}, {}, {}, {}}},
        {"phi", {{"b-file", "p", "rule", "eps", "l", "out", "threads"}, {"matrix-file"}, {}, {"matrix-file", "b-file"}}},
    };
    static const std::map<std::string, std::function<int(const Options&)>> run = {
        {"plan", run_plan}, {"bench", run_bench}, {"converge", run_converge}, {"phi", run_phi}};
    try {
        const auto it = specs.find(sub);
        if (it == specs.end()) throw UsageError("unknown subcommand: " + sub);
        const Options opts = parse(rest, it->second);
        return run.at(sub)(opts);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const ConvergenceError& e) {
        std::cerr << "numerical failure: " << e.what() << '\n';
        return 3;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
