// Problem-assembly dump written against the reference's phiquad API (problems.hpp).  Built against
// the reference headers it produces tests/golden/problems_ref_output.txt; built against this
// repo's drop-in headers it must print identical lines (tests/test_problems.py): every operator
// entry, data vector, mesh node, source value and error norm, "%.17g" (round-trip exact).
#include <phiquad/phiquad.hpp>
#include <phiquad/problems.hpp>

#include <cstdio>
#include <string>
#include <vector>

using namespace phiquad;

static void put(const std::string& k, double v) { std::printf("%s %.17g\n", k.c_str(), v); }
static void put_vec(const std::string& k, const std::vector<double>& v) {
    for (size_t i = 0; i < v.size(); ++i) put(k + "[" + std::to_string(i) + "]", v[i]);
}
static void put_mat(const std::string& k, const DenseMatrix& m) {
    put(k + ".rows", m.rows());
    put(k + ".cols", m.cols());
    for (int i = 0; i < m.rows(); ++i)
        for (int j = 0; j < m.cols(); ++j) put(k + "(" + std::to_string(i) + "," + std::to_string(j) + ")", m(i, j));
}

int main() {
    put_vec("uniform_mesh", uniform_mesh(7, -0.5, 0.5).nodes);
    put_vec("shishkin_default", shishkin_mesh(16, 1e-2).nodes);
    put_vec("shishkin_1_16", shishkin_mesh(8, 1e-2, 1.0 / 16.0).nodes);
    put_mat("fe_laplacian_5_0_2", fe_laplacian_1d(5, 0.0, 2.0));
    const Mesh1D sm = shishkin_mesh(8, 1e-2, 1.0 / 16.0);
    put_mat("advdiff_nd", fe_advdiff_1d(sm, 1e-2, 1.0, BC::neumann, BC::dirichlet));
    put_mat("advdiff_dd", fe_advdiff_1d(uniform_mesh(6, -0.5, 0.5), 1e-2, 0.0, BC::dirichlet, BC::dirichlet));
    put_mat("advdiff_nn", fe_advdiff_1d(uniform_mesh(5, 0.0, 1.0), 0.3, -2.0, BC::neumann, BC::neumann));
    for (int r : {1, 2}) {
        const TensorProblem p1 = make_problem1(r);
        const std::string k = "p1r" + std::to_string(r);
        for (int f = 0; f < p1.a.order(); ++f) put_mat(k + ".a" + std::to_string(f), p1.a.factor(f));
        put_vec(k + ".b", p1.b);
    }
    for (int r : {2, 3}) {
        const TensorProblem p2 = make_problem2(r);
        const std::string k = "p2r" + std::to_string(r);
        for (int f = 0; f < p2.a.order(); ++f) put_mat(k + ".a" + std::to_string(f), p2.a.factor(f));
        put_vec(k + ".b", p2.b);
    }
    const SemilinearProblem p3 = make_problem3(2);
    put_mat("p3.a0", p3.a.factor(0));
    put_vec("p3.u0", p3.u0);
    std::vector<double> u(p3.u0.size());
    for (size_t i = 0; i < u.size(); ++i) u[i] = 0.1 * static_cast<double>(i) - 0.3;
    put_vec("p3.f", p3.f(0.37, u));
    put_vec("p3.exact", p3.exact(0.7));
    put("relerr", relative_error_inf({1.0, 2.5, -3.0}, {1.1, 2.0, -3.5}));
    put("relerr_zero", relative_error_inf({0.25, -0.5}, {0.0, 0.0}));
    return 0;
}
