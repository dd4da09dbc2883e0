// The drop-in's multi-GPU extension (include/phiquad/distributed.hpp) from C++ on one rank: the
// distributed call (world 1: node phase, slab combine, slab squaring and the flips all run, the
// exchanges are local copies) against the single-GPU phiquadmv_multi of the same inputs.
// Prints "max_rel <x>" and "plans_equal <0|1>"; tests/test_gpu_dropin.py checks them.
#include <phiquad/phiquad.hpp>

#include <cmath>
#include <cstdio>
#include <random>

using namespace phiquad;

int main() {
    std::vector<DenseMatrix> fs;
    for (int k = 0; k < 3; ++k) {
        const int n = 24 - 4 * k;
        DenseMatrix f(n, n);
        const double h = 1.0 / (n + 1), s = 1.0 / (h * h);
        for (int i = 0; i < n; ++i) {
            f(i, i) = 2.0 * s * (1.0 + 0.3 * k);
            if (i > 0) f(i, i - 1) = -s - 4.0 / h;
            if (i + 1 < n) f(i, i + 1) = -s + 4.0 / h;
        }
        fs.push_back(f);
    }
    const KroneckerSum arg = KroneckerSum(fs).scaled(-2e-3);
    std::mt19937 rng(7);
    std::normal_distribution<double> g(0.0, 1.0);
    std::vector<std::vector<double>> bs(2, std::vector<double>(static_cast<size_t>(arg.dim())));
    for (auto& b : bs)
        for (double& x : b) x = g(rng);
    double worst = 0.0;
    int plans_equal = 1;
    for (QuadKind kind : {QuadKind::gauss_legendre, QuadKind::clenshaw_curtis}) {
        PhiRequest req;
        req.p = 4;
        req.eps = 1e-10;
        req.mode = kind;
        PhiInfo i1, i2;
        const auto want = phiquadmv_multi(arg, bs, req, &i1);
        auto comm = b200::Communicator::single();
        const auto got = b200::phiquadmv_multi(arg, bs, req, comm, &i2);
        plans_equal &= (i1.l == i2.l && i1.n == i2.n && i1.points == i2.points) ? 1 : 0;
        for (size_t m = 0; m < bs.size(); ++m)
            for (int j = 1; j <= req.p; ++j) {
                double num = 0.0, den = 0.0;
                for (size_t t = 0; t < want[m].col(j).size(); ++t) {
                    const double d = got[m].col(j)[t] - want[m].col(j)[t];
                    num += d * d;
                    den += want[m].col(j)[t] * want[m].col(j)[t];
                }
                worst = std::max(worst, std::sqrt(num / den));
            }
    }
    std::printf("max_rel %.3e\nplans_equal %d\n", worst, plans_equal);
    return 0;
}
