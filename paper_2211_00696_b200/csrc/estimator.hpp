// Host-side estimator of the phi engine: quadrature rules, quartic roots, the a-priori
// quadrature bound and the (l, n) planner.  This is product code (it decides the scaling level
// and the node count of every GPU call), restated from the paper's Algorithms 3-5 and kept
// arithmetic-for-arithmetic equivalent to the reference so that plans are identical
// (reference: quadrature.hpp, roots.hpp, bounds.hpp).  Pure C++20, no CUDA.
#pragma once

#include <array>
#include <complex>
#include <stdexcept>
#include <string>
#include <vector>

namespace pqb {

// Exception vocabulary shared with the C ABI (return codes in include/pq_b200.h).
struct ConvergenceFailure : std::runtime_error {
    explicit ConvergenceFailure(const std::string& w) : std::runtime_error(w) {}
};

enum Rule : int { kGauss = 0, kClenshaw = 1 };

struct NodesWeights {
    std::vector<double> x;  // ascending on [0, 1]
    std::vector<double> w;
    int size() const { return static_cast<int>(x.size()); }
};

NodesWeights gauss_legendre01(int m);                  // quadrature.hpp:31-62
NodesWeights clenshaw_curtis01(int m);                 // quadrature.hpp:67-86
const NodesWeights& memo_rule(int kind, int m);        // quadrature.hpp:90-102

// rho^4 + c[0] rho^3 + c[1] rho^2 + c[2] rho + c[3]
using Quartic = std::array<double, 4>;
std::array<std::complex<double>, 4> quartic_zeros(const Quartic& q);   // roots.hpp:34-81
std::vector<double> real_zeros_above_one(const Quartic& q);            // roots.hpp:88-118

struct BoundArgs {
    double n = 0.0;
    int p = 0;
    double alpha = 0.0;
    double beta = 1.0;
    int kind = kGauss;
};
double log_bound_rho(const BoundArgs& q, double rho);   // bounds.hpp:71-84
Quartic stationary_quartic(const BoundArgs& q);         // bounds.hpp:88-102
double log_theorem_bound(const BoundArgs& q);           // bounds.hpp:107-115
double log_corollary_bound(const BoundArgs& q);         // bounds.hpp:122-142
double log_quaderr(double n, int p, double alpha, double beta, int kind);   // bounds.hpp:146-154
int node_count(double eps, int p, double alpha, double beta, int kind);     // bounds.hpp:159-180

struct Cost {
    double c1 = 0.0, c2 = 1.0;
    int d = 1;
    double operator()(double n, int l, int p) const { return c1 * d * n + c2 * (n + static_cast<double>(l) * p); }
};
struct Plan {
    int l = 0, n = 0;
    double cost = 0.0;
};
Plan plan_quadrature(double eps, int p, double alpha, double beta, int kind, const Cost& cost); // bounds.hpp:185-207

}  // namespace pqb
