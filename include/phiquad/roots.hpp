#pragma once
// Quartic roots and the monotone root finder of the planner (reference roots.hpp:14-151).
#include <array>
#include <cmath>
#include <complex>
#include <stdexcept>
#include <vector>

#include "phiquad/b200.hpp"

namespace phiquad {

struct MonicQuartic {
    double a3 = 0.0, a2 = 0.0, a1 = 0.0, a0 = 1.0;
    template <class T>
    T eval(T x) const {
        return (((x + a3) * x + a2) * x + a1) * x + a0;
    }
    template <class T>
    T deriv(T x) const {
        return ((4.0 * x + 3.0 * a3) * x + 2.0 * a2) * x + a1;
    }
};

inline std::array<std::complex<double>, 4> quartic_roots(const MonicQuartic& q) {
    const double c[4] = {q.a3, q.a2, q.a1, q.a0};
    double z[8];
    b200::check(pq_quartic_roots(c, z));
    return {std::complex<double>(z[0], z[1]), std::complex<double>(z[2], z[3]), std::complex<double>(z[4], z[5]),
            std::complex<double>(z[6], z[7])};
}

inline std::vector<double> real_roots_greater_one(const MonicQuartic& q) {
    const double c[4] = {q.a3, q.a2, q.a1, q.a0};
    double r[4];
    int cnt = 0;
    b200::check(pq_real_roots_greater_one(c, r, &cnt));
    return std::vector<double>(r, r + cnt);
}

/// Illinois regula falsi on a bracketing [lo, hi] (bisection fallback), stops at width <= tol.
template <class F>
double find_root_monotone(F&& f, double lo, double hi, double tol) {
    if (!(lo < hi)) throw std::invalid_argument("find_root_monotone: empty interval");
    double flo = f(lo), fhi = f(hi);
    if (flo == 0.0) return lo;
    if (fhi == 0.0) return hi;
    if ((flo > 0.0) == (fhi > 0.0)) throw std::invalid_argument("find_root_monotone: endpoints do not bracket a root");
    int side = 0;
    for (int it = 0; it < 200 && hi - lo > tol; ++it) {
        double mid = hi - fhi * (hi - lo) / (fhi - flo);
        if (!(mid > lo && mid < hi) || !std::isfinite(mid)) mid = 0.5 * (lo + hi);
        const double fm = f(mid);
        if (fm == 0.0) return mid;
        if ((fm > 0.0) == (flo > 0.0)) {
            lo = mid;
            flo = fm;
            if (side == -1) fhi *= 0.5;
            side = -1;
        } else {
            hi = mid;
            fhi = fm;
            if (side == 1) flo *= 0.5;
            side = 1;
        }
    }
    return 0.5 * (lo + hi);
}

}  // namespace phiquad
