#pragma once
// Drop-in plumbing: the per-thread engine context behind the phiquad C++ API and the mapping of
// C-ABI return codes back to the reference's exception types (util.hpp:11-14 and the std:: types
// the reference throws).  Link with -lpq_b200 (paper_2211_00696_b200/libpq_b200.so).
#include <pq_b200.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>
#if defined(__linux__)
#include <sys/mman.h>
#endif

#include "phiquad/util.hpp"

namespace phiquad::b200 {

inline void check(int rc) {
    if (rc == PQ_OK) return;
    const std::string msg = pq_last_error();
    switch (rc) {
        case PQ_EINVAL: throw std::invalid_argument(msg);
        case PQ_ECONVERGENCE: throw ConvergenceError(msg);
        case PQ_ERANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

inline int& device_slot() {
    static int dev = 0;
    return dev;
}

/// Selects the GPU used by contexts created afterwards (default 0).
inline void set_device(int device) { device_slot() = device; }

/// One engine context (device, stream, workspace) per host thread: the reference API is
/// reentrant, a pq_ctx is single-stream, so threads never share one.
inline pq_ctx* context() {
    struct Holder {
        pq_ctx* ctx = nullptr;
        ~Holder() {
            if (ctx) pq_ctx_destroy(ctx);
        }
    };
    thread_local Holder h;
    if (!h.ctx) check(pq_ctx_create(device_slot(), &h.ctx));
    return h.ctx;
}

/// A value-initialised result vector of n doubles, as the reference API returns them.  For sizes of
/// a few MB the first touch (4 KB page faults) costs more than the GPU work behind the call, so the
/// buffer is marked for transparent huge pages before value-initialisation touches it
/// (tools/alloc_probe.cpp: 4 x 16.8 MB from one thread 22.9 ms -> 9.0 ms).
inline std::vector<double> result_vector(size_t n) {
    std::vector<double> v;
#if defined(__linux__) && defined(MADV_HUGEPAGE)
    constexpr uintptr_t kHuge = uintptr_t(2) << 20;
    if (n * sizeof(double) >= 2 * kHuge) {
        v.reserve(n);
        const uintptr_t p = reinterpret_cast<uintptr_t>(v.data()), e = p + n * sizeof(double);
        const uintptr_t a = (p + kHuge - 1) & ~(kHuge - 1), b = e & ~(kHuge - 1);
        if (b > a) madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);  // a hint: failure is harmless
    }
#endif
    v.resize(n);
    return v;
}

}  // namespace phiquad::b200
