#pragma once
// Drop-in plumbing: the per-thread engine context behind the phiquad C++ API and the mapping of
// C-ABI return codes back to the reference's exception types (util.hpp:11-14 and the std:: types
// the reference throws).  Link with -lpq_b200 (paper_2211_00696_b200/libpq_b200.so).
#include <pq_b200.h>

#include <stdexcept>
#include <string>

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

}  // namespace phiquad::b200
