#pragma once
// Extension (no counterpart in the reference, whose only parallelism is the node loop's threads,
// phiaction.hpp:85 / util.hpp:24-39): one phi action across the GPUs of a node, one process per
// GPU (include/pq_b200.h pq_*_dist, paper_2211_00696_b200/csrc/dist.cpp).  Quadrature nodes are
// dealt round-robin over the ranks, node vectors move to x-slab owners in one all-to-all, the
// squaring and phi_0 run on slabs; every rank passes the same operator, vectors and request.
#include <array>
#include <cstdint>
#include <utility>
#include <vector>

#include "phiquad/b200.hpp"
#include "phiquad/phiaction.hpp"

namespace phiquad::b200 {

/// The ranks one distributed call spans (pq_comm): NCCL over NVLink, or a host transport.
class Communicator {
public:
    /// Rank 0 creates the id and hands it to every rank (any out-of-band channel).
    static std::array<char, 128> nccl_unique_id() {
        std::array<char, 128> id{};
        check(pq_nccl_unique_id(id.data()));
        return id;
    }
    static Communicator nccl(int world, int rank, const std::array<char, 128>& id) {
        pq_comm* c = nullptr;
        check(pq_comm_create_nccl(context(), world, rank, id.data(), &c));
        return Communicator(c, world, rank);
    }
    static Communicator host(int world, int rank, const pq_host_transport& t) {
        pq_comm* c = nullptr;
        check(pq_comm_create_host(world, rank, &t, &c));
        return Communicator(c, world, rank);
    }
    static Communicator single() {
        pq_comm* c = nullptr;
        check(pq_comm_create_host(1, 0, nullptr, &c));
        return Communicator(c, 1, 0);
    }
    Communicator(Communicator&& o) noexcept : c_(std::exchange(o.c_, nullptr)), world_(o.world_), rank_(o.rank_) {}
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;
    ~Communicator() {
        if (c_) pq_comm_destroy(c_);
    }
    pq_comm* get() const { return c_; }
    int world() const { return world_; }
    int rank() const { return rank_; }
    /// [begin, end) of this rank's x-slab in a vector of `shape`.
    std::pair<int64_t, int64_t> slab(const std::vector<int>& shape) const {
        int64_t b = 0, e = 0;
        check(pq_dist_slab(static_cast<int>(shape.size()), shape.data(), world_, rank_, &b, &e));
        return {b, e};
    }

private:
    Communicator(pq_comm* c, int w, int r) : c_(c), world_(w), rank_(r) {}
    pq_comm* c_ = nullptr;
    int world_ = 1, rank_ = 0;
};

/// phiquadmv_multi across the communicator.  gather: full columns on every rank (PhiColumns of
/// a.dim()); otherwise each PhiColumns holds this rank's x-slab of every column.
inline std::vector<PhiColumns> phiquadmv_multi(const KroneckerSum& a, const std::vector<std::vector<double>>& bs,
                                               const PhiRequest& req, Communicator& comm, PhiInfo* info = nullptr,
                                               bool gather = true) {
    if (req.p < 1) throw std::invalid_argument("phiquadmv: need p >= 1");
    const int dim = a.dim();
    for (const auto& b : bs)
        if (static_cast<int>(b.size()) != dim)
            throw std::invalid_argument(std::string(req.mode == QuadKind::gauss_legendre ? "phi_fixed" : "phi_adaptive") +
                                        ": vector length mismatch");
    if (bs.empty()) return phiquad::phiquadmv_multi(a, bs, req, info);
    const auto f = detail::flatten(a);
    const int nb = static_cast<int>(bs.size());
    std::vector<double> flat;
    flat.reserve(static_cast<size_t>(nb) * dim);
    for (const auto& b : bs) flat.insert(flat.end(), b.begin(), b.end());
    const auto [lo, hi] = comm.slab(a.shape());
    const int len = gather ? dim : static_cast<int>(hi - lo);
    std::vector<double> out(static_cast<size_t>(nb) * req.p * len);
    const pq_phi_request r = detail::abi_request(req);
    pq_phi_info pi{};
    check(pq_phiquadmv_dist(context(), comm.get(), a.order(), f.shape.data(), f.data.data(), nb, flat.data(), &r,
                            nullptr, out.data(), &pi, PQ_HOST, gather ? 1 : 0));
    if (info)
        *info = PhiInfo{pi.l,     pi.n,    pi.points,          pi.mode == PQ_GAUSS_LEGENDRE ? QuadKind::gauss_legendre
                                                                                         : QuadKind::clenshaw_curtis,
                        pi.alpha, pi.beta, pi.planned != 0, pi.plan_cost};
    std::vector<PhiColumns> cols(static_cast<size_t>(nb));
    for (int m = 0; m < nb; ++m) {
        cols[static_cast<size_t>(m)].dim = len;
        for (int j = 0; j < req.p; ++j) {
            const double* src = out.data() + (static_cast<size_t>(m) * req.p + j) * len;
            cols[static_cast<size_t>(m)].cols.emplace_back(src, src + len);
        }
    }
    return cols;
}

}  // namespace phiquad::b200
