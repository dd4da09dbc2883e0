// Multi-GPU phi actions, one process per GPU.  Replaces the reference's node
// loop parallel_for (phiaction.hpp:85, util.hpp:24-39) and its serial squaring
// (phiaction.hpp:255-272, 293-301) with a partition over the ranks of one node:
//
//  1. quadrature nodes: rank r evaluates the node vectors v_i = (E_i0 (x) E_i1 (x) E_i2) b of the
//     nodes it owns (i % G == r; the adaptive CC ladder deals each level's fresh nodes the same
//     way) -- exponentials and DMMA mode products for its nodes only;
//  2. node transpose: ONE all-to-all moves every node vector's x-slab to the slab's owner (rank h
//     owns x-indices i0 in [s_h, s_h+1), a contiguous range of every vector).  Each rank then holds
//     all q node vectors of its slab and forms the weighted sums y_j = sum_i w_i theta_i^(j-1)/(j-1)! v_i
//     in ascending node order exactly as the single-GPU combine (phiaction.hpp:96-111) -- no
//     floating-point reduction across ranks, so the node phase is bitwise independent of G.
//     Bytes per rank: (q/G) nb N (G-1)/G doubles, versus p nb N (G-1)/G for a reduce-scatter of
//     the partial sums -- fewer whenever q/G < p (configs 3 and 5 at G >= 4), and the CC ladder
//     needs no per-level reduction of fine AND coarse sums (its error statistics are max-norms:
//     one all-reduce(max) of 2 nb p scalars per level, exact);
//  3. distributed squaring on slabs: per step modes 1..d-1 act inside the slab, the slab is
//     packed into per-destination blocks and flipped to pencils (rank r: all i0, trailing indices
//     [c_r, c_r+1)) by an all-to-all, mode 0 acts on the pencil, a second all-to-all flips back,
//     the blocks are unpacked, and the doubling combination is elementwise (k_sq_combine2).
//     phi_0 = exp_action(b) is one more distributed Kronecker apply;
//  4. optionally, the slabs are all-gathered into full vectors on every rank.
//
// Transport: NCCL (loaded with dlopen -- the copy torch already mapped when present, else the
// system libnccl.so.2) with grouped ncclSend/ncclRecv and ncclAllReduce on the context stream;
// or a host transport (caller-supplied alltoallv / allreduce-max callbacks on pinned host
// buffers -- e.g. torch.distributed over gloo), which lets several processes share ONE GPU in the
// tests: collectives go through the host, so no kernel ever waits on another process.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "engine.hpp"
#include "pq_b200.h"

using namespace pqb;

struct pq_comm {
    int world = 1, rank = 0;
    int kind = PQ_COMM_HOST;
    ncclComm_t nccl = nullptr;
    pq_host_transport host{};
    double* hs = nullptr;  // pinned staging (host transport)
    size_t hs_cap = 0;
    double* hr = nullptr;
    size_t hr_cap = 0;
    double bytes_sent = 0.0;  // doubles * 8 sent to other ranks
    uint64_t exchanges = 0;
    // peer transport: symmetric buffers (cudaMalloc + CUDA IPC), every rank's copy mapped here
    struct PeerBuf {
        double* local = nullptr;
        size_t bytes = 0;
        std::vector<double*> peer;  // [rank] -> mapped pointer (peer[rank] = local)
    };
    std::map<std::string, PeerBuf> pbufs;
};

namespace {

void need(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(what);
}

// ------------------------------------------------------------------ NCCL (dlopen) --------

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    std::string why;
};

const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        const char* env = std::getenv("PQ_NCCL_LIB");
        void* h = env ? nullptr : dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if mapped
        if (!h) h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("cannot load NCCL: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            if (!f && a.why.empty()) a.why = std::string("NCCL symbol missing: ") + name;
        };
        sym(a.getUniqueId, "ncclGetUniqueId");
        sym(a.commInitRank, "ncclCommInitRank");
        sym(a.commDestroy, "ncclCommDestroy");
        sym(a.send, "ncclSend");
        sym(a.recv, "ncclRecv");
        sym(a.groupStart, "ncclGroupStart");
        sym(a.groupEnd, "ncclGroupEnd");
        sym(a.allReduce, "ncclAllReduce");
        sym(a.errorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.why.empty()) throw CudaError(api.why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string("NCCL ") + what + ": " + nccl_api().errorString(r));
}

// ------------------------------------------------------------------ transport ------------

struct Piece {
    int peer;
    double* ptr;
    long long count;
};

double* grow_pinned(double*& buf, size_t& cap, size_t count) {
    if (cap < count) {
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        cap = 0;
        cuda_check(cudaMallocHost(reinterpret_cast<void**>(&buf), std::max<size_t>(count, 1) * sizeof(double)),
                   "cudaMallocHost(transport)");
        cap = std::max<size_t>(count, 1);
    }
    return buf;
}

// Point-to-point exchange on the context stream.  Pieces to / from the same peer are matched in
// the order given (sender and receiver enumerate them in the same order).  Self pieces are local
// device copies (the i-th self send lands in the i-th self receive).
void exchange(pq_ctx& c, pq_comm& m, const std::vector<Piece>& sends, const std::vector<Piece>& recvs) {
    NvtxRange nvtx("pq_exchange");
    ++m.exchanges;
    std::vector<const Piece*> self_s, self_r;
    for (const auto& s : sends)
        if (s.peer == m.rank && s.count > 0) self_s.push_back(&s);
    for (const auto& r : recvs)
        if (r.peer == m.rank && r.count > 0) self_r.push_back(&r);
    need(self_s.size() == self_r.size(), "exchange: unmatched local pieces");
    for (size_t i = 0; i < self_s.size(); ++i) {
        need(self_s[i]->count == self_r[i]->count, "exchange: local piece size mismatch");
        cuda_check(cudaMemcpyAsync(self_r[i]->ptr, self_s[i]->ptr, sizeof(double) * self_s[i]->count,
                                   cudaMemcpyDeviceToDevice, c.stream),
                   "exchange (local)");
    }
    for (const auto& s : sends)
        if (s.peer != m.rank) m.bytes_sent += 8.0 * static_cast<double>(s.count);
    if (m.world == 1) return;
    if (m.kind == PQ_COMM_NCCL) {
        const NcclApi& api = nccl_api();
        nccl_check(api.groupStart(), "group start");
        for (const auto& s : sends)
            if (s.peer != m.rank && s.count > 0)
                nccl_check(api.send(s.ptr, static_cast<size_t>(s.count), ncclFloat64, s.peer, m.nccl, c.stream), "send");
        for (const auto& r : recvs)
            if (r.peer != m.rank && r.count > 0)
                nccl_check(api.recv(r.ptr, static_cast<size_t>(r.count), ncclFloat64, r.peer, m.nccl, c.stream), "recv");
        nccl_check(api.groupEnd(), "group end");
        return;
    }
    // host transport: stage per-peer concatenations through pinned memory, one alltoallv callback
    std::vector<int64_t> sc(static_cast<size_t>(m.world), 0), rc(static_cast<size_t>(m.world), 0);
    for (const auto& s : sends)
        if (s.peer != m.rank) sc[static_cast<size_t>(s.peer)] += s.count;
    for (const auto& r : recvs)
        if (r.peer != m.rank) rc[static_cast<size_t>(r.peer)] += r.count;
    const size_t st = std::accumulate(sc.begin(), sc.end(), size_t(0));
    const size_t rt = std::accumulate(rc.begin(), rc.end(), size_t(0));
    double* hs = grow_pinned(m.hs, m.hs_cap, st);
    double* hr = grow_pinned(m.hr, m.hr_cap, rt);
    std::vector<size_t> off(static_cast<size_t>(m.world), 0);
    for (int h = 1; h < m.world; ++h) off[static_cast<size_t>(h)] = off[static_cast<size_t>(h) - 1] + sc[static_cast<size_t>(h) - 1];
    for (const auto& s : sends) {
        if (s.peer == m.rank || s.count == 0) continue;
        size_t& o = off[static_cast<size_t>(s.peer)];
        cuda_check(cudaMemcpyAsync(hs + o, s.ptr, sizeof(double) * s.count, cudaMemcpyDeviceToHost, c.stream), "D2H (send)");
        o += static_cast<size_t>(s.count);
    }
    cuda_check(cudaStreamSynchronize(c.stream), "exchange sync");
    need(m.host.alltoallv != nullptr, "host transport: no alltoallv");
    if (m.host.alltoallv(m.host.user, hs, sc.data(), hr, rc.data()) != 0)
        throw CudaError("host transport: alltoallv callback failed");
    std::fill(off.begin(), off.end(), 0);
    for (int h = 1; h < m.world; ++h) off[static_cast<size_t>(h)] = off[static_cast<size_t>(h) - 1] + rc[static_cast<size_t>(h) - 1];
    for (const auto& r : recvs) {
        if (r.peer == m.rank || r.count == 0) continue;
        size_t& o = off[static_cast<size_t>(r.peer)];
        cuda_check(cudaMemcpyAsync(r.ptr, hr + o, sizeof(double) * r.count, cudaMemcpyHostToDevice, c.stream), "H2D (recv)");
        o += static_cast<size_t>(r.count);
    }
}

// In-place all-reduce (max) of n device doubles.
void allreduce_max(pq_ctx& c, pq_comm& m, double* dev, int n) {
    if (m.world == 1 || n == 0) return;
    if (m.kind == PQ_COMM_NCCL) {
        nccl_check(nccl_api().allReduce(dev, dev, static_cast<size_t>(n), ncclFloat64, ncclMax, m.nccl, c.stream),
                   "allreduce");
        return;
    }
    double* hs = grow_pinned(m.hs, m.hs_cap, static_cast<size_t>(n));
    cuda_check(cudaMemcpyAsync(hs, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream), "D2H (allreduce)");
    cuda_check(cudaStreamSynchronize(c.stream), "allreduce sync");
    need(m.host.allreduce_max != nullptr, "host transport: no allreduce_max");
    if (m.host.allreduce_max(m.host.user, hs, n) != 0) throw CudaError("host transport: allreduce_max callback failed");
    cuda_check(cudaMemcpyAsync(dev, hs, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream), "H2D (allreduce)");
}

// ------------------------------------------------------------------ geometry -------------

struct Geom {
    int G = 1, r = 0, d = 1;
    int n[3] = {1, 1, 1};
    long long N = 1, rest = 1;
    std::vector<int> s;  // x-slab bounds, G + 1
    SlabCuts cuts;       // pencil bounds over the trailing index
    int sg(int h) const { return s[static_cast<size_t>(h) + 1] - s[static_cast<size_t>(h)]; }
    long long S(int h) const { return static_cast<long long>(sg(h)) * rest; }
    long long lo(int h) const { return static_cast<long long>(s[static_cast<size_t>(h)]) * rest; }
    long long C(int h) const { return cuts.cb[h + 1] - cuts.cb[h]; }
};

Geom make_geom(int d, const int* shape, int world, int rank) {
    need(world >= 1 && world <= 16, "distributed phi: 1 to 16 ranks");
    need(rank >= 0 && rank < world, "distributed phi: bad rank");
    Geom g;
    g.G = world;
    g.r = rank;
    g.d = d;
    for (int k = 0; k < d; ++k) {
        g.n[k] = shape[k];
        g.N *= shape[k];
    }
    g.rest = g.N / shape[0];
    need(shape[0] >= world, "distributed phi: the first factor needs at least one x-slab per rank");
    g.s.resize(static_cast<size_t>(world) + 1);
    for (int h = 0; h <= world; ++h) g.s[static_cast<size_t>(h)] = static_cast<int>(static_cast<long long>(shape[0]) * h / world);
    g.cuts.G = world;
    for (int h = 0; h <= world; ++h) g.cuts.cb[h] = g.rest * h / world;
    return g;
}

// ------------------------------------------------------------------ distributed pieces ---

// y[col] = (E_0 (x) ... (x) E_{d-1}) x[col] for ncols columns in slab layout (x[col] at
// x + col*x_stride, S_r doubles; y[col] at y + col*S_r).  Modes 1..d-1 inside the slab, slab ->
// pencil all-to-all, mode 0 on the pencil, pencil -> slab all-to-all.
void dist_kron(pq_ctx& c, pq_comm& m, const Geom& g, const double* const* E, const int2* const* B, const double* x,
               long long x_stride, int ncols, double* y) {
    const int r = g.r, sg = g.sg(r);
    const long long S = g.S(r), Cr = g.C(r);
    const size_t tot = static_cast<size_t>(ncols) * std::max<long long>(S, 1);
    const size_t ptot = static_cast<size_t>(ncols) * g.n[0] * std::max<long long>(Cr, 1);
    double* U = ws(c, "dk_U", std::max(tot, ptot));
    double* Bk = ws(c, "dk_B", tot);
    double* P = ws(c, "dk_P", ptot);
    // 1. modes 1..d-1 on the slab (each column a (sg, n1[, n2]) tensor)
    if (g.d == 1) {
        for (int col = 0; col < ncols; ++col)
            cuda_check(cudaMemcpyAsync(U + col * S, x + col * x_stride, sizeof(double) * S, cudaMemcpyDeviceToDevice,
                                       c.stream),
                       "slab copy");
    } else if (sg > 0) {
        const int sh[3] = {sg, g.n[1], g.d > 2 ? g.n[2] : 1};
        if (g.d == 2) {
            mode_product_dev(c, 2, sh, 1, E[1], B ? B[1] : nullptr, x, x_stride, U, S, ncols);
        } else {
            double* T = ws(c, "dk_T", tot);
            mode_product_dev(c, 3, sh, 1, E[1], B ? B[1] : nullptr, x, x_stride, T, S, ncols);
            mode_product_dev(c, 3, sh, 2, E[2], B ? B[2] : nullptr, T, S, U, S, ncols);
        }
    }
    // 2. pack into per-destination blocks, 3. flip to pencils
    SlabCuts cuts = g.cuts;
    cuts.ncols = ncols;
    {
        KernelProbe kp(c, "k_slab_blocks(pack)", 16.0 * static_cast<double>(tot));
        launch_slab_blocks(true, sg, g.rest, cuts, U, Bk, c.stream);
        count_launch(c);
    }
    std::vector<Piece> sends, recvs;
    for (int h = 0; h < g.G; ++h)
        for (int col = 0; col < ncols; ++col) {
            sends.push_back({h, Bk + ncols * sg * cuts.cb[h] + col * sg * g.C(h), sg * g.C(h)});
            recvs.push_back({h, P + (col * g.n[0] + g.s[static_cast<size_t>(h)]) * Cr, g.sg(h) * Cr});
        }
    exchange(c, m, sends, recvs);
    // 4. mode 0 on the pencil (n0 x C_r per column)
    if (Cr > 0) {
        const int sh[2] = {g.n[0], static_cast<int>(Cr)};
        mode_product_dev(c, 2, sh, 0, E[0], B ? B[0] : nullptr, P, g.n[0] * Cr, U, g.n[0] * Cr, ncols);
    }
    // 5. flip back into blocks, 6. unpack into the slab
    sends.clear();
    recvs.clear();
    for (int h = 0; h < g.G; ++h)
        for (int col = 0; col < ncols; ++col) {
            sends.push_back({h, U + (col * g.n[0] + g.s[static_cast<size_t>(h)]) * Cr, g.sg(h) * Cr});
            recvs.push_back({h, Bk + ncols * sg * cuts.cb[h] + col * sg * g.C(h), sg * g.C(h)});
        }
    exchange(c, m, sends, recvs);
    KernelProbe kp(c, "k_slab_blocks(unpack)", 16.0 * static_cast<double>(tot));
    launch_slab_blocks(false, sg, g.rest, cuts, Bk, y, c.stream);
    count_launch(c);
}

// ------------------------------------------------------------------ peer transport -------
// Symmetric buffers mapped into every rank (CUDA IPC: NVLink loads/stores between the GPUs of a
// node; in the tests, processes sharing one GPU) and mode products whose epilogue stores each
// output row straight into the rank that owns it (kernels.hpp RemoteMap): the slab <-> pencil
// flips need no pack / unpack kernel and no staging -- the transfer is the GEMM's own store
// stream.  Ranks synchronise at each flip with a stream drain and a host barrier (the host
// transport's allreduce), so no kernel ever waits on another rank's kernel.

void peer_barrier(pq_ctx& c, pq_comm& m) {
    NvtxRange nvtx("pq_peer_barrier");
    cuda_check(cudaStreamSynchronize(c.stream), "peer barrier sync");
    if (m.world == 1) return;
    double token = 0.0;
    if (m.host.allreduce_max(m.host.user, &token, 1) != 0) throw CudaError("peer transport: barrier failed");
}

// collective: every rank calls it with the same name and byte count at the same point
// (keep: leading bytes of the old buffer carried into a grown one)
pq_comm::PeerBuf& peer_buffer(pq_ctx& c, pq_comm& m, const std::string& name, size_t bytes, size_t keep = 0) {
    pq_comm::PeerBuf& b = m.pbufs[name];
    if (b.bytes >= bytes && b.local) return b;
    peer_barrier(c, m);  // nobody writes into the old buffers any more
    for (int h = 0; h < m.world; ++h)
        if (h != m.rank && h < static_cast<int>(b.peer.size()) && b.peer[static_cast<size_t>(h)])
            cudaIpcCloseMemHandle(b.peer[static_cast<size_t>(h)]);
    double* old = b.local;
    const size_t old_bytes = b.bytes;
    b = pq_comm::PeerBuf{};
    cuda_check(cudaMalloc(&b.local, std::max<size_t>(bytes, 256)), "cudaMalloc(peer buffer)");
    if (old) {
        if (keep > 0)
            cuda_check(cudaMemcpy(b.local, old, std::min(keep, old_bytes), cudaMemcpyDeviceToDevice), "peer buffer copy");
        cudaFree(old);
    }
    b.bytes = std::max<size_t>(bytes, 256);
    b.peer.assign(static_cast<size_t>(m.world), nullptr);
    b.peer[static_cast<size_t>(m.rank)] = b.local;
    if (m.world > 1) {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        cudaIpcMemHandle_t mine;
        cuda_check(cudaIpcGetMemHandle(&mine, b.local), "cudaIpcGetMemHandle");
        // all-gather of the 64-byte handles through the host transport (8 doubles each)
        std::vector<double> send(static_cast<size_t>(m.world - 1) * 8), recv(static_cast<size_t>(m.world - 1) * 8);
        std::vector<int64_t> sc(static_cast<size_t>(m.world), 8), rc(static_cast<size_t>(m.world), 8);
        sc[static_cast<size_t>(m.rank)] = rc[static_cast<size_t>(m.rank)] = 0;
        for (int k = 0; k < m.world - 1; ++k) std::memcpy(send.data() + 8 * k, &mine, 64);
        if (m.host.alltoallv(m.host.user, send.data(), sc.data(), recv.data(), rc.data()) != 0)
            throw CudaError("peer transport: handle exchange failed");
        int k = 0;
        for (int h = 0; h < m.world; ++h) {
            if (h == m.rank) continue;
            cudaIpcMemHandle_t theirs;
            std::memcpy(&theirs, recv.data() + 8 * k++, 64);
            void* ptr = nullptr;
            cuda_check(cudaIpcOpenMemHandle(&ptr, theirs, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            b.peer[static_cast<size_t>(h)] = static_cast<double*>(ptr);
        }
    }
    return b;
}

// the fused flips apply when every pencil owns whole n2-rows of the trailing plane (G | n1) and
// all row offsets keep 16-byte alignment
bool peer_fused_ok(const Geom& g) {
    if (g.d != 3 || g.n[1] % g.G != 0 || g.n[2] % 2 != 0 || g.rest % 2 != 0) return false;
    for (int h = 0; h <= g.G; ++h)
        if (g.cuts.cb[h] % g.n[2] != 0) return false;
    return true;
}

// dist_kron with the flips fused into the mode products: modes 1 (local) -> mode 2 storing into
// every rank's pencil buffer -> barrier -> mode 0 on the pencil storing into every rank's slab of
// `ydst` -> barrier.  The result is ydst.local [col][S_r].
void dist_kron_peer(pq_ctx& c, pq_comm& m, const Geom& g, const double* const* E, const int2* const* B,
                    const double* x, long long x_stride, int ncols, pq_comm::PeerBuf& ydst) {
    const int r = g.r, sg = g.sg(r);
    const long long S = g.S(r);
    long long cmax = 0;
    for (int h = 0; h < g.G; ++h) cmax = std::max(cmax, g.C(h));
    pq_comm::PeerBuf& pen = peer_buffer(c, m, "ppencil", sizeof(double) * ncols * g.n[0] * std::max<long long>(cmax, 1));
    RemoteMap rm1, rm2;
    rm1.mode = 1;
    rm2.mode = 2;
    for (RemoteMap* rm : {&rm1, &rm2}) {
        rm->G = g.G;
        rm->me = r;
        rm->n0 = g.n[0];
        rm->n1 = g.n[1];
        rm->n2 = g.n[2];
        rm->rest = g.rest;
        for (int h = 0; h <= g.G; ++h) {
            rm->s[h] = g.s[static_cast<size_t>(h)];
            rm->cb[h] = g.cuts.cb[h];
        }
    }
    for (int h = 0; h < g.G; ++h) {
        rm1.base[h] = pen.peer[static_cast<size_t>(h)];
        rm2.base[h] = ydst.peer[static_cast<size_t>(h)];
    }
    const RemoteMap* rm1_dev = static_cast<const RemoteMap*>(arena_push(c, &rm1, sizeof rm1));
    const RemoteMap* rm2_dev = static_cast<const RemoteMap*>(arena_push(c, &rm2, sizeof rm2));
    arena_flush(c);
    const size_t tot = static_cast<size_t>(ncols) * std::max<long long>(S, 1);
    double* U = ws(c, "dk_U", tot);
    const int sh[3] = {sg, g.n[1], g.n[2]};
    mode_product_dev(c, 3, sh, 1, E[1], B ? B[1] : nullptr, x, x_stride, U, S, ncols);
    // mode 2: each output row (r, i1) is an n2-row of the pencil of the rank owning i1*n2
    mode_product_dev(c, 3, sh, 2, E[2], B ? B[2] : nullptr, U, S, U, S, ncols, rm1_dev);
    for (int h = 0; h < g.G; ++h)
        if (h != r) m.bytes_sent += 8.0 * ncols * sg * static_cast<double>(g.C(h));
    ++m.exchanges;
    peer_barrier(c, m);
    const long long Cr = g.C(r);
    if (Cr > 0) {
        const int shp[2] = {g.n[0], static_cast<int>(Cr)};
        // mode 0: output row i0 goes to the rank owning x-slab row i0, at its pencil columns
        mode_product_dev(c, 2, shp, 0, E[0], B ? B[0] : nullptr, pen.local, g.n[0] * Cr, pen.local, g.n[0] * Cr, ncols,
                         rm2_dev);
        for (int h = 0; h < g.G; ++h)
            if (h != r) m.bytes_sent += 8.0 * ncols * g.sg(h) * static_cast<double>(Cr);
    }
    ++m.exchanges;
    peer_barrier(c, m);
}

// node vectors of the owned nodes (full length, pool [a][m][N]) -> every node's slab on its
// owner (slab pool [slot][m][S_r]); `owner_of(slot)` and the local index of owned slots
void node_transpose(pq_ctx& c, pq_comm& m, const Geom& g, int nb, const std::vector<int>& slots, const double* pool,
                    double* slab_pool) {
    if (m.kind == PQ_COMM_PEER) {
        // straight into every rank's IPC-mapped slab pool (peer copies over NVLink), one barrier
        pq_comm::PeerBuf& sp = m.pbufs["pslabpool"];
        int a = 0;
        for (int slot : slots) {
            if (slot % g.G != g.r) continue;
            for (int mm = 0; mm < nb; ++mm)
                for (int h = 0; h < g.G; ++h) {
                    double* dst = sp.peer[static_cast<size_t>(h)] + (static_cast<long long>(slot) * nb + mm) * g.S(h);
                    const double* src = pool + (static_cast<long long>(a) * nb + mm) * g.N + g.lo(h);
                    cuda_check(cudaMemcpyAsync(dst, src, sizeof(double) * g.S(h), cudaMemcpyDeviceToDevice, c.stream),
                               "node transpose (peer)");
                    if (h != g.r) m.bytes_sent += 8.0 * g.S(h);
                }
            ++a;
        }
        ++m.exchanges;
        peer_barrier(c, m);
        return;
    }
    std::vector<Piece> sends, recvs;
    int a = 0;
    for (int slot : slots) {
        const int owner = slot % g.G;
        if (owner == g.r) {
            for (int mm = 0; mm < nb; ++mm)
                for (int h = 0; h < g.G; ++h)
                    sends.push_back({h, const_cast<double*>(pool) + (static_cast<long long>(a) * nb + mm) * g.N + g.lo(h),
                                     g.S(h)});
            ++a;
        }
        for (int mm = 0; mm < nb; ++mm)
            recvs.push_back({owner, slab_pool + (static_cast<long long>(slot) * nb + mm) * g.S(g.r), g.S(g.r)});
    }
    exchange(c, m, sends, recvs);
}

std::vector<int> owned(const std::vector<int>& slots, const Geom& g) {
    std::vector<int> o;
    for (int s : slots)
        if (s % g.G == g.r) o.push_back(s);
    return o;
}

double* slab_pool_grow(pq_ctx& c, pq_comm& m, const Geom& g, int slots, int nb, long long S, int used) {
    if (m.kind == PQ_COMM_PEER) {  // symmetric, sized for the largest slab
        long long smax = 0;
        for (int h = 0; h < g.G; ++h) smax = std::max(smax, g.S(h));
        const size_t want = static_cast<size_t>(std::max(slots, 1)) * nb * std::max<long long>(smax, 1) * sizeof(double);
        return peer_buffer(c, m, "pslabpool", want, static_cast<size_t>(used) * nb * S * sizeof(double)).local;
    }
    DevBuf& b = c.bufs["dslabpool"];
    const size_t want = static_cast<size_t>(std::max(slots, 1)) * nb * std::max<long long>(S, 1) * sizeof(double);
    if (b.bytes < want) {
        double* np = static_cast<double*>(ws_alloc(c, want, "dslabpool"));
        if (b.p && used > 0)
            cuda_check(cudaMemcpyAsync(np, b.p, static_cast<size_t>(used) * nb * S * sizeof(double), cudaMemcpyDeviceToDevice,
                                       c.stream),
                       "pool copy");
        ws_retire(c, b.p);
        b.p = np;
        b.bytes = want;
    }
    return static_cast<double*>(b.p);
}

// Gauss node phase: acc [nb][p][S_r] = the slab of phi_j(2^-l A) b (phiaction.hpp:134-145)
// The reduce-scatter alternative: every rank forms the weighted partial sums of its
// own nodes over the FULL vector (node_sweep's fused combine), sends slab h of them to rank h, and
// each rank adds the G partial slabs in ascending rank order.  Moves p nb (N - S_r) doubles per rank
// against (q/G) nb (N - S_r) for the node transpose: used when ceil(q/G) > p.
bool gauss_use_reduce_scatter(int q, int G, int p) { return G > 1 && (q + G - 1) / G > p; }

void gauss_nodes_rs(pq_ctx& c, pq_comm& m, const Geom& g, const DevOp& op, int nb, const double* bs, int p,
                    const NodesWeights& rule, const PhiExps& px, const std::vector<int>& own, double* acc) {
    const long long S = g.S(g.r), N = op.N;
    long long Es[3];
    for (int k = 0; k < op.d; ++k) Es[k] = static_cast<long long>(op.n[k]) * op.n[k];
    double* part = ws(c, "dpart", static_cast<size_t>(nb) * p * N);  // [m][j][N]
    std::vector<double> coef;
    node_coefs(rule, own, p, coef);
    node_sweep(c, op, px.node, Es, static_cast<int>(own.size()), nb, bs, p, &coef, part, 1, nullptr, 0, px.node_band);
    const int cols = nb * p;
    double* recv = ws(c, "dpartslabs", static_cast<size_t>(g.G) * cols * std::max<long long>(S, 1));  // [h][col][S]
    std::vector<Piece> sends, recvs;
    for (int h = 0; h < g.G; ++h)
        for (int col = 0; col < cols; ++col) {
            sends.push_back({h, part + col * N + g.lo(h), g.S(h)});
            recvs.push_back({h, recv + (static_cast<long long>(h) * cols + col) * S, S});
        }
    exchange(c, m, sends, recvs);
    // acc[col] = sum over ranks h ascending of their partial slab (coefficient 1, fixed order)
    std::vector<double> ones(static_cast<size_t>(g.G), 1.0);
    std::vector<int> slots(static_cast<size_t>(g.G));
    std::iota(slots.begin(), slots.end(), 0);
    const double* one_dev = static_cast<const double*>(arena_push(c, ones.data(), ones.size() * sizeof(double)));
    const int* sl_dev = static_cast<const int*>(arena_push(c, slots.data(), slots.size() * sizeof(int)));
    arena_flush(c);
    for (int col = 0; col < cols; ++col) {
        KernelProbe kp(c, "k_combine(rank sum)", 8.0 * S * (g.G + 1));
        launch_combine(S, 1, g.G, recv + static_cast<long long>(col) * S, static_cast<long long>(cols) * S, sl_dev,
                       one_dev, acc + static_cast<long long>(col) * S, S, 1, c.stream);
        count_launch(c);
    }
}

void gauss_nodes(pq_ctx& c, pq_comm& m, const Geom& g, const DevOp& op, int nb, const double* bs, int p,
                 const NodesWeights& rule, const PhiExps& px, const std::vector<int>& own, double* acc) {
    const int q = rule.size();
    // (the peer transport moves node slabs with direct peer copies: no staging to save)
    if (m.kind != PQ_COMM_PEER && gauss_use_reduce_scatter(q, g.G, p)) {
        gauss_nodes_rs(c, m, g, op, nb, bs, p, rule, px, own, acc);
        return;
    }
    const long long S = g.S(g.r);
    long long Es[3];
    for (int k = 0; k < op.d; ++k) Es[k] = static_cast<long long>(op.n[k]) * op.n[k];
    double* pool = ws(c, "dpool", std::max<size_t>(own.size(), 1) * nb * op.N);
    node_sweep(c, op, px.node, Es, static_cast<int>(own.size()), nb, bs, p, nullptr, nullptr, 0, pool, 0, px.node_band);
    std::vector<int> all(static_cast<size_t>(q));
    std::iota(all.begin(), all.end(), 0);
    double* slab = slab_pool_grow(c, m, g, q, nb, S, 0);
    node_transpose(c, m, g, nb, all, pool, slab);
    std::vector<double> coef;
    node_coefs(rule, all, p, coef);
    const double* coef_dev = static_cast<const double*>(arena_push(c, coef.data(), coef.size() * sizeof(double)));
    const int* sl_dev = static_cast<const int*>(arena_push(c, all.data(), all.size() * sizeof(int)));
    arena_flush(c);
    if (S == 0) return;
    for (int mm = 0; mm < nb; ++mm) {
        KernelProbe kp(c, "k_combine", 8.0 * S * (q + p));
        launch_combine(S, p, q, slab + mm * S, static_cast<long long>(nb) * S, sl_dev, coef_dev, acc + mm * p * S, S, 1,
                       c.stream);
        count_launch(c);
    }
}

// Adaptive CC ladder (phiaction.hpp:156-245) on slabs.  Pool slots as in the single-GPU ladder:
// 0..12 = the 13-point rule, then each level's fresh (odd) nodes; slot s is evaluated by rank
// s % G.  px25 holds the exponentials of the owned slots among the first 25 (own25 order).
void cc_nodes(pq_ctx& c, pq_comm& m, const Geom& g, const DevOp& op, int l, int nb, const double* bs, int p,
              double eps, const PhiExps& px25, const std::vector<int>& own25, double* out, int* points_used) {
    if (!(eps > 0.0)) throw std::invalid_argument("phi_adaptive: need eps > 0");
    const long long S = g.S(g.r);
    const size_t col = static_cast<size_t>(nb) * p * S;
    long long nn[3], Es[3];
    for (int k = 0; k < op.d; ++k) Es[k] = nn[k] = static_cast<long long>(op.n[k]) * op.n[k];
    const NodesWeights& r25 = memo_rule(kClenshaw, 25);
    // sweeps the owned slots among `slots` (exponentials E[k] + idx*nn[k], idx = position among the
    // owned ones) and moves every slot's slab to this rank's slab pool
    double* slab = slab_pool_grow(c, m, g, 25, nb, S, 0);
    int used = 0;
    auto sweep = [&](const std::vector<int>& slots, const double* const* E, const int2* const* B) {
        const std::vector<int> mine = owned(slots, g);
        double* pool = ws(c, "dpool", std::max<size_t>(mine.size(), 1) * nb * op.N);
        if (!mine.empty()) node_sweep(c, op, E, Es, static_cast<int>(mine.size()), nb, bs, p, nullptr, nullptr, 0, pool, 0, B);
        slab = slab_pool_grow(c, m, g, used + static_cast<int>(slots.size()), nb, S, used);
        node_transpose(c, m, g, nb, slots, pool, slab);
        used += static_cast<int>(slots.size());
    };
    // exponentials of owned slots in a contiguous subrange [first, first+count) of own25
    auto sub = [&](int first, const double** E, const int2** B) {
        for (int k = 0; k < op.d; ++k) {
            E[k] = px25.node[k] ? px25.node[k] + first * nn[k] : nullptr;
            B[k] = px25.node_band[k] ? px25.node_band[k] + first * band_row_blocks(op.n[k]) : nullptr;
        }
    };
    {
        std::vector<int> s13(13);
        std::iota(s13.begin(), s13.end(), 0);
        const double* E[3];
        const int2* B[3];
        sub(0, E, B);
        sweep(s13, E, B);
    }
    int half = 3;
    const NodesWeights* rule = &memo_rule(kClenshaw, 2 * half + 1);
    std::vector<int> slot_of(static_cast<size_t>(rule->size()));
    for (int i = 0; i < rule->size(); ++i) slot_of[static_cast<size_t>(i)] = 2 * i;
    double* accs[2] = {out, ws(c, "dccacc", std::max<size_t>(col, 1))};
    int cur = 0;
    const bool fused = p <= 8;
    double* stats = ws(c, "dccstats", 2 * static_cast<size_t>(nb) * p);
    std::vector<double> hstats(2 * static_cast<size_t>(nb) * p);
    int level = 0;
    (void)r25;
    while (true) {
        const int half_next = 2 * half;
        if (half_next > (1 << 14)) throw ConvergenceFailure("phi_adaptive: no convergence within the node budget");
        const NodesWeights& fine = memo_rule(kClenshaw, 2 * half_next + 1);
        const int fresh = fine.size() / 2;
        ++level;
        int base = 2 * 0 + 1;  // level 1: fresh 13-rule nodes are slots 1, 3, ..., 11
        if (level >= 2) {
            base = used;
            std::vector<int> fs(static_cast<size_t>(fresh));
            std::iota(fs.begin(), fs.end(), used);
            const std::vector<int> mine = owned(fs, g);
            const double* E[3];
            const int2* B[3];
            PhiExps pxl;
            if (level == 2) {  // 25-rule odd nodes: own25 entries after the owned slots < 13
                const int first = static_cast<int>(std::count_if(own25.begin(), own25.end(), [](int s) { return s < 13; }));
                sub(first, E, B);
            } else {
                std::vector<double> th;
                for (int s : mine) th.push_back(fine.x[static_cast<size_t>(2 * (s - used) + 1)]);
                pxl = phi_exponentials(c, op, 1.0, l, th, false, false, "dccE" + std::to_string(level));
                for (int k = 0; k < op.d; ++k) {
                    E[k] = pxl.node[k];
                    B[k] = pxl.node_band[k];
                }
            }
            sweep(fs, E, B);
        }
        std::vector<int> fine_slot(static_cast<size_t>(fine.size()));
        for (int i = 0; i < rule->size(); ++i) fine_slot[static_cast<size_t>(2 * i)] = slot_of[static_cast<size_t>(i)];
        for (int k = 0; k < fresh; ++k)
            fine_slot[static_cast<size_t>(2 * k + 1)] = level == 1 ? 2 * k + 1 : base + k;
        const int nxt = 1 - cur;
        std::vector<int> idx(static_cast<size_t>(fine.size()));
        std::iota(idx.begin(), idx.end(), 0);
        std::vector<double> cf;
        node_coefs(fine, idx, p, cf);
        const double* cf_dev = static_cast<const double*>(arena_push(c, cf.data(), cf.size() * sizeof(double)));
        const int* sl_dev = static_cast<const int*>(arena_push(c, fine_slot.data(), fine_slot.size() * sizeof(int)));
        const double* cc_dev = nullptr;
        if (fused && level == 1) {  // coarse rule node k = fine node 2k
            std::vector<int> cidx(static_cast<size_t>(rule->size()));
            std::iota(cidx.begin(), cidx.end(), 0);
            std::vector<double> c7, cc(cf.size(), 0.0);
            node_coefs(*rule, cidx, p, c7);
            for (int k = 0; k < rule->size(); ++k)
                for (int j = 0; j < p; ++j) cc[static_cast<size_t>(2 * k) * p + j] = c7[static_cast<size_t>(k) * p + j];
            cc_dev = static_cast<const double*>(arena_push(c, cc.data(), cc.size() * sizeof(double)));
        }
        arena_flush(c);
        cuda_check(cudaMemsetAsync(stats, 0, sizeof(double) * 2 * nb * p, c.stream), "cc stats zero");
        if (S > 0) {
            if (fused) {
                for (int mm = 0; mm < nb; ++mm) {
                    KernelProbe kp(c, "k_node_combine_ring", 8.0 * S * (fine.size() + p + (level == 1 ? 0 : p)));
                    launch_combine_stats(S, p, fine.size(), slab + mm * S, static_cast<long long>(nb) * S, sl_dev, cf_dev,
                                         cc_dev, level == 1 ? nullptr : accs[cur] + mm * p * S, accs[nxt] + mm * p * S, S,
                                         stats + 2 * mm * p, c.stream);
                    count_launch(c);
                }
            } else {
                if (level == 1) {  // the 7-point sums this level is compared against
                    std::vector<int> cidx(static_cast<size_t>(rule->size()));
                    std::iota(cidx.begin(), cidx.end(), 0);
                    std::vector<double> c7;
                    node_coefs(*rule, cidx, p, c7);
                    const double* c7_dev = static_cast<const double*>(arena_push(c, c7.data(), c7.size() * sizeof(double)));
                    const int* s7_dev = static_cast<const int*>(arena_push(c, slot_of.data(), slot_of.size() * sizeof(int)));
                    arena_flush(c);
                    for (int mm = 0; mm < nb; ++mm) {
                        launch_combine(S, p, rule->size(), slab + mm * S, static_cast<long long>(nb) * S, s7_dev, c7_dev,
                                       accs[cur] + mm * p * S, S, 1, c.stream);
                        count_launch(c);
                    }
                }
                for (int mm = 0; mm < nb; ++mm) {
                    launch_combine(S, p, fine.size(), slab + mm * S, static_cast<long long>(nb) * S, sl_dev, cf_dev,
                                   accs[nxt] + mm * p * S, S, 1, c.stream);
                    count_launch(c);
                }
                launch_colstats(S, nb * p, accs[nxt], accs[cur], stats, c.stream);
                count_launch(c);
            }
        }
        // the statistics are max-norms: one exact all-reduce(max) gives every rank the global
        // ||y - y_prev||_inf and ||y||_inf per column (phiaction.hpp:225-239)
        allreduce_max(c, m, stats, 2 * nb * p);
        cuda_check(cudaMemcpyAsync(hstats.data(), stats, hstats.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream),
                   "cc stats readback");
        cuda_check(cudaStreamSynchronize(c.stream), "cc stats wait");
        half = half_next;
        rule = &fine;
        slot_of = std::move(fine_slot);
        cur = nxt;
        double err = 0.0;
        for (int k = 0; k < nb * p; ++k) {
            const double diff = hstats[2 * static_cast<size_t>(k)], norm = hstats[2 * static_cast<size_t>(k) + 1];
            if (diff == 0.0) continue;
            err = std::max(err, norm == 0.0 ? std::numeric_limits<double>::infinity() : diff / norm);
        }
        if (err <= eps) break;
    }
    if (accs[cur] != out && col > 0)
        cuda_check(cudaMemcpyAsync(out, accs[cur], col * sizeof(double), cudaMemcpyDeviceToDevice, c.stream), "cc copy");
    if (points_used) *points_used = rule->size();
}

// The whole distributed call: out [nb][p][S_r] (phi_1..phi_p slabs), phi0 [nb][S_r] (nullable).
void phi_dist(pq_ctx& c, pq_comm& m, const Geom& g, const DevOp& op, int nb, const double* bs, int p, int l, int n,
              int kind, double eps, double* out, double* phi0, int* points_used) {
    if (l < 0) throw std::invalid_argument("phi_with_plan: need l >= 0");
    const long long S = g.S(g.r);
    const NodesWeights& rule = kind == kGauss ? memo_rule(kGauss, n + 1) : memo_rule(kClenshaw, 25);
    // owned node slots and their thetas: Gauss slot i = node i; CC slots 0..12 = 25-rule nodes 2s,
    // slots 13..24 = 25-rule nodes 2(s - 13) + 1
    std::vector<int> all(static_cast<size_t>(rule.size()));
    std::iota(all.begin(), all.end(), 0);
    const std::vector<int> own = owned(all, g);
    std::vector<double> th;
    for (int s : own) th.push_back(kind == kGauss ? rule.x[static_cast<size_t>(s)]
                                                  : rule.x[static_cast<size_t>(s < 13 ? 2 * s : 2 * (s - 13) + 1)]);
    const PhiExps px = phi_exponentials(c, op, 1.0, l, th, l > 0, phi0 != nullptr, "dnodeE", true, false);
    mark(c, "exps");
    const size_t col = static_cast<size_t>(nb) * p * std::max<long long>(S, 1);
    // the peer transport fuses the squaring's flips into the mode products: the ping-pong columns
    // and phi_0 then live in symmetric (IPC-mapped) buffers, sized for the largest slab
    const bool fused = m.kind == PQ_COMM_PEER && peer_fused_ok(g);
    long long smax = 0;
    for (int h = 0; h < g.G; ++h) smax = std::max(smax, g.S(h));
    pq_comm::PeerBuf* pa = nullptr;
    pq_comm::PeerBuf* pb = nullptr;
    if (fused) {
        pa = &peer_buffer(c, m, "psqA", sizeof(double) * nb * p * std::max<long long>(smax, 1));
        pb = &peer_buffer(c, m, "psqB", sizeof(double) * nb * p * std::max<long long>(smax, 1));
    }
    double* t = l > 0 ? (fused ? pb->local : ws(c, "dsqT", col)) : nullptr;
    double* base_out = fused ? pa->local : out;
    double* first = (l % 2 == 1) ? t : base_out;
    if (kind == kGauss) {
        gauss_nodes(c, m, g, op, nb, bs, p, rule, px, own, first);
        if (points_used) *points_used = rule.size();
    } else {
        cc_nodes(c, m, g, op, l, nb, bs, p, eps, px, own, first, points_used);
    }
    mark(c, "nodes");
    // phi_0: one distributed Kronecker apply of expm(A) to the slabs of b (b is replicated)
    if (phi0) {
        if (fused) {
            pq_comm::PeerBuf& p0 = peer_buffer(c, m, "pphi0", sizeof(double) * nb * std::max<long long>(smax, 1));
            dist_kron_peer(c, m, g, px.phi0, px.phi0_band, bs + g.lo(g.r), op.N, nb, p0);
            cuda_check(cudaMemcpyAsync(phi0, p0.local, sizeof(double) * nb * S, cudaMemcpyDeviceToDevice, c.stream),
                       "phi_0 slab");
        } else {
            dist_kron(c, m, g, px.phi0, px.phi0_band, bs + g.lo(g.r), op.N, nb, phi0);
        }
    }
    // l modified-squaring steps on the slabs (phiaction.hpp:255-272): T = (E (x) E (x) E) y,
    // T_i <- 2^-i (T_i + sum_{j<=i} y_j/(i-j)!); E_j = expm(2^(j-l) A) from the chain
    double* res = first;
    if (l > 0) {
        std::vector<double> inv(static_cast<size_t>(p), 1.0);
        for (int k = 1; k < p; ++k) inv[static_cast<size_t>(k)] = inv[static_cast<size_t>(k) - 1] / k;
        std::vector<double> coef(static_cast<size_t>(p) * p, 0.0);
        for (int i = 0; i < p; ++i)
            for (int j = 0; j <= i; ++j)
                coef[static_cast<size_t>(i) * p + j] = std::ldexp(1.0, -(i + 1)) * inv[static_cast<size_t>(i - j)];
        const double* coef_dev = static_cast<const double*>(arena_push(c, coef.data(), coef.size() * sizeof(double)));
        arena_flush(c);
        double* cur = first;
        double* nxt = first == base_out ? t : base_out;
        for (int step = 0; step < l; ++step) {
            const double* E[3];
            const int2* B[3];
            for (int k = 0; k < op.d; ++k) {
                const long long nk = static_cast<long long>(op.n[k]) * op.n[k];
                E[k] = px.sq[k] + step * nk;
                B[k] = px.sq_band[k] ? px.sq_band[k] + step * band_row_blocks(op.n[k]) : nullptr;
            }
            if (fused)
                dist_kron_peer(c, m, g, E, B, cur, S, nb * p, nxt == pa->local ? *pa : *pb);
            else
                dist_kron(c, m, g, E, B, cur, S, nb * p, nxt);
            if (S > 0) {
                KernelProbe kp(c, "k_sq_combine2", 8.0 * S * nb * 3 * p);
                launch_sq_combine(S, p, nb, nxt, cur, coef_dev, c.stream);
                count_launch(c);
            }
            std::swap(cur, nxt);
        }
        res = cur;
    }
    if (res != out)
        cuda_check(cudaMemcpyAsync(out, res, sizeof(double) * col, cudaMemcpyDeviceToDevice, c.stream), "slab result");
    mark(c, "squaring");
}

// slabs [ncols][S_r] -> full vectors [ncols][N] on every rank
void gather_slabs(pq_ctx& c, pq_comm& m, const Geom& g, const double* slab, int ncols, double* full) {
    std::vector<Piece> sends, recvs;
    for (int col = 0; col < ncols; ++col)
        for (int h = 0; h < g.G; ++h) {
            sends.push_back({h, const_cast<double*>(slab) + col * g.S(g.r), g.S(g.r)});
            recvs.push_back({h, full + col * g.N + g.lo(h), g.S(h)});
        }
    exchange(c, m, sends, recvs);
}

void need_comm(pq_comm* m) {
    if (!m) throw std::invalid_argument("pq: null communicator");
}

long long dim_of(int d, const int* shape) {
    need(d >= 1 && d <= 3 && shape, "KroneckerSum: need one to three factors");
    long long n = 1;
    for (int k = 0; k < d; ++k) {
        need(shape[k] > 0, "KroneckerSum: factors must be square and nonempty");
        n *= shape[k];
    }
    return n;
}

// common body of the two distributed entry points
void run_dist(pq_ctx* c, pq_comm* m, int d, const int* shape, const double* factors, int nb, const double* bs,
              const pq_phi_request* req, bool plan, int p, int l, int n, int kind, double eps, double* out0, double* out,
              pq_phi_info* info, int* points_used, int space, int gather) {
    if (!c) throw std::invalid_argument("pq: null context");
    need_comm(m);
    cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
    const long long N = dim_of(d, shape);
    need(nb >= 1, "phiquadmv: need at least one right-hand side");
    const Geom g = make_geom(d, shape, m->world, m->rank);
    arena_begin(*c);
    DevOp op = upload_op(*c, d, shape, factors, "factors");
    const double* db = bs;
    if (space == PQ_HOST) {
        double* t = ws(*c, "hin_b", static_cast<size_t>(nb) * N);
        cuda_check(cudaMemcpyAsync(t, bs, sizeof(double) * nb * N, cudaMemcpyHostToDevice, c->stream), "H2D");
        db = t;
    }
    PlanInfo pi;
    if (plan) {
        pi = plan_phi(*c, op, nb, db, req->p, req->eps, req->mode, req->has_l != 0, req->l, req->c1, req->c2);
        p = req->p;
        l = pi.l;
        n = pi.n;
        kind = req->mode;
        eps = req->eps;
    }
    if (p < 1) throw std::invalid_argument(kind == kGauss ? "phi_fixed: need p >= 1" : "phi_adaptive: need p >= 1");
    const long long S = g.S(g.r);
    double* os = ws(*c, "dout", static_cast<size_t>(nb) * p * std::max<long long>(S, 1));
    double* o0 = out0 ? ws(*c, "dout0", static_cast<size_t>(nb) * std::max<long long>(S, 1)) : nullptr;
    int points = 0;
    phi_dist(*c, *m, g, op, nb, db, p, l, n, kind, eps, os, o0, &points);
    // results: slabs (gather == 0) or full vectors on every rank
    auto deliver = [&](const double* slab, int ncols, double* dst) {
        if (!dst) return;
        if (gather) {
            double* full = space == PQ_DEVICE ? dst : ws(*c, "dgather", static_cast<size_t>(ncols) * N);
            gather_slabs(*c, *m, g, slab, ncols, full);
            if (space == PQ_HOST)
                cuda_check(cudaMemcpyAsync(dst, full, sizeof(double) * ncols * N, cudaMemcpyDeviceToHost, c->stream), "D2H");
        } else {
            cuda_check(cudaMemcpyAsync(dst, slab, sizeof(double) * ncols * S,
                                       space == PQ_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream),
                       "slab out");
        }
    };
    deliver(os, nb * p, out);
    deliver(o0, nb, out0);
    if (space == PQ_HOST) cuda_check(cudaStreamSynchronize(c->stream), "sync");
    if (info) {
        info->l = l;
        info->n = n;
        info->points = points;
        info->mode = kind;
        info->planned = pi.planned;
        info->alpha = pi.alpha;
        info->beta = pi.beta;
        info->plan_cost = pi.cost;
    }
    if (points_used) *points_used = points;
}

}  // namespace

extern "C" {

int pq_nccl_unique_id(char* out128) {
    return guarded([&] {
        need(out128 != nullptr, "pq_nccl_unique_id: null output");
        ncclUniqueId id;
        nccl_check(nccl_api().getUniqueId(&id), "get unique id");
        static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(out128, id.internal, 128);
    });
}

int pq_comm_create_nccl(pq_ctx* ctx, int world, int rank, const char* id128, pq_comm** out) {
    return guarded([&] {
        need(ctx && out && id128, "pq_comm_create_nccl: null argument");
        need(world >= 1 && world <= 16 && rank >= 0 && rank < world, "pq_comm_create_nccl: bad world/rank");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        auto* m = new pq_comm();
        m->world = world;
        m->rank = rank;
        m->kind = PQ_COMM_NCCL;
        if (world > 1) {
            ncclUniqueId id;
            std::memcpy(id.internal, id128, 128);
            const ncclResult_t r = nccl_api().commInitRank(&m->nccl, world, id, rank);
            if (r != ncclSuccess) {
                delete m;
                nccl_check(r, "comm init");
            }
        }
        *out = m;
    });
}

int pq_comm_create_host(int world, int rank, const pq_host_transport* t, pq_comm** out) {
    return guarded([&] {
        need(out != nullptr, "pq_comm_create_host: null output");
        need(world >= 1 && world <= 16 && rank >= 0 && rank < world, "pq_comm_create_host: bad world/rank");
        need(world == 1 || (t && t->alltoallv && t->allreduce_max), "pq_comm_create_host: transport callbacks missing");
        auto* m = new pq_comm();
        m->world = world;
        m->rank = rank;
        m->kind = PQ_COMM_HOST;
        if (t) m->host = *t;
        *out = m;
    });
}

int pq_comm_create_peer(pq_ctx* ctx, int world, int rank, const pq_host_transport* t, pq_comm** out) {
    return guarded([&] {
        need(ctx && out, "pq_comm_create_peer: null argument");
        need(world >= 1 && world <= 16 && rank >= 0 && rank < world, "pq_comm_create_peer: bad world/rank");
        need(world == 1 || (t && t->alltoallv && t->allreduce_max), "pq_comm_create_peer: transport callbacks missing");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        auto* m = new pq_comm();
        m->world = world;
        m->rank = rank;
        m->kind = PQ_COMM_PEER;
        if (t) m->host = *t;
        *out = m;
    });
}

int pq_comm_destroy(pq_comm* m) {
    return guarded([&] {
        if (!m) return;
        for (auto& kv : m->pbufs) {
            for (int h = 0; h < m->world; ++h)
                if (h != m->rank && h < static_cast<int>(kv.second.peer.size()) && kv.second.peer[static_cast<size_t>(h)])
                    cudaIpcCloseMemHandle(kv.second.peer[static_cast<size_t>(h)]);
            if (kv.second.local) cudaFree(kv.second.local);
        }
        if (m->nccl) nccl_api().commDestroy(m->nccl);
        if (m->hs) cudaFreeHost(m->hs);
        if (m->hr) cudaFreeHost(m->hr);
        delete m;
    });
}

int pq_comm_stats(pq_comm* m, int reset, double* bytes_sent, uint64_t* exchanges) {
    return guarded([&] {
        need_comm(m);
        if (bytes_sent) *bytes_sent = m->bytes_sent;
        if (exchanges) *exchanges = m->exchanges;
        if (reset) {
            m->bytes_sent = 0.0;
            m->exchanges = 0;
        }
    });
}

int pq_dist_slab(int d, const int* shape, int world, int rank, int64_t* begin, int64_t* end) {
    return guarded([&] {
        dim_of(d, shape);
        const Geom g = make_geom(d, shape, world, rank);
        if (begin) *begin = g.lo(rank);
        if (end) *end = g.lo(rank) + g.S(rank);
    });
}

int pq_phiquadmv_dist(pq_ctx* ctx, pq_comm* comm, int d, const int* shape, const double* factors, int nb,
                      const double* bs, const pq_phi_request* req, double* out0, double* out, pq_phi_info* info,
                      int space, int gather) {
    return guarded([&] {
        NvtxRange nvtx("pq_phiquadmv_dist");
        need(req != nullptr, "phiquadmv: null request");
        need(req->p >= 1, "phiquadmv: need p >= 1");
        need(req->mode == PQ_GAUSS_LEGENDRE || req->mode == PQ_CLENSHAW_CURTIS, "QuadKind: unknown rule");
        run_dist(ctx, comm, d, shape, factors, nb, bs, req, true, 0, 0, 0, 0, 0.0, out0, out, info, nullptr, space,
                 gather);
    });
}

int pq_phi_with_plan_dist(pq_ctx* ctx, pq_comm* comm, int d, const int* shape, const double* factors, int nb,
                          const double* bs, int p, int l, int n, int kind, double eps, double* out, int* points_used,
                          int space, int gather) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_with_plan_dist");
        need(l >= 0, "phi_with_plan: need l >= 0");
        need(kind == PQ_GAUSS_LEGENDRE || kind == PQ_CLENSHAW_CURTIS, "QuadKind: unknown rule");
        if (kind == PQ_GAUSS_LEGENDRE) need(n + 1 >= 1, "gauss_legendre: need at least one point");
        need(p >= 1, kind == PQ_GAUSS_LEGENDRE ? "phi_fixed: need p >= 1" : "phi_adaptive: need p >= 1");
        run_dist(ctx, comm, d, shape, factors, nb, bs, nullptr, false, p, l, n, kind, eps, nullptr, out, nullptr,
                 points_used, space, gather);
    });
}

}  // extern "C"
