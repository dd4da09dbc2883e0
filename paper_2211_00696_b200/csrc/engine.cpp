// The phi pipeline on the device (reference: phiaction.hpp, kron.hpp, integrators.hpp).
//
// Data layout in HBM (N = prod n_k doubles per vector, vec order):
//   factors      d blocks n_k x n_k, uploaded once per call
//   node E       per dim k: q blocks n_k x n_k (expm((1-theta_i) 2^-l A_k)), contiguous
//   chainA/B     Qc*N mode-product intermediates (Qc = node chunk fitting the workspace budget)
//   nodeV        Qc*N node vectors v_i = (E_i0 (x) E_i1 (x) E_i2) b, consumed by the combine
//   out / sqT    nb*p*N phi columns, ping-pong through the l squaring steps
//   ccpool       adaptive CC: every node vector of the current ladder rule (reused next level)
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>

namespace pqb {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ context helpers ------

static size_t budget_bytes(pq_ctx& c) {
    if (c.ws_limit == 0) {
        size_t fr = 0, tot = 0;
        cuda_check(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
        size_t held = 0;
        for (auto& kv : c.bufs) held += kv.second.bytes;
        c.ws_limit = static_cast<uint64_t>(0.85 * static_cast<double>(fr + held));
    }
    return static_cast<size_t>(c.ws_limit);
}

// Workspace memory comes from a per-device stream-ordered pool that keeps what it holds
// (release threshold = max): after the first calls at a size no allocation reaches the driver,
// and retired buffers return to the pool with cudaFreeAsync at the next call's start.  Plain
// cudaMalloc / cudaFree inside a call cost 10-100 ms on the B200 in the acceptance gate's
// criterion 7 (PQ_SLOWLOG timelines, profiles/r02_summary.md).
static cudaMemPool_t device_pool(int dev) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> hold(mu);
    auto it = pools.find(dev);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    cuda_check(cudaMemPoolCreate(&p, &props), "cudaMemPoolCreate");
    uint64_t keep = ~uint64_t(0);
    cuda_check(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep), "pool threshold");
    pools[dev] = p;
    return p;
}

void trim_pool(pq_ctx& c) { cudaMemPoolTrimTo(device_pool(c.device), 0); }

static bool ws_guard_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PQ_WS_GUARD");
        return v && v[0] == '1';
    }();
    return on;
}
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kCanary = 0xA7;

void* ws_alloc(pq_ctx& c, size_t bytes, const std::string& name) {
    if (!ws_guard_enabled()) return dev_alloc(c, bytes, name.c_str());
    const size_t body = (bytes + 255) & ~size_t(255);
    char* base = static_cast<char*>(dev_alloc(c, body + 2 * kGuardBytes, name.c_str()));
    cuda_check(cudaMemsetAsync(base, kCanary, kGuardBytes, c.stream), "guard fill");
    cuda_check(cudaMemsetAsync(base + kGuardBytes + bytes, kCanary, body - bytes + kGuardBytes, c.stream), "guard fill");
    void* p = base + kGuardBytes;
    c.guards[p] = {base, bytes, name};
    return p;
}

static void* base_of(pq_ctx& c, void* p) {
    auto it = c.guards.find(p);
    if (it == c.guards.end()) return p;
    void* b = it->second.base;
    c.guards.erase(it);
    return b;
}

void ws_retire(pq_ctx& c, void* p) {
    if (p) c.graveyard.push_back(base_of(c, p));
}

void ws_free_now(pq_ctx& c, void* p) {
    if (p) cudaFree(base_of(c, p));
}

int check_guards(pq_ctx& c, std::string* what) {
    cuda_check(cudaDeviceSynchronize(), "guard check sync");
    int bad = 0;
    std::vector<unsigned char> h(kGuardBytes + 256);
    for (const auto& kv : c.guards) {
        const char* base = static_cast<const char*>(kv.second.base);
        const size_t bytes = kv.second.bytes, body = (bytes + 255) & ~size_t(255);
        bool ok = true;
        cuda_check(cudaMemcpy(h.data(), base, kGuardBytes, cudaMemcpyDeviceToHost), "guard read");
        for (size_t i = 0; i < kGuardBytes; ++i) ok = ok && h[i] == kCanary;
        const size_t tail = body - bytes + kGuardBytes;
        std::vector<unsigned char> t(tail);
        cuda_check(cudaMemcpy(t.data(), base + kGuardBytes + bytes, tail, cudaMemcpyDeviceToHost), "guard read");
        for (size_t i = 0; i < tail; ++i) ok = ok && t[i] == kCanary;
        if (!ok) {
            ++bad;
            if (what) *what += kv.second.name + " ";
        }
    }
    return bad;
}

void free_graveyard(pq_ctx& c) {
    if (c.graveyard.empty()) return;
    cuda_check(cudaDeviceSynchronize(), "sync before workspace free");
    for (void* p : c.graveyard) cudaFree(p);
    c.graveyard.clear();
}

// retired buffers back to the pool, stream-ordered after everything this context enqueued so far
// (every call joins its helper streams into c.stream before returning)
void recycle_graveyard(pq_ctx& c) {
    for (void* p : c.graveyard) cuda_check(cudaFreeAsync(p, c.stream), "cudaFreeAsync(workspace)");
    c.graveyard.clear();
}

void* dev_alloc(pq_ctx& c, size_t bytes, const char* what) {
    void* p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, device_pool(c.device), c.stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        free_graveyard(c);
        trim_pool(c);
        e = cudaMallocFromPoolAsync(&p, bytes, device_pool(c.device), c.stream);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw CudaError(std::string("device workspace '") + what + "': cannot allocate " + std::to_string(bytes >> 20) +
                        " MiB");
    }
    return p;
}

void* ws_bytes(pq_ctx& c, const std::string& name, size_t bytes) {
    DevBuf& b = c.bufs[name];
    if (b.bytes >= bytes && b.p) return b.p;
    // the old buffer may still be read by enqueued work: retire it (pq_ctx::graveyard)
    ws_retire(c, b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t want = std::max<size_t>(bytes, 256);
    mark(c, ("ws_grow:" + name).c_str());
    b.p = ws_alloc(c, want, name);
    b.bytes = want;
    return b.p;
}

double* ws(pq_ctx& c, const std::string& name, size_t count) {
    return static_cast<double*>(ws_bytes(c, name, count * sizeof(double)));
}

void arena_begin(pq_ctx& c) {
    c.deferred.clear();  // never carry side-stream work from an earlier (failed) call
    recycle_graveyard(c);
    ParamArena& a = c.arena;
    if (!a.host) {
        a.cap = size_t(8) << 20;
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&a.host), a.cap, cudaHostAllocMapped | cudaHostAllocPortable),
                   "cudaHostAlloc(arena)");
        cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&a.host_d), a.host, 0), "arena device view");
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&a.dev), a.cap), "cudaMalloc(arena)");
        cuda_check(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming), "event(arena)");
        cuda_check(cudaEventRecord(a.done, c.stream), "record(arena)");
    }
    // the previous call's uploads must have left the pinned buffer before we overwrite it
    cuda_check(cudaEventSynchronize(a.done), "arena wait");
    a.used = a.flushed = 0;
}

const void* arena_push(pq_ctx& c, const void* data, size_t bytes) {
    ParamArena& a = c.arena;
    const size_t off = (a.used + 15) & ~size_t(15);
    if (off + bytes > a.cap) {
        if (bytes > a.cap) throw std::invalid_argument("parameter table larger than the 8 MB staging arena");
        // wrap around: every table pushed so far may still be read by enqueued work on any of the
        // context's streams (and by deferred side-stream work not yet enqueued), so enqueue that,
        // let all of it finish, then rewind
        arena_flush(c);
        run_deferred(c);
        cuda_check(cudaStreamSynchronize(c.stream), "arena wrap");
        if (c.side) cuda_check(cudaStreamSynchronize(c.side), "arena wrap");
        if (c.sq2) cuda_check(cudaStreamSynchronize(c.sq2), "arena wrap");
        a.used = a.flushed = 0;
        return arena_push(c, data, bytes);
    }
    std::memcpy(a.host + off, data, bytes);
    a.used = off + bytes;
    return a.dev + off;
}

void arena_flush(pq_ctx& c) {
    ParamArena& a = c.arena;
    if (a.used > a.flushed) {
        // up to 256 KB: SM loads from the mapped staging buffer (the H2D engine may be busy with
        // another call's right-hand sides for 0.3 ms); the 16-byte rounding only rewrites bytes
        // with their current staged values or bytes not handed out yet (cap is 16-byte aligned)
        const size_t lo = a.flushed & ~size_t(15), hi = (a.used + 15) & ~size_t(15);
        if (hi - lo <= (256u << 10) && hi <= a.cap) {
            launch_copy_vec4(a.host_d + lo, a.dev + lo, (hi - lo) / 16, c.stream);
            count_launch(c);
        } else {
            cuda_check(cudaMemcpyAsync(a.dev + a.flushed, a.host + a.flushed, a.used - a.flushed, cudaMemcpyHostToDevice,
                                       c.stream),
                       "arena upload");
        }
        a.flushed = a.used;
        cuda_check(cudaEventRecord(a.done, c.stream), "record(arena)");
    }
}

// device-to-device copy of `count` doubles: on the SMs when small and 16-byte aligned (matrix-sized
// copies would otherwise queue on a copy engine behind MB-sized transfers), else cudaMemcpyAsync
void dev_copy(pq_ctx& c, double* dst, const double* src, size_t count, cudaStream_t s) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
    if (aligned && count % 2 == 0 && count * sizeof(double) <= (4u << 20)) {
        launch_copy_vec4(src, dst, count / 2, s);
        count_launch(c);
        return;
    }
    cuda_check(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToDevice, s), "device copy");
}

// Every launch site counts its kernels here, so launch-configuration errors surface at the launch
// that caused them (cudaGetLastError is a host-side query, no synchronisation).
void count_launch(pq_ctx& c, int n) {
    c.launches += static_cast<uint64_t>(n);
    cuda_check(cudaGetLastError(), "kernel launch");
}

static cudaEvent_t prof_event(pq_ctx& c) {
    if (c.ev_used == c.ev_pool.size()) {
        cudaEvent_t e;
        cuda_check(cudaEventCreate(&e), "event create");
        c.ev_pool.push_back(e);
    }
    return c.ev_pool[c.ev_used++];
}

int gemm(pq_ctx& c, const GemmArgs& g) {
    if (!c.profiling) {
        const int k = launch_gemm(g, c.stream);
        count_launch(c, k);
        return k;
    }
    if (c.ev_used + 2 > 4096) prof_collect(c);
    if (!c.d_flops) cuda_check(cudaMalloc(&c.d_flops, sizeof(unsigned long long) * 2048), "flop counters");
    const size_t slot = c.ev_used / 2;
    if (slot == 0)
        cuda_check(cudaMemsetAsync(c.d_flops, 0, sizeof(unsigned long long) * 2048, c.stream), "flop counters zero");
    GemmArgs gp = g;
    gp.flop_counter = c.d_flops + slot;
    cudaEvent_t a = prof_event(c), b = prof_event(c);
    cuda_check(cudaEventRecord(a, c.stream), "event record");
    const int k = launch_gemm(gp, c.stream);
    cuda_check(cudaEventRecord(b, c.stream), "event record");
    count_launch(c, k);
    c.ev_flops.push_back(2.0 * g.M * static_cast<double>(g.N) * g.K * g.Z);
    char key[160];
    std::snprintf(key, sizeof key, "%s M%d N%d K%d Z%d %s%s", g.tag ? g.tag : "?", g.M, g.N, g.K, g.Z,
                  g.b_kmajor ? "kk" : "nk", g.band ? " band" : "");
    c.ev_keys.push_back(key);
    c.prof_launches += static_cast<uint64_t>(k);
    return k;
}

// Fused mode-1+2 launch (slab12.cu), profiled like gemm(): one event pair, executed-flop counter,
// dense-equivalent flops of the two mode products it replaces.
int slab12(pq_ctx& c, const Slab12Args& g, const char* tag) {
    if (!c.profiling) {
        const int k = launch_slab12(g, c.stream);
        count_launch(c, k);
        return k;
    }
    if (c.ev_used + 2 > 4096) prof_collect(c);
    if (!c.d_flops) cuda_check(cudaMalloc(&c.d_flops, sizeof(unsigned long long) * 2048), "flop counters");
    const size_t slot = c.ev_used / 2;
    if (slot == 0)
        cuda_check(cudaMemsetAsync(c.d_flops, 0, sizeof(unsigned long long) * 2048, c.stream), "flop counters zero");
    Slab12Args gp = g;
    gp.flop_counter = c.d_flops + slot;
    cudaEvent_t a = prof_event(c), b = prof_event(c);
    cuda_check(cudaEventRecord(a, c.stream), "event record");
    const int k = launch_slab12(gp, c.stream);
    cuda_check(cudaEventRecord(b, c.stream), "event record");
    count_launch(c, k);
    const double slabs = static_cast<double>(g.n0) * g.Z1;
    c.ev_flops.push_back(2.0 * 2.0 * 128.0 * 128.0 * 128.0 * slabs);
    char key[160];
    std::snprintf(key, sizeof key, "%s M128 N128 K128 Z%lld slab12%s", tag ? tag : "?",
                  static_cast<long long>(g.n0) * g.Z1, g.band1 || g.band2 ? " band" : "");
    c.ev_keys.push_back(key);
    c.prof_launches += static_cast<uint64_t>(k);
    return k;
}

// PQ_SLAB12=0 runs modes 1 and 2 of 3-D applies as two band-tile launches (A/B switch; the fused
// kernel is bitwise the same)
static bool slab12_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PQ_SLAB12");
        return !(v && v[0] == '0');
    }();
    return on;
}

constexpr int kMaxChainLevels = 12;  // kernels.hpp launch_gemm_chain (gemm.cuh kMaxChain)

// PQ_GEMM_CHAIN=1: chained cooperative launches for the Taylor powers and the expm squaring
// rounds.  Measured (profiles/r02_summary.md): the Taylor chain is as slow as its 5 launches
// (55 vs 56 us: each level is bound by one tile's dependent K loop, not by launch gaps), the
// squaring chain saves 20 us, but the cooperative grid occupies every SM and blocks the side
// stream's overlap: 462 vs 471 actions/s at config 2.  Off by default.
static bool chain_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PQ_GEMM_CHAIN");
        return v && v[0] == '1';
    }();
    return on;
}

// Dependent levels of small batched products in one cooperative launch (launch_gemm_chain);
// per-level launches when the chain does not qualify or PQ_GEMM_CHAIN=0.
int gemm_chain(pq_ctx& c, std::vector<GemmArgs> levels, const char* tag) {
    if (levels.empty()) return 0;
    for (auto& g : levels) g.tag = tag;
    if (!chain_enabled() || levels.size() == 1) {
        int k = 0;
        for (const auto& g : levels) k += gemm(c, g);
        return k;
    }
    unsigned* bar = static_cast<unsigned*>(ws_bytes(c, "chain_bar", 256));
    cudaEvent_t a = nullptr, b = nullptr;
    size_t slot = 0;
    if (c.profiling) {
        if (c.ev_used + 2 > 4096) prof_collect(c);
        if (!c.d_flops) cuda_check(cudaMalloc(&c.d_flops, sizeof(unsigned long long) * 2048), "flop counters");
        slot = c.ev_used / 2;
        if (slot == 0)
            cuda_check(cudaMemsetAsync(c.d_flops, 0, sizeof(unsigned long long) * 2048, c.stream), "flop counters zero");
        for (auto& g : levels) g.flop_counter = c.d_flops + slot;
        a = prof_event(c);
        b = prof_event(c);
        cuda_check(cudaEventRecord(a, c.stream), "event record");
    }
    const int k = launch_gemm_chain(levels.data(), static_cast<int>(levels.size()), bar, c.stream);
    if (k == 0) {  // not eligible: one launch per level (undo the profiling slot)
        if (c.profiling) c.ev_used -= 2;
        int n = 0;
        for (auto& g : levels) {
            g.flop_counter = nullptr;
            n += gemm(c, g);
        }
        return n;
    }
    count_launch(c, k);
    if (c.profiling) {
        cuda_check(cudaEventRecord(b, c.stream), "event record");
        double dense = 0.0;
        for (const auto& g : levels) dense += 2.0 * g.M * static_cast<double>(g.N) * g.K * g.Z;
        c.ev_flops.push_back(dense);
        char key[160];
        std::snprintf(key, sizeof key, "%s chain of %zu levels M%d N%d K%d", tag, levels.size(), levels[0].M,
                      levels[0].N, levels[0].K);
        c.ev_keys.push_back(key);
        c.prof_launches += static_cast<uint64_t>(k);
    }
    return k;
}

KernelProbe::KernelProbe(pq_ctx& ctx, const char* t, double b) : c(ctx), tag(t), bytes(b) {
    if (!c.profiling) return;
    s = c.stream;
    cuda_check(cudaEventCreate(&a), "probe event");
    cuda_check(cudaEventRecord(a, s), "probe record");
}

KernelProbe::~KernelProbe() {
    if (!a) return;
    cudaEvent_t b = nullptr;
    if (cudaEventCreate(&b) != cudaSuccess || cudaEventRecord(b, s) != cudaSuccess) {
        cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
        return;
    }
    c.krecs.push_back({tag, a, b, bytes});
}

static void kstats_collect(pq_ctx& c) {
    if (c.krecs.empty()) return;
    cuda_check(cudaDeviceSynchronize(), "probe sync");  // probes may sit on side streams
    for (const auto& r : c.krecs) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, r.a, r.b), "probe elapsed");
        auto& st = c.kstats[r.tag];
        st.launches += 1;
        st.ms += ms;
        st.bytes += r.bytes;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    c.krecs.clear();
}

void prof_collect(pq_ctx& c) {
    kstats_collect(c);
    if (c.ev_used == 0) return;
    cuda_check(cudaStreamSynchronize(c.stream), "prof sync");
    std::vector<unsigned long long> executed(c.ev_used / 2);
    cuda_check(cudaMemcpy(executed.data(), c.d_flops, sizeof(unsigned long long) * executed.size(),
                          cudaMemcpyDeviceToHost),
               "flop counters readback");
    for (size_t i = 0; i + 1 < c.ev_used; i += 2) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, c.ev_pool[i], c.ev_pool[i + 1]), "event elapsed");
        c.prof_ms += ms;
        c.prof_flops += static_cast<double>(executed[i / 2]);
        c.prof_flops_dense += c.ev_flops[i / 2];
        auto& gs = c.gstats[c.ev_keys[i / 2]];
        gs.launches += 1;
        gs.ms += ms;
        gs.flops += static_cast<double>(executed[i / 2]);
        gs.dense += c.ev_flops[i / 2];
    }
    c.ev_used = 0;
    c.ev_flops.clear();
    c.ev_keys.clear();
}

namespace {
// per device: the compute-done events of the call that last held the gate
struct ComputeGate {
    std::mutex mu;
    const pq_ctx* owner = nullptr;
    std::vector<cudaEvent_t> done;
};
ComputeGate& device_gate(int dev) {
    static ComputeGate gates[64];
    return gates[static_cast<unsigned>(dev) % 64];
}
}  // namespace

// The compute gate orders concurrent host-buffer calls' compute so one call's result D2H runs
// under the next call's compute.  Default: on for results of 512 MB and more per call -- where the
// D2H is a large share of the call (config 3: 4.3 GB per call, e2e 77.1 -> 86.6 RHS/s; config 5:
// 6.4 GB, 3.01 -> 3.57 actions/s) -- and off below (config 2, 84 MB: 386-388 gated vs 407-421
// ungated with 4 callers, the serialised compute losing the overlap of one call's low-occupancy
// phases with another's).  PQ_COMPUTE_GATE=1 gates every call of 8 MB and more, =0 none.
bool gate_wanted(size_t result_bytes) {
    static const int mode = [] {
        const char* e = std::getenv("PQ_COMPUTE_GATE");
        return e ? (std::atoi(e) != 0 ? 1 : 0) : -1;
    }();
    if (mode == 1) return result_bytes >= (size_t(8) << 20);
    if (mode == 0) return false;
    return result_bytes >= (size_t(512) << 20);
}

void gate_acquire(pq_ctx& c) {
    ComputeGate& g = device_gate(c.device);
    g.mu.lock();  // held until gate_enqueued: the next caller chains behind this call's events
    for (cudaEvent_t e : g.done) cuda_check(cudaStreamWaitEvent(c.stream, e, 0), "gate wait");
    c.gate_held = true;
    c.gate_covered = false;
    c.gate_used = 0;
}

void gate_point(pq_ctx& c, cudaStream_t s) {
    if (!c.gate_held) return;
    if (c.gate_ev.size() <= c.gate_used) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "gate event");
        c.gate_ev.push_back(e);
    }
    cuda_check(cudaEventRecord(c.gate_ev[c.gate_used++], s), "gate record");
}

void gate_enqueued(pq_ctx& c) {
    if (!c.gate_held) return;
    ComputeGate& g = device_gate(c.device);
    try {
        if (!c.gate_covered) gate_point(c, c.stream);
        g.done.assign(c.gate_ev.begin(), c.gate_ev.begin() + static_cast<long>(c.gate_used));
        g.owner = &c;
    } catch (...) {
        g.done.clear();
        g.owner = nullptr;
    }
    c.gate_held = false;
    g.mu.unlock();
}

void gate_forget(pq_ctx& c) {
    ComputeGate& g = device_gate(c.device);
    std::lock_guard<std::mutex> lk(g.mu);
    if (g.owner == &c) {
        g.done.clear();
        g.owner = nullptr;
    }
    for (cudaEvent_t e : c.gate_ev) cudaEventDestroy(e);
    c.gate_ev.clear();
}

void note_early_copy(pq_ctx& c, cudaStream_t s, double* host, size_t count) {
    const size_t i = c.early.size();
    if (c.ev_early.size() <= i) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "early copy event");
        c.ev_early.push_back(e);
    }
    cuda_check(cudaEventRecord(c.ev_early[i], s), "early copy record");
    c.early.push_back({c.ev_early[i], host, count});
}

void mark(pq_ctx& c, const char* name) {
    nvtxMarkA(name);
    if (!c.profiling && !c.trace) return;
    static const auto t0 = std::chrono::steady_clock::now();
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "mark event");
    cuda_check(cudaEventRecord(e, c.stream), "mark record");
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    c.marks.push_back({name, e, us});
}

void check_launch(pq_ctx& c) {
    (void)c;
    cuda_check(cudaGetLastError(), "kernel launch");
}

// ------------------------------------------------------------------ operator upload ------

DevOp upload_op(pq_ctx& c, int d, const int* shape, const double* factors, const std::string& slot) {
    if (d < 1 || d > 3) throw std::invalid_argument("KroneckerSum: need one to three factors");
    DevOp op;
    op.d = d;
    size_t total = 0;
    for (int k = 0; k < d; ++k) {
        if (shape[k] <= 0) throw std::invalid_argument("KroneckerSum: factors must be square and nonempty");
        op.n[k] = shape[k];
        op.N *= shape[k];
        total += static_cast<size_t>(shape[k]) * shape[k];
    }
    double* dev = ws(c, slot, total);
    pq_ctx::FacCache& fc = c.fac_cache[slot];
    bool same = fc.host && fc.d == d && fc.dev == dev && fc.host->size() == total &&
                std::memcmp(fc.host->data(), factors, total * sizeof(double)) == 0;
    for (int k = 0; k < d && same; ++k) same = fc.n[k] == shape[k];
    if (!same) {
        auto host = std::make_shared<std::vector<double>>(factors, factors + total);
        for (double v : *host)
            if (!std::isfinite(v)) throw std::invalid_argument("DenseMatrix: non-finite entry");
        // stage through pinned memory so the copy is asynchronous (a pageable H2D copy would wait
        // for the stream to drain, idling the GPU while the host prepares the call)
        if (!c.ev_fac) cuda_check(cudaEventCreateWithFlags(&c.ev_fac, cudaEventDisableTiming), "factor event");
        cuda_check(cudaEventSynchronize(c.ev_fac), "factor staging wait");
        if (c.pin_fac_cap < total) {
            if (c.pin_fac) cudaFreeHost(c.pin_fac);
            cuda_check(cudaMallocHost(reinterpret_cast<void**>(&c.pin_fac), total * sizeof(double)), "pinned factors");
            c.pin_fac_cap = total;
        }
        std::memcpy(c.pin_fac, factors, total * sizeof(double));
        cuda_check(cudaMemcpyAsync(dev, c.pin_fac, total * sizeof(double), cudaMemcpyHostToDevice, c.stream),
                   "upload factors");
        cuda_check(cudaEventRecord(c.ev_fac, c.stream), "factor record");
        // dense.hpp:122-141 (host copies; the planner's alpha uses the inf-norms)
        size_t off = 0;
        size_t offs[3] = {0, 0, 0};
        for (int k = 0; k < d; ++k) {
            const int n = shape[k];
            offs[k] = off;
            const double* f = host->data() + off;
            std::vector<double> col(static_cast<size_t>(n), 0.0);
            double best_row = 0.0;
            for (int i = 0; i < n; ++i) {
                double rs = 0.0;
                for (int j = 0; j < n; ++j) {
                    const double a = std::abs(f[static_cast<size_t>(i) * n + j]);
                    rs += a;
                    col[static_cast<size_t>(j)] += a;
                }
                if (rs > best_row) best_row = rs;
            }
            fc.inf_norm[k] = best_row;
            fc.one_norm[k] = *std::max_element(col.begin(), col.end());
            off += static_cast<size_t>(n) * n;
        }
        // bit-identical factors (the isotropic Laplacians of configs 1, 3, 4, 5) are exponentiated once
        for (int k = 0; k < d; ++k) {
            fc.canon[k] = k;
            for (int j = 0; j < k; ++j)
                if (fc.canon[j] == j && shape[j] == shape[k] &&
                    std::memcmp(host->data() + offs[j], host->data() + offs[k],
                                sizeof(double) * shape[k] * shape[k]) == 0) {
                    fc.canon[k] = j;
                    break;
                }
        }
        fc.d = d;
        for (int k = 0; k < 3; ++k) fc.n[k] = k < d ? shape[k] : 0;
        fc.host = host;
        fc.dev = dev;
    }
    op.host = fc.host;
    op.serial = ++c.op_serial;
    size_t off = 0;
    for (int k = 0; k < d; ++k) {
        op.F[k] = dev + off;
        op.inf_norm[k] = fc.inf_norm[k];
        op.one_norm[k] = fc.one_norm[k];
        op.canon[k] = fc.canon[k];
        off += static_cast<size_t>(op.n[k]) * op.n[k];
    }
    return op;
}


// ------------------------------------------------------------------ batched expm ---------

static constexpr double kTheta13 = 5.371920351148152;

// Upper bound of the expm squaring count for ||scale * A||_1 (device norms round differently).
static int squaring_bound(double abs_scale, double one_norm) {
    const double b = abs_scale * one_norm * (1.0 + 1e-10);
    if (!(b > kTheta13)) return 0;
    return static_cast<int>(std::ceil(std::log2(b / kTheta13)));
}

static GemmArgs square_batch(int n, int count, const double* A, const double* B, double* C) {
    GemmArgs g;
    g.A = A;
    g.B = B;
    g.C = C;
    g.M = g.N = g.K = n;
    g.lda = g.ldb = g.ldc = n;
    g.Z = count;
    g.sA1 = g.sB1 = g.sC1 = static_cast<long long>(n) * n;
    return g;
}

static void squaring_rounds(pq_ctx& c, int n, int count, const std::vector<int>& hint, const int* s_dev, int s_max,
                            double* cur, double* other, double* out);

// Negligible-block tables for the exponentials of a phi call (kernels.hpp launch_band_ranges);
// only the band mode-product tiles (vec2 paths of the 64x64 family) read them, so they are built
// for n >= 64.  PQ_BAND=0
// disables the skip (every mode product then runs its full K).
static bool band_enabled(int n, long long N) {
    static const bool disabled = [] {
        const char* v = std::getenv("PQ_BAND");
        return v && v[0] == '0';
    }();
    // tiny operators are launch-latency bound: the table launches would cost more than they save
    // (config 1, N = 4096: 4568 actions/s without, 3665 with)
    return !disabled && n >= 64 && n <= 512 && N >= (1LL << 18);
}
// Fragment-major copies of an exponential batch for k_slab12's phase 2 (PQ_E2PACK=0 disables: the
// kernel then reads E2 row-major).  Written by the same k_band_ranges launch as the batch's band
// table and found again from the table pointer, so they follow the tables through every call path.
static bool e2pack_enabled(int n) {
    static const bool on = [] {
        const char* v = std::getenv("PQ_E2PACK");
        return !(v && v[0] == '0');
    }();
    return on && slab12_enabled() && slab12_supported(n, n);
}
static void band_pack_register(pq_ctx& c, const int2* band, size_t matrices, double* pack, int n) {
    const size_t recs = matrices * static_cast<size_t>(band_row_blocks(n));
    auto& v = c.band_packs;
    v.erase(std::remove_if(v.begin(), v.end(),
                           [&](const pq_ctx::BandPack& e) { return e.lo < band + recs && band < e.lo + e.recs; }),
            v.end());
    if (pack) v.push_back({band, recs, pack, n});  // pack == null: only forget what overlapped
}
// pack of the matrix whose band record starts at `band` (null: none); *stride_per_matrix = doubles
static double* band_pack_find(const pq_ctx& c, const int2* band, int n, long long* per_matrix = nullptr) {
    if (!band) return nullptr;
    for (const auto& e : c.band_packs)
        if (e.n == n && band >= e.lo && band < e.lo + e.recs) {
            const long long pd = band_pack_doubles(n);
            if (per_matrix) *per_matrix = pd;
            return e.pack + static_cast<long long>((band - e.lo) / band_row_blocks(n)) * pd;
        }
    return nullptr;
}
static void band_ranges(pq_ctx& c, int n, int count, const double* E, int2* band) {
    if (!band || count <= 0) return;
    launch_band_ranges(n, count, E, band, c.stream, band_pack_find(c, band, n));
    count_launch(c);
}

// Two-stream squaring (squaring_pingpong): one RHS, p >= 2, vectors large enough that a step's
// GEMMs outweigh the per-step event traffic (config 1, N = 4096: 4330 actions/s without the
// split, 3368 with it), not while profiling (per-launch events must stay unambiguous);
// PQ_SQ_SPLIT=0 disables it.
static bool squaring_split_ok(const pq_ctx& c, int nb, int p, long long N) {
    static const bool disabled = [] {
        const char* v = std::getenv("PQ_SQ_SPLIT");
        return v && v[0] == '0';
    }();
    return !disabled && nb == 1 && p >= 2 && N >= (1LL << 18) && !c.profiling;
}

// helper streams inherit the priority of the context's stream, so a caller that runs its
// context on a high-priority stream (bench.py's overlapped end-to-end leg) keeps it end to end
void make_helper_stream(pq_ctx& c, cudaStream_t* s, const char* what) {
    int prio = 0;
    if (cudaStreamGetPriority(c.stream, &prio) != cudaSuccess) {
        cudaGetLastError();
        prio = 0;
    }
    cuda_check(cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, prio), what);
}

// Rotating buffers of the two-stream squaring.  Three suffice for the data dependencies; when the
// results go to pinned host memory the lower half gets l + 1 (no reuse, so it never waits for the
// upper half and finishes -- and starts its D2H -- while the upper half still computes), as long
// as the extra buffers stay under 2 GB (config 2: 5 x 67 MB).
static int squaring_ring(int nb, int p, long long N, int l, bool host_out) {
    const int R = std::max(3, l + 1);
    if (!host_out || R == 3) return 3;
    const double extra = static_cast<double>(R - 3) * nb * p * static_cast<double>(N) * sizeof(double);
    return extra <= 2.0e9 ? R : 3;
}

// helper streams of the per-column squaring cascade: descending priority from the top of the
// device's range down to the context stream's own level (equal where the range runs out)
static void ensure_sq_cascade(pq_ctx& c, int G) {
    if (static_cast<int>(c.sqs.size()) >= G) return;
    int prio = 0, least = 0, greatest = 0;
    if (cudaStreamGetPriority(c.stream, &prio) != cudaSuccess) {
        cudaGetLastError();
        prio = 0;
    }
    cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
    while (static_cast<int>(c.sqs.size()) < G) {
        const int g = static_cast<int>(c.sqs.size());
        cudaStream_t s;
        cuda_check(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, std::max(greatest, prio - (G - 1 - g))),
                   "sq cascade stream");
        c.sqs.push_back(s);
    }
}

// second squaring stream and its fork event
static void ensure_sq2(pq_ctx& c) {
    if (!c.sq2) {
        make_helper_stream(c, &c.sq2, "sq2 stream");
        if (!c.ev_sqfork) cuda_check(cudaEventCreateWithFlags(&c.ev_sqfork, cudaEventDisableTiming), "sq fork event");
    }
}

static void ensure_ccs(pq_ctx& c) {
    if (c.ccs) return;
    int prio = 0, least = 0, greatest = 0;
    if (cudaStreamGetPriority(c.stream, &prio) != cudaSuccess || cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) {
        cudaGetLastError();
        prio = greatest = 0;
    }
    cuda_check(cudaStreamCreateWithPriority(&c.ccs, cudaStreamNonBlocking, std::max(greatest, prio - 1)), "cc stream");
    if (!c.ev_ccfork) cuda_check(cudaEventCreateWithFlags(&c.ev_ccfork, cudaEventDisableTiming), "cc fork event");
}

// PQ_CC_DEFER=0: the host checks every CC level's error before it enqueues anything that depends
// on the result (the pre-deferral schedule; results are the same either way)
static bool cc_defer_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PQ_CC_DEFER");
        return !(v && v[0] == '0');
    }();
    return on;
}

// The side stream (late exponentials, phi_0) runs one priority step above the main stream, so its
// short dependent launches are not queued behind the node sweep's CTA waves (config 2: 476.7 ->
// 478.5 actions/s); PQ_SIDE_PRIO=0 gives it the main stream's priority.
static bool side_prio_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PQ_SIDE_PRIO");
        return !(v && v[0] == '0');
    }();
    return on;
}

void ensure_side(pq_ctx& c) {
    if (c.side) return;
    if (side_prio_enabled()) {
        int prio = 0, least = 0, greatest = 0;
        if (cudaStreamGetPriority(c.stream, &prio) != cudaSuccess ||
            cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) {
            cudaGetLastError();
            prio = greatest = 0;
        }
        cuda_check(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, std::max(greatest, prio - 1)),
                   "side stream");
    } else {
        make_helper_stream(c, &c.side, "side stream");
    }
    if (!c.ev_fork) cuda_check(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming), "fork event");
    if (!c.ev_join) cuda_check(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming), "join event");
}

struct ExpmEntry {
    long long base_off;  // doubles from `base`
    double scale;        // exact multiplier applied after fl(op_scale * a)
    double one_norm;     // host 1-norm of the base matrix (< 0: unknown -> read counts back)
};

// dense.hpp:194-228 for a batch of n x n matrices: out[z] = expm(scale_z * fl(op_scale * base_z)).
// Six batched DMMA products, two elementwise Pade combinations, one LU solve for all z, then
// max_z s_z squaring rounds in which a finished matrix is carried through unchanged.
static void expm_core(pq_ctx& c, int n, const double* base, double op_scale, const std::vector<ExpmEntry>& es,
                      double* out) {
    const int count = static_cast<int>(es.size());
    if (count <= 0) return;
    const size_t nn = static_cast<size_t>(n) * n, blk = nn * count;
    double* w = ws(c, "expm", 11 * blk);
    double *X = w, *A2 = w + blk, *A4 = w + 2 * blk, *A6 = w + 3 * blk, *TZ = w + 4 * blk, *WZ = w + 6 * blk,
           *W2 = w + 8 * blk, *V = w + 9 * blk, *U = w + 10 * blk;
    int* s_dev = static_cast<int*>(ws_bytes(c, "expm_s", sizeof(int) * count));
    std::vector<double> scales(static_cast<size_t>(count));
    std::vector<long long> offs(static_cast<size_t>(count));
    int s_max = 0;
    bool known = true;
    std::vector<int> hint(static_cast<size_t>(count), 0);  // host upper bound of each s_z
    for (int z = 0; z < count; ++z) {
        scales[static_cast<size_t>(z)] = es[static_cast<size_t>(z)].scale;
        offs[static_cast<size_t>(z)] = es[static_cast<size_t>(z)].base_off;
        if (es[static_cast<size_t>(z)].one_norm < 0.0) {
            known = false;
        } else {
            hint[static_cast<size_t>(z)] = squaring_bound(std::abs(es[static_cast<size_t>(z)].scale * op_scale),
                                                          es[static_cast<size_t>(z)].one_norm);
            s_max = std::max(s_max, hint[static_cast<size_t>(z)]);
        }
    }
    const double* scale_dev = static_cast<const double*>(arena_push(c, scales.data(), sizeof(double) * count));
    const long long* off_dev = static_cast<const long long*>(arena_push(c, offs.data(), sizeof(long long) * count));
    arena_flush(c);
    cudaStream_t st = c.stream;
    launch_expm_prep(n, count, base, 0, off_dev, op_scale, scale_dev, X, s_dev, st);
    count_launch(c);
    if (!known) {  // standalone device expm: read the squaring counts back
        launch_imax(s_dev, count, c.d_int, st);
        count_launch(c);
        int h = 0;
        cuda_check(cudaMemcpyAsync(&h, c.d_int, sizeof(int), cudaMemcpyDeviceToHost, st), "expm s readback");
        cuda_check(cudaStreamSynchronize(st), "expm s sync");
        s_max = h;
    }
    { GemmArgs t = square_batch(n, count, X, X, A2); t.tag = "pade"; gemm(c, t); }
    { GemmArgs t = square_batch(n, count, A2, A2, A4); t.tag = "pade"; gemm(c, t); }
    { GemmArgs t = square_batch(n, count, A2, A4, A6); t.tag = "pade"; gemm(c, t); }
    launch_pade_mid(n, count, A2, A4, A6, TZ, TZ + blk, st);
    count_launch(c);
    {
        GemmArgs g = square_batch(n, 2 * count, A6, TZ, WZ);
        g.zdiv = count;
        g.sA1 = 0;
        g.sA2 = static_cast<long long>(nn);
        g.sB1 = g.sC1 = static_cast<long long>(blk);
        g.sB2 = g.sC2 = static_cast<long long>(nn);
        g.tag = "pade";
        gemm(c, g);
    }
    launch_pade_fin(n, count, WZ, WZ + blk, A2, A4, A6, W2, V, st);
    count_launch(c);
    { GemmArgs t = square_batch(n, count, X, W2, U); t.tag = "pade"; gemm(c, t); }
    double* P = TZ;
    double* Q = (s_max % 2 == 0) ? out : WZ;
    double* other = (s_max % 2 == 0) ? WZ : out;
    launch_pade_pq(static_cast<long long>(blk), V, U, P, Q, st);
    count_launch(c);
    if (n <= 128) {
        int* piv = static_cast<int*>(ws_bytes(c, "expm_piv", 2 * sizeof(int) * count * n));
        launch_lu_factor_solve(n, count, P, Q, piv, c.d_err, st);
        count_launch(c, 2);
    } else {
        launch_lu_solve(n, count, P, Q, c.d_err, st);
        count_launch(c);
    }
    if (!known) std::fill(hint.begin(), hint.end(), s_max);
    squaring_rounds(c, n, count, hint, s_dev, s_max, Q, other, out);
}

// Squaring phase of a batched expm (dense.hpp:222-226): entry z is squared s_z <= hint_z times
// (device counts s_dev decide; the GEMM carries finished entries through).  Rounds cover only
// the suffix that may still need them: matrices before the first z with hint_z > r are finished
// and are flushed to `out` from wherever the ping-pong left them.
static void squaring_rounds(pq_ctx& c, int n, int count, const std::vector<int>& hint, const int* s_dev, int s_max,
                            double* cur, double* other, double* out) {
    const size_t nn = static_cast<size_t>(n) * n;
    if (chain_enabled() && s_max > 1 && s_max <= kMaxChainLevels) {
        // all rounds in one chained launch over every entry: an entry whose squarings are done
        // (sq_round >= its count) is carried through unchanged, so after s_max rounds every entry
        // sits in the buffer round s_max - 1 wrote
        std::vector<GemmArgs> levels;
        double* a = cur;
        double* b = other;
        for (int r = 0; r < s_max; ++r) {
            GemmArgs g = square_batch(n, count, a, a, b);
            g.sq_count = s_dev;
            g.sq_round = r;
            levels.push_back(g);
            std::swap(a, b);
        }
        gemm_chain(c, levels, "expm_squaring");
        if (a != out) dev_copy(c, out, a, static_cast<size_t>(count) * nn, c.stream);
        check_launch(c);
        return;
    }
    cudaStream_t st = c.stream;
    int z_done = 0;
    auto flush = [&](int z_from, int z_to) {
        if (z_to > z_from && cur != out)
            dev_copy(c, out + static_cast<size_t>(z_from) * nn, cur + static_cast<size_t>(z_from) * nn,
                     static_cast<size_t>(z_to - z_from) * nn, st);
    };
    for (int r = 0; r < s_max; ++r) {
        int z0 = z_done;
        while (z0 < count && hint[static_cast<size_t>(z0)] <= r) ++z0;
        flush(z_done, z0);
        z_done = z0;
        if (z0 >= count) break;
        GemmArgs g = square_batch(n, count - z0, cur + static_cast<size_t>(z0) * nn, cur + static_cast<size_t>(z0) * nn,
                                  other + static_cast<size_t>(z0) * nn);
        g.sq_count = s_dev + z0;
        g.sq_round = r;
        g.tag = "expm_squaring";
        gemm(c, g);
        std::swap(cur, other);
    }
    flush(z_done, count);
    check_launch(c);
}

// The exponentials one phi call needs are all scalar multiples of a few factors,
// exp(c_z * G_f) with G_f = fl(op_scale * A_f).  Instead of one Pade-13 solve per matrix (an LU
// each, latency-bound), evaluate a degree-m Taylor polynomial on SHARED powers: with
// B_f = 2^-e_f G_f (exact, ||B_f||_1 <= 1) and alpha_z = c_z 2^(e_f - s_z) (exact),
//   exp(c_z G_f) = (sum_k alpha_z^k / k! B_f^k)^(2^s_z),   ||alpha_z B_f||_1 <= theta_m,
// where theta_m bounds the relative backward error of the truncated series by u = 2^-53 (the
// same criterion dense.hpp's Pade-13 threshold 5.37 encodes; tools/taylor_theta.py computes it
// in exact rational arithmetic).  m = 32 (theta_32 = 4.0076): the powers B^2..B^32 of every factor
// take five batched DMMA launches that do not depend on the plan, so phiquadmv enqueues them
// before it waits for beta (taylor_prefetch); the combination is one elementwise pass and the
// squarings reuse squaring_rounds.  Against an eigendecomposition ground truth this is as
// accurate as the reference's Pade-13.
constexpr int kTaylorM = 32;
constexpr double kTaylorTheta = 4.00756108611804;

static bool taylor_disabled() {
    static const bool disabled = [] {
        const char* v = std::getenv("PQ_EXPM");
        return v && std::string(v) == "pade";
    }();
    return disabled;
}

// per canonical factor: gnorm >= ||fl(op_scale A_f)||_1, 2^-e_f and 2^e_f with 2^e_f >= gnorm
struct TaylorFactors {
    std::vector<long long> foff;
    std::vector<double> gnorm, pow2, nu;
};
static bool taylor_factors(double op_scale, const std::vector<long long>& foff, const std::vector<double>& fnorm,
                           TaylorFactors& tf) {
    tf.foff = foff;
    const size_t nf = foff.size();
    tf.gnorm.assign(nf, 0.0);
    tf.pow2.assign(nf, 1.0);
    tf.nu.assign(nf, 1.0);
    for (size_t f = 0; f < nf; ++f) {
        // ||fl(op_scale A_f)||_1 <= |op_scale| ||A_f||_1 (1 + n u); the margin keeps the theta test safe
        const double g = std::abs(op_scale) * fnorm[f] * (1.0 + 1e-12);
        if (!std::isfinite(g)) return false;
        tf.gnorm[f] = g;
        int ex = 0;
        if (g > 0.0) std::frexp(g, &ex);  // 2^ex >= g
        tf.nu[f] = std::ldexp(1.0, ex);
        tf.pow2[f] = std::ldexp(1.0, -ex);
    }
    return true;
}

// B_f^k, k = 1..kTaylorM, stored [f][k-1][n x n] in ws "taylorP<n>"; reused within one API call
// (same DevOp serial, scale and factor set), recomputed otherwise.
static const double* taylor_powers(pq_ctx& c, int n, const double* base, double op_scale, const TaylorFactors& tf,
                                   uint64_t serial) {
    const int nf = static_cast<int>(tf.foff.size());
    const size_t nn = static_cast<size_t>(n) * n;
    double* P = ws(c, "taylorP" + std::to_string(n), static_cast<size_t>(nf) * kTaylorM * nn);
    pq_ctx::PowCache& pc = c.pow_cache[n];
    // The powers only depend on the scale's mantissa: fl(2^k m A) = 2^k fl(m A) exactly and the
    // normalisation 2^-e_f absorbs 2^k, so B_f is bit-identical for every power-of-two multiple of
    // the scale (the ETD stages' sigma = 1/2 and 1 share one set of powers within a call).
    int e_new = 0, e_old = 0;
    const double m_new = std::frexp(op_scale, &e_new), m_old = std::frexp(pc.scale, &e_old);
    if (serial != 0 && pc.serial == serial && pc.P == P && pc.base == base && pc.foff == tf.foff && m_new == m_old &&
        std::abs(e_new - e_old) <= 64)
        return P;
    const long long* foff_dev = static_cast<const long long*>(arena_push(c, tf.foff.data(), sizeof(long long) * nf));
    const double* pow2_dev = static_cast<const double*>(arena_push(c, tf.pow2.data(), sizeof(double) * nf));
    arena_flush(c);
    launch_taylor_base(n, nf, kTaylorM, base, foff_dev, op_scale, pow2_dev, P, c.stream);
    count_launch(c);
    const long long lnn = static_cast<long long>(nn), fs = static_cast<long long>(kTaylorM) * lnn;
    // P^(h+j) = P^h P^j, j = 1..min(h, m-h), all factors per level; the log2(m) dependent levels
    // run as one chained cooperative launch (gemm_chain)
    std::vector<GemmArgs> levels;
    for (int h = 1; h < kTaylorM; h *= 2) {
        const int J = std::min(h, kTaylorM - h);
        GemmArgs g = square_batch(n, nf * J, P + (h - 1) * lnn, P, P + h * lnn);
        g.zdiv = J;
        g.sA1 = fs;
        g.sA2 = 0;
        g.sB1 = fs;
        g.sB2 = lnn;
        g.sC1 = fs;
        g.sC2 = lnn;
        levels.push_back(g);
    }
    gemm_chain(c, levels, "taylor_powers");
    pc.P = P;
    pc.base = base;
    pc.foff = tf.foff;
    pc.scale = op_scale;
    pc.serial = serial;
    return P;
}

// Entries [split, count) are "late" (needed only after the node sweep: the squaring chain and
// phi_0): with late_async their combination and squaring rounds run on the side stream, which
// records c.ev_late when done; entries [0, split) are finished on c.stream.  Returns false
// (caller uses expm_core) when a norm is unknown or PQ_EXPM=pade.
static bool expm_taylor(pq_ctx& c, int n, const double* base, double op_scale, const std::vector<ExpmEntry>& es,
                        double* out, int split = -1, bool late_async = false, int2* band = nullptr,
                        uint64_t serial = 0) {
    const int count = static_cast<int>(es.size());
    if (taylor_disabled() || count <= 0) return false;
    std::vector<long long> foff;
    std::vector<double> fnorm;
    std::vector<int> fidx(static_cast<size_t>(count));
    for (int z = 0; z < count; ++z) {
        const ExpmEntry& e = es[static_cast<size_t>(z)];
        if (!(e.one_norm >= 0.0) || !std::isfinite(e.scale)) return false;
        size_t f = 0;
        while (f < foff.size() && foff[f] != e.base_off) ++f;
        if (f == foff.size()) {
            foff.push_back(e.base_off);
            fnorm.push_back(e.one_norm);
        }
        fidx[static_cast<size_t>(z)] = static_cast<int>(f);
    }
    TaylorFactors tf;
    if (!taylor_factors(op_scale, foff, fnorm, tf)) return false;
    if (split < 0 || split > count) split = count;
    constexpr int m = kTaylorM;
    std::vector<int> hint(static_cast<size_t>(count));
    std::vector<double> coef(static_cast<size_t>(count) * (m + 1));
    for (int z = 0; z < count; ++z) {
        const size_t f = static_cast<size_t>(fidx[static_cast<size_t>(z)]);
        const double x = std::abs(es[static_cast<size_t>(z)].scale) * tf.gnorm[f];
        const int s = x > kTaylorTheta ? static_cast<int>(std::ceil(std::log2(x / kTaylorTheta))) : 0;
        hint[static_cast<size_t>(z)] = s;
        const double alpha = std::ldexp(es[static_cast<size_t>(z)].scale * tf.nu[f], -s);
        double* t = coef.data() + static_cast<size_t>(z) * (m + 1);
        t[0] = 1.0;
        for (int k = 1; k <= m; ++k) t[k] = t[k - 1] * alpha / k;
    }
    // int4 {factor, first entry, count, 0}: runs of one factor, <= kTaylorChunk, per range
    auto chunks_of = [&](int z_begin, int z_end) {
        std::vector<int> ch;
        for (int z = z_begin; z < z_end;) {
            int e = z + 1;
            while (e < z_end && e - z < kTaylorChunk && fidx[static_cast<size_t>(e)] == fidx[static_cast<size_t>(z)]) ++e;
            ch.insert(ch.end(), {fidx[static_cast<size_t>(z)], z, e - z, 0});
            z = e;
        }
        return ch;
    };
    const std::vector<int> ch_early = chunks_of(0, split), ch_late = chunks_of(split, count);
    const size_t nn = static_cast<size_t>(n) * n;
    const double* P = taylor_powers(c, n, base, op_scale, tf, serial);
    double* T = ws(c, "taylorT", static_cast<size_t>(count) * nn);
    const double* coef_dev = static_cast<const double*>(arena_push(c, coef.data(), sizeof(double) * coef.size()));
    const int* che_dev = ch_early.empty() ? nullptr
                                          : static_cast<const int*>(arena_push(c, ch_early.data(), sizeof(int) * ch_early.size()));
    const int* chl_dev = ch_late.empty() ? nullptr
                                         : static_cast<const int*>(arena_push(c, ch_late.data(), sizeof(int) * ch_late.size()));
    const int* s_dev = static_cast<const int*>(arena_push(c, hint.data(), sizeof(int) * count));
    arena_flush(c);
    // combination + squaring rounds of entries [z_begin, z_end) on c.stream; the ping-pong partner
    // of entry z is tbase + (z - z_begin) n^2 (the late range has its own scratch, see below)
    auto finish = [c_ = &c, n, nn, out, P, coef_dev, s_dev, band, hint](int z_begin, int z_end, const std::vector<int>& ch,
                                                                         const int* ch_dev, double* tbase) {
        pq_ctx& c = *c_;
        if (z_end <= z_begin) return;
        const std::vector<int> h(hint.begin() + z_begin, hint.begin() + z_end);
        const int s_max = *std::max_element(h.begin(), h.end());
        double* o = out + static_cast<size_t>(z_begin) * nn;
        double* t = tbase;
        double* first = (s_max % 2 == 0) ? o : t;
        // the combination kernel indexes absolute entries: shift the base so entry z_begin lands at `first`
        launch_taylor_combine(n, m, static_cast<int>(ch.size() / 4), ch_dev, coef_dev, P,
                              first - static_cast<size_t>(z_begin) * nn, c.stream);
        count_launch(c);
        squaring_rounds(c, n, z_end - z_begin, h, s_dev + z_begin, s_max, first, first == o ? t : o, o);
        band_ranges(c, n, z_end - z_begin, o, band ? band + static_cast<size_t>(z_begin) * band_row_blocks(n) : nullptr);
    };
    finish(0, split, ch_early, che_dev, T);
    if (split < count) {
        if (late_async) {
            // the late entries depend only on the powers already enqueued: fork here, but enqueue
            // their work after the first node sweep (run_deferred), so it does not delay the sweep
            ensure_side(c);
            if (!c.ev_late) cuda_check(cudaEventCreateWithFlags(&c.ev_late, cudaEventDisableTiming), "late event");
            if (!c.ev_latefork) cuda_check(cudaEventCreateWithFlags(&c.ev_latefork, cudaEventDisableTiming), "late fork");
            cuda_check(cudaEventRecord(c.ev_latefork, c.stream), "late fork");
            double* tl = ws(c, "taylorTlate", static_cast<size_t>(count - split) * nn);
            c.deferred.push_back([c_ = &c, finish, split, count, ch_late, chl_dev, tl] {
                pq_ctx& c = *c_;
                cuda_check(cudaStreamWaitEvent(c.side, c.ev_latefork, 0), "late fork wait");
                const cudaStream_t main_stream = c.stream;
                c.stream = c.side;
                try {
                    finish(split, count, ch_late, chl_dev, tl);
                } catch (...) {
                    c.stream = main_stream;
                    throw;
                }
                c.stream = main_stream;
                cuda_check(cudaEventRecord(c.ev_late, c.side), "late record");
            });
        } else {
            finish(split, count, ch_late, chl_dev, T + static_cast<size_t>(split) * nn);
        }
    }
    check_launch(c);
    return true;
}

void run_deferred(pq_ctx& c) {
    std::vector<std::function<void()>> work;
    work.swap(c.deferred);
    for (auto& w : work) w();
}

void expm_batch(pq_ctx& c, int n, int count, const double* base, long long base_stride, const std::vector<double>& scales,
                double base_one_norm, double* out) {
    // Large dense matrices (the dense phi oracle's augmented matrix): the
    // per-matrix LU of the Pade solve runs in one CTA and is impractical beyond n ~ 512, so they
    // take the shared-power Taylor path (DMMA products + squarings over the whole GPU; as accurate,
    // DESIGN.md 3a).  Its degree/scaling choice needs the 1-norm on the host.
    if (n > 512 && base_stride == 0) {
        if (base_one_norm < 0.0) {
            std::vector<double> h(static_cast<size_t>(n) * n), col(static_cast<size_t>(n), 0.0);
            cuda_check(cudaMemcpyAsync(h.data(), base, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c.stream),
                       "expm norm readback");
            cuda_check(cudaStreamSynchronize(c.stream), "expm norm sync");
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) col[static_cast<size_t>(j)] += std::abs(h[static_cast<size_t>(i) * n + j]);
            base_one_norm = *std::max_element(col.begin(), col.end());
        }
        std::vector<ExpmEntry> es;
        for (int z = 0; z < count; ++z) es.push_back({0, scales[static_cast<size_t>(z)], base_one_norm});
        if (expm_taylor(c, n, base, 1.0, es, out)) return;
    }
    std::vector<ExpmEntry> es;
    for (int z = 0; z < count; ++z) es.push_back({z * base_stride, scales[static_cast<size_t>(z)], base_one_norm});
    expm_core(c, n, base, 1.0, es, out);
}

// All 1-D exponentials one phi call needs, computed in ONE batch per distinct factor size:
//   node[k] + a*n_k^2 = expm((1 - theta_a) 2^-l fl(s A_k))   (phiaction.hpp:90, :197)
//   sq[k] + j*n_k^2   = expm(2^(j-l) fl(s A_k)), j < sq_len  (phiaction.hpp:294-296: the reference
//                       squares E after every doubling step; with sq_chain the whole chain
//                       E, E^2, E^4, ... is evaluated directly, sq_len = l, else sq_len = 1)
//   phi0[k]           = expm(fl(s A_k))                       (kron.hpp:125)
// Bitwise-identical factors are exponentiated once (e.g. the isotropic Laplacians of configs
// 1, 3, 4, 5): dims sharing a factor share the pointers.  With late_async the squaring chain and
// phi_0 matrices are finished on the side stream (late = true: wait on c.ev_late before use).


PhiExps phi_exponentials(pq_ctx& c, const DevOp& op, double s, int l, const std::vector<double>& thetas,
                         bool want_sq, bool want_phi0, const std::string& tag, bool sq_chain, bool late_async) {
    PhiExps px;
    const int q = static_cast<int>(thetas.size());
    const int L = want_sq ? (sq_chain ? std::max(l, 1) : 1) : 0;
    px.sq_len = std::max(L, 1);
    const int per = q + L + (want_phi0 ? 1 : 0);
    if (per == 0) return px;
    // canonical factors (upload_op: bit-identical factors share one exponential)
    int canon[3] = {0, 1, 2};
    size_t off[3] = {0, 0, 0};
    for (int k = 1; k < op.d; ++k) off[k] = off[k - 1] + static_cast<size_t>(op.n[k - 1]) * op.n[k - 1];
    for (int k = 0; k < op.d; ++k) canon[k] = op.canon[k];
    // one batch per distinct n over the canonical factors with that n
    std::vector<int> done(3, 0);
    const double* base = op.F[0];  // factors are contiguous on the device
    for (int k = 0; k < op.d; ++k) {
        if (canon[k] != k || done[k]) continue;
        const int n = op.n[k];
        std::vector<int> group;
        for (int j = k; j < op.d; ++j)
            if (canon[j] == j && op.n[j] == n) {
                group.push_back(j);
                done[j] = 1;
            }
        // batch layout [nodes of every factor][squaring chain of every factor][phi_0 matrices]:
        // the large-norm late arguments form the suffix, so only they take squaring rounds
        std::vector<ExpmEntry> es;
        for (int f : group) {
            const long long bo = static_cast<long long>(off[f]);
            for (int a = 0; a < q; ++a) es.push_back({bo, std::ldexp(1.0 - thetas[static_cast<size_t>(a)], -l), op.one_norm[f]});
        }
        const int split = static_cast<int>(es.size());
        for (int f : group)
            for (int j = 0; j < L; ++j) es.push_back({static_cast<long long>(off[f]), std::ldexp(1.0, j - l), op.one_norm[f]});
        if (want_phi0)
            for (int f : group) es.push_back({static_cast<long long>(off[f]), 1.0, op.one_norm[f]});
        const size_t nn = static_cast<size_t>(n) * n, ng = group.size();
        double* out = ws(c, tag + "_n" + std::to_string(n), es.size() * nn);
        const int RB = band_row_blocks(n);
        int2* band = band_enabled(n, op.N)
                         ? static_cast<int2*>(ws_bytes(c, tag + "_band" + std::to_string(n), sizeof(int2) * es.size() * RB))
                         : nullptr;
        if (band)
            band_pack_register(c, band, es.size(),
                               op.d == 3 && e2pack_enabled(n)
                                   ? ws(c, tag + "_pack" + std::to_string(n), es.size() * band_pack_doubles(n))
                                   : nullptr,
                               n);
        // the side stream is in order, so waiting on the last ev_late covers every group's late work
        const bool async = late_async && split < static_cast<int>(es.size());
        if (expm_taylor(c, n, base, s, es, out, split, async, band, op.serial)) {
            px.late = px.late || async;
        } else {
            expm_core(c, n, base, s, es, out);
            band_ranges(c, n, static_cast<int>(es.size()), out, band);
        }
        for (size_t g = 0; g < ng; ++g) {
            px.node[group[g]] = out + g * q * nn;
            px.sq[group[g]] = L > 0 ? out + (ng * q + g * L) * nn : nullptr;
            px.phi0[group[g]] = want_phi0 ? out + (ng * q + ng * L + g) * nn : nullptr;
            if (band) {
                px.node_band[group[g]] = band + g * q * RB;
                px.sq_band[group[g]] = L > 0 ? band + (ng * q + g * L) * RB : nullptr;
                px.phi0_band[group[g]] = want_phi0 ? band + (ng * q + ng * L + g) * RB : nullptr;
            }
        }
    }
    for (int k = 0; k < op.d; ++k) {
        px.node[k] = px.node[canon[k]];
        px.sq[k] = px.sq[canon[k]];
        px.phi0[k] = px.phi0[canon[k]];
        px.node_band[k] = px.node_band[canon[k]];
        px.sq_band[k] = px.sq_band[canon[k]];
        px.phi0_band[k] = px.phi0_band[canon[k]];
    }
    return px;
}

// Canonical factors grouped by size exactly as phi_exponentials batches them, so the prefetched
// powers carry the same factor set (and cache key) as the exponentials that use them.
void taylor_prefetch(pq_ctx& c, const DevOp& op, double scale) {
    if (taylor_disabled()) return;
    size_t off[3] = {0, 0, 0};
    for (int k = 1; k < op.d; ++k) off[k] = off[k - 1] + static_cast<size_t>(op.n[k - 1]) * op.n[k - 1];
    int canon[3] = {0, 1, 2};
    for (int k = 0; k < op.d; ++k) canon[k] = op.canon[k];
    std::vector<int> done(3, 0);
    for (int k = 0; k < op.d; ++k) {
        if (canon[k] != k || done[k]) continue;
        const int n = op.n[k];
        std::vector<long long> foff;
        std::vector<double> fnorm;
        for (int j = k; j < op.d; ++j)
            if (canon[j] == j && op.n[j] == n) {
                foff.push_back(static_cast<long long>(off[j]));
                fnorm.push_back(op.one_norm[j]);
                done[j] = 1;
            }
        TaylorFactors tf;
        if (taylor_factors(scale, foff, fnorm, tf)) taylor_powers(c, n, op.F[0], scale, tf, op.serial);
    }
}

// ------------------------------------------------------------------ mode products --------

// One mode product of the chain (kron.hpp:65-87 accumulate_mode_apply, as a GEMM).
static GemmArgs mode_gemm(int d, const int* n, int k, const double* E, long long E_stride, const double* x,
                          long long x_stride, double* y, long long y_stride, int Z1, long long N) {
    long long O = 1, I = 1;
    for (int i = 0; i < k; ++i) O *= n[i];
    for (int i = k + 1; i < d; ++i) I *= n[i];
    const int nk = n[k];
    GemmArgs g;
    if (I > 1) {
        // Y_o = E_k X_o, X_o an nk x I row-major slab
        g.A = E;
        g.lda = nk;
        g.B = x;
        g.ldb = I;
        g.C = y;
        g.ldc = I;
        g.K = nk;
        g.N = static_cast<int>(I);
        if (O == 1 && x_stride == 0 && E_stride == static_cast<long long>(nk) * nk && y_stride == N && Z1 > 1) {
            // shared input, consecutive E blocks: stack the node exponentials along M (one GEMM)
            g.M = Z1 * nk;
            g.Z = 1;
        } else {
            g.M = nk;
            g.Z = static_cast<int>(Z1 * O);
            g.zdiv = static_cast<int>(O);
            g.sA1 = E_stride;
            g.sB1 = x_stride;
            g.sB2 = nk * I;
            g.sC1 = y_stride;
            g.sC2 = nk * I;
        }
    } else {
        // last mode: Y (O x nk) = X (O x nk) E_k^T ; E_k row-major is E_k^T column-major
        g.A = x;
        g.lda = nk;
        g.B = E;
        g.b_kmajor = 1;
        g.ldb = nk;
        g.C = y;
        g.ldc = nk;
        g.M = static_cast<int>(O);
        g.N = nk;
        g.K = nk;
        g.Z = Z1;
        g.sA1 = x_stride;
        g.sB1 = E_stride;
        g.sC1 = y_stride;
    }
    (void)d;
    return g;
}

GemmArgs mode_gemm_public(int d, const int* n, int mode, const double* E, const double* x, double* y, int nb,
                          long long N) {
    return mode_gemm(d, n, mode, E, 0, x, N, y, N, nb, N);
}

void mode_product_dev(pq_ctx& c, int d, const int* n, int k, const double* E, const int2* band, const double* x,
                      long long x_stride, double* y, long long y_stride, int Z1, const RemoteMap* remote) {
    long long N = 1;
    for (int i = 0; i < d; ++i) N *= n[i];
    GemmArgs g = mode_gemm(d, n, k, E, 0, x, x_stride, y, y_stride, Z1, N);
    g.remote = remote;
    if (band) {  // one exponential shared by the batch (E_stride 0), as mode_chain sets it up
        g.band = band;
        g.band_rows = n[k];
        g.band_stride = 0;
        g.band_mode = g.b_kmajor ? 3 : 2;
    }
    g.tag = "mode_product";
    gemm(c, g);
    check_launch(c);
}

void mode_chain(pq_ctx& c, int d, const int* n, const double* const* E, const long long* E_stride, const double* x,
                long long x_stride, double* y, long long y_stride, int Z1, const Epilogue& ep, const char* tmp_tag,
                const int2* const* band, const std::function<void()>& before_last) {
    long long N = 1;
    for (int k = 0; k < d; ++k) N *= n[k];
    // modes 1 and 2 of a 3-D apply in one kernel (slab12.cu) when the last mode's epilogue is a
    // plain store and the operands are 16-byte aligned
    const bool fuse12 = d == 3 && slab12_enabled() && slab12_supported(n[1], n[2]) && !ep.alpha_z && !ep.ext &&
                        !ep.coef && !ep.nterms && !ep.accumulate && E_stride[1] % 2 == 0 && E_stride[2] % 2 == 0 &&
                        y_stride % 2 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
                        (reinterpret_cast<uintptr_t>(E[1]) & 15) == 0 && (reinterpret_cast<uintptr_t>(E[2]) & 15) == 0;
    double* tmp[2] = {nullptr, nullptr};
    if (d > 1) tmp[0] = ws(c, std::string(tmp_tag) + "A", static_cast<size_t>(Z1) * N);
    if (d > 2 && !fuse12) tmp[1] = ws(c, std::string(tmp_tag) + "B", static_cast<size_t>(Z1) * N);
    const double* src = x;
    long long sstride = x_stride;
    for (int k = 0; k < d; ++k) {
        if (fuse12 && k == 1) {
            Slab12Args sg;
            for (int m = 1; m <= 2; ++m) {
                const long long nn = static_cast<long long>(n[m]) * n[m];
                const int2* bt = band && band[m] && E_stride[m] % nn == 0 ? band[m] : nullptr;
                const long long bs = bt ? (E_stride[m] / nn) * band_row_blocks(n[m]) : 0;
                if (m == 1) {
                    sg.E1 = E[1];
                    sg.sE1 = E_stride[1];
                    sg.band1 = bt;
                    sg.sband1 = bs;
                } else {
                    sg.E2 = E[2];
                    sg.sE2 = E_stride[2];
                    sg.band2 = bt;
                    sg.sband2 = bs;
                    long long pd = 0;
                    sg.E2p = band_pack_find(c, bt, n[m], &pd);
                    sg.sE2p = (E_stride[m] / nn) * pd;
                }
            }
            sg.X = src;
            sg.sX = sstride;
            sg.Y = y;
            sg.sY = y_stride;
            sg.n0 = n[0];
            sg.Z1 = Z1;
            if (before_last) before_last();
            slab12(c, sg, (std::string(tmp_tag) + ":mode12").c_str());
            break;
        }
        const bool last = k == d - 1;
        double* dst = last ? y : tmp[k % 2];
        const long long dstride = last ? y_stride : N;
        GemmArgs g = mode_gemm(d, n, k, E[k], E_stride[k], src, sstride, dst, dstride, Z1, N);
        const std::string tagk = std::string(tmp_tag) + ":mode" + std::to_string(k);
        const long long nn = static_cast<long long>(n[k]) * n[k];
        if (band && band[k] && E_stride[k] % nn == 0) {
            // which operand holds the exponentials, and how the tile finds its matrix (gemm.cuh)
            const int RB = band_row_blocks(n[k]);
            g.band = band[k];
            g.band_rows = n[k];
            g.band_stride = (E_stride[k] / nn) * RB;
            g.band_mode = g.b_kmajor ? 3 : (g.Z == 1 && g.M == Z1 * n[k] && Z1 > 1 ? 1 : 2);
            if (g.band_mode == 1) g.band_stride = RB;
        }
        if (last) {
            g.alpha_z = ep.alpha_z;
            g.ext = ep.ext;
            g.ext_s = ep.ext_s;
            g.coef = ep.coef;
            g.cld = ep.cld;
            g.nterms = ep.nterms;
            g.accumulate = ep.accumulate;
            if (ep.cld > 0) g.ext_group = ep.cld;
        }
        g.tag = tagk.c_str();
        if (last && before_last) before_last();
        gemm(c, g);
        src = dst;
        sstride = dstride;
    }
    check_launch(c);
}

// Negligible-block tables of the unscaled factors (scaling does not move them); the factors of
// the benchmark operators are tridiagonal, so a 32-row block needs ~5 of 16 k-slices.  Exact:
// the dropped blocks hold only entries below 2^-64 of the block's max (for these factors, zeros,
// which the reference skips too, kron.hpp:81).  Cached per operator upload.
static void factor_bands(pq_ctx& c, const DevOp& op, const int2** out) {
    for (int k = 0; k < op.d; ++k) out[k] = nullptr;
    bool any = false;
    for (int k = 0; k < op.d; ++k) any = any || band_enabled(op.n[k], op.N);
    if (!any) return;
    if (c.fac_band_serial != op.serial || op.serial == 0) {
        for (int k = 0; k < op.d; ++k) {
            c.fac_band[k] = nullptr;
            if (!band_enabled(op.n[k], op.N)) continue;
            int2* b = static_cast<int2*>(ws_bytes(c, "facband" + std::to_string(k), sizeof(int2) * band_row_blocks(op.n[k])));
            band_pack_register(c, b, 1, nullptr, op.n[k]);
            band_ranges(c, op.n[k], 1, op.F[k], b);
            c.fac_band[k] = b;
        }
        c.fac_band_serial = op.serial;
    }
    for (int k = 0; k < op.d; ++k) out[k] = c.fac_band[k];
}

// kron.hpp:111-119: y = sum_k mode_k(A_k) x (factor scaled by `scale` first when != 1).
// every factor tridiagonal (|i - j| > 1 -> 0)?  From the operator's host copy, cached per upload.
static bool factors_tridiagonal(pq_ctx& c, const DevOp& op) {
    if (op.serial != 0 && c.tri_serial == op.serial) return c.tri;
    bool tri = op.host != nullptr;
    size_t off = 0;
    for (int k = 0; k < op.d && tri; ++k) {
        const int n = op.n[k];
        const double* f = op.host->data() + off;
        for (int i = 0; i < n && tri; ++i)
            for (int j = 0; j < n; ++j)
                if ((j < i - 1 || j > i + 1) && f[static_cast<size_t>(i) * n + j] != 0.0) {
                    tri = false;
                    break;
                }
        off += static_cast<size_t>(n) * n;
    }
    c.tri_serial = op.serial;
    c.tri = tri;
    return tri;
}

static bool stencil_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PQ_KMV_STENCIL");
        return !(v && v[0] == '0');
    }();
    return on;
}

void kron_matvec_dev(pq_ctx& c, const DevOp& op, double scale, const double* x, double* y) {
    if (stencil_enabled() && factors_tridiagonal(c, op)) {
        // tridiagonal factors (the FD operators of every BASELINE config): one streaming pass,
        // the reference's term order (bitwise its kron_matvec)
        int nmax = 1;
        for (int k = 0; k < op.d; ++k) nmax = std::max(nmax, op.n[k]);
        double* diag = ws(c, "kmv_diag", 9 * static_cast<size_t>(nmax));
        KernelProbe kp(c, "k_kron_tridiag", 16.0 * op.N);
        launch_kron_tridiag(op.d, op.n, op.N, op.F, scale, x, y, diag, c.stream);
        count_launch(c, 2);
        return;
    }
    const double* F[3] = {op.F[0], op.F[1], op.F[2]};
    if (scale != 1.0) {
        size_t total = 0;
        for (int k = 0; k < op.d; ++k) total += static_cast<size_t>(op.n[k]) * op.n[k];
        double* sf = ws(c, "kmv_scaled", total);
        launch_scale_copy(static_cast<long long>(total), scale, op.F[0], sf, c.stream);
        count_launch(c);
        size_t off = 0;
        for (int k = 0; k < op.d; ++k) {
            F[k] = sf + off;
            off += static_cast<size_t>(op.n[k]) * op.n[k];
        }
    }
    const int2* fb[3];
    factor_bands(c, op, fb);
    for (int k = 0; k < op.d; ++k) {
        GemmArgs g = mode_gemm(op.d, op.n, k, F[k], 0, x, 0, y, 0, 1, op.N);
        g.accumulate = k > 0;
        if (fb[k]) {
            g.band = fb[k];
            g.band_rows = op.n[k];
            g.band_stride = 0;
            g.band_mode = g.b_kmajor ? 3 : 2;
        }
        g.tag = "kron_matvec";
        gemm(c, g);
    }
    check_launch(c);
}

void apply_phi0(pq_ctx& c, const DevOp& op, const PhiExps& px, int nb, const double* b, double* y) {
    long long Es[3] = {0, 0, 0};
    mode_chain(c, op.d, op.n, px.phi0, Es, b, op.N, y, op.N, nb, Epilogue{}, "phi0", px.phi0_band);
}

// kron.hpp:123-128 (phi_0): expm of every (scaled) factor, then one mode chain per RHS.
void exp_action_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* b, double* y) {
    const PhiExps px = phi_exponentials(c, op, scale, 0, {}, false, true, "phi0E");
    apply_phi0(c, op, px, nb, b, y);
}

double max_inf_norm_dev(pq_ctx& c, const double* v, long long N, int ncols) {
    double* out = ws(c, "colstats", 2 * static_cast<size_t>(ncols));
    launch_colstats(N, ncols, v, nullptr, out, c.stream);
    count_launch(c);
    std::vector<double> h(2 * static_cast<size_t>(ncols));
    cuda_check(cudaMemcpyAsync(h.data(), out, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "norm readback");
    cuda_check(cudaStreamSynchronize(c.stream), "norm sync");
    double best = 0.0;
    for (int k = 0; k < ncols; ++k) best = std::max(best, h[2 * k + 1]);
    return best;
}

// ------------------------------------------------------------------ the node sweep -------

// phiaction.hpp:102-107: coefficient w_i theta_i^{j-1}/(j-1)! by the same running product.
void node_coefs(const NodesWeights& r, const std::vector<int>& idx, int p, std::vector<double>& out) {
    out.assign(idx.size() * static_cast<size_t>(p), 0.0);
    for (size_t a = 0; a < idx.size(); ++a) {
        const double th = r.x[static_cast<size_t>(idx[a])];
        double coeff = r.w[static_cast<size_t>(idx[a])];
        for (int j = 1; j <= p; ++j) {
            out[a * p + (j - 1)] = coeff;
            coeff *= th / j;
        }
    }
}

static int node_chunk(pq_ctx& c, long long N, int q, int per_node_vectors) {
    const double budget = static_cast<double>(budget_bytes(c)) * 0.9;
    const double per = static_cast<double>(N) * sizeof(double) * per_node_vectors;
    int qc = static_cast<int>(budget / per);
    if (qc < 1) qc = 1;
    return std::min(q, qc);
}

std::vector<double> thetas_of(const NodesWeights& r, const std::vector<int>& idx) {
    std::vector<double> t;
    for (int i : idx) t.push_back(r.x[static_cast<size_t>(i)]);
    return t;
}

// For the selected nodes (exponentials E[k] + a*Es[k], a < q), v_a = (E_a0 (x) E_a1 (x) E_a2) b_m;
// either combined into acc [nb][p][N] with coefficients coef [q][p] (zeroing first if `zero`),
// or stored into pool + (slot0 + a)*nb*N + m*N.
void node_sweep(pq_ctx& c, const DevOp& op, const double* const* E, const long long* Es, int q, int nb,
                const double* bs, int p, const std::vector<double>* coef, double* acc, int zero, double* pool,
                int slot0, const int2* const* band) {
    // band tables follow their exponentials: matrix a of E[k] (stride Es[k]) <-> band[k] + a (Es[k]/n^2) RB
    auto band_at = [&](int a0, const int2** out) {
        for (int k = 0; k < op.d; ++k) {
            const long long nn = static_cast<long long>(op.n[k]) * op.n[k];
            out[k] = band && band[k] ? band[k] + (a0 * (Es[k] / nn)) * band_row_blocks(op.n[k]) : nullptr;
        }
    };
    const long long N = op.N;
    if (q == 0) {
        if (acc && zero) cuda_check(cudaMemsetAsync(acc, 0, sizeof(double) * nb * p * N, c.stream), "zero acc");
        return;
    }
    if (pool) {
        const int qc = node_chunk(c, N, q, 2);
        for (int m = 0; m < nb; ++m)
            for (int a0 = 0; a0 < q; a0 += qc) {
                const int cnt = std::min(qc, q - a0);
                const double* Ec[3];
                const int2* Bc[3];
                for (int k = 0; k < op.d; ++k) Ec[k] = E[k] + a0 * Es[k];
                band_at(a0, Bc);
                mode_chain(c, op.d, op.n, Ec, Es, bs + m * N, 0, pool + (static_cast<long long>(slot0 + a0) * nb + m) * N,
                           nb * N, cnt, Epilogue{}, "chain", Bc);
            }
        return;
    }
    const double* coef_dev = static_cast<const double*>(arena_push(c, coef->data(), coef->size() * sizeof(double)));
    std::vector<int> slots(static_cast<size_t>(q));
    std::iota(slots.begin(), slots.end(), 0);
    const int* slot_dev = static_cast<const int*>(arena_push(c, slots.data(), slots.size() * sizeof(int)));
    arena_flush(c);
    const int qc = node_chunk(c, N, q, 3);
    double* V = ws(c, "nodeV", static_cast<size_t>(qc) * N);
    for (int m = 0; m < nb; ++m)
        for (int a0 = 0; a0 < q; a0 += qc) {
            const int cnt = std::min(qc, q - a0);
            const double* Ec[3];
            const int2* Bc[3];
            for (int k = 0; k < op.d; ++k) Ec[k] = E[k] + a0 * Es[k];
            band_at(a0, Bc);
            mode_chain(c, op.d, op.n, Ec, Es, bs + m * N, 0, V, N, cnt, Epilogue{}, "chain", Bc);
            KernelProbe kp(c, "k_combine", 8.0 * N * (cnt + p + ((zero && a0 == 0) ? 0 : p)));
            launch_combine(N, p, cnt, V, N, slot_dev, coef_dev + static_cast<size_t>(a0) * p,
                           acc + static_cast<long long>(m) * p * N, N, (zero && a0 == 0) ? 1 : 0, c.stream);
            count_launch(c);
        }
    check_launch(c);
}

// phiaction.hpp:134-145 (Alg. 1 on an explicit rule) on 2^-l fl(s A).
static void phi_fixed_shift(pq_ctx& c, const DevOp& op, double s, int l, int nb, const double* bs, int p,
                            const NodesWeights& rule, const PhiExps& px, double* out) {
    std::vector<int> idx(static_cast<size_t>(rule.size()));
    std::iota(idx.begin(), idx.end(), 0);
    std::vector<double> coef;
    node_coefs(rule, idx, p, coef);
    long long Es[3];
    for (int k = 0; k < op.d; ++k) Es[k] = static_cast<long long>(op.n[k]) * op.n[k];
    (void)s;
    (void)l;
    node_sweep(c, op, px.node, Es, rule.size(), nb, bs, p, &coef, out, 1, nullptr, 0, px.node_band);
    run_deferred(c);  // the late exponentials' side-stream work, now that the sweep is enqueued
}

void phi_fixed_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p, const NodesWeights& rule,
                   double* out) {
    std::vector<int> idx(static_cast<size_t>(rule.size()));
    std::iota(idx.begin(), idx.end(), 0);
    const PhiExps px = phi_exponentials(c, op, scale, 0, thetas_of(rule, idx), false, false, "nodeE");
    phi_fixed_shift(c, op, scale, 0, nb, bs, p, rule, px, out);
}

void phi_nodes_partial_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p,
                           const NodesWeights& rule, const std::vector<int>& nodes, int zero, double* acc) {
    const PhiExps px = phi_exponentials(c, op, scale, 0, thetas_of(rule, nodes), false, false, "nodeE");
    std::vector<double> coef;
    node_coefs(rule, nodes, p, coef);
    long long Es[3];
    for (int k = 0; k < op.d; ++k) Es[k] = static_cast<long long>(op.n[k]) * op.n[k];
    node_sweep(c, op, px.node, Es, static_cast<int>(nodes.size()), nb, bs, p, &coef, acc, zero, nullptr, 0,
               px.node_band);
}

// phiaction.hpp:156-245 (Alg. 2): nested CC ladder, node vectors kept in a device pool, all sums
// rebuilt in ascending node order at every level.  The first three levels (7 -> 13 -> 25 points)
// take their exponentials from `px25` (the 25-point rule's nodes, exponentiated in the call's
// single expm batch: CC nodes nest bitwise, so 7-rule node i is 25-rule node 4i); deeper levels
// exponentiate their fresh nodes on demand.
// A CC ladder whose convergence checks were deferred (phi_adaptive_shift with `pend`): the error
// statistics of levels 1..levels sit in c.h_small at stride 2*nb*p, complete once c.ev_cc fires.
// The speculation holds when every level but the last failed the test and the last passed it --
// exactly the levels the reference evaluates (phiaction.hpp:175-240).
struct CcPending {
    bool active = false;
    bool forked = false;  // the phi_0 fork event was recorded before the last level's combination
    int levels = 0, nb = 0, p = 0;
    double eps = 0.0;
};

static bool cc_pending_holds(pq_ctx& c, const CcPending& pd) {
    cuda_check(cudaEventSynchronize(c.ev_cc), "cc stats wait");
    mark(c, "cc_deferred_synced");
    const int w = 2 * pd.nb * pd.p;
    for (int lv = 0; lv < pd.levels; ++lv) {
        const volatile double* hs = c.h_small + static_cast<size_t>(lv) * w;
        double err = 0.0;
        for (int k = 0; k < pd.nb * pd.p; ++k) {
            const double diff = hs[2 * k], norm = hs[2 * k + 1];
            if (diff == 0.0) continue;
            err = std::max(err, norm == 0.0 ? std::numeric_limits<double>::infinity() : diff / norm);
        }
        const bool conv = err <= pd.eps;
        if (conv != (lv == pd.levels - 1)) return false;
    }
    return true;
}

static void phi_adaptive_shift(pq_ctx& c, const DevOp& op, double s, int l, int nb, const double* bs, int p,
                               double eps, const PhiExps& px25, double* out, int* points_used, int spec_points,
                               CcPending* pend = nullptr, cudaEvent_t fork_ev = nullptr) {
    if (p < 1) throw std::invalid_argument("phi_adaptive: need p >= 1");
    if (!(eps > 0.0)) throw std::invalid_argument("phi_adaptive: need eps > 0");
    const long long N = op.N;
    const size_t col = static_cast<size_t>(nb) * p * N;
    long long nn[3];
    for (int k = 0; k < op.d; ++k) nn[k] = static_cast<long long>(op.n[k]) * op.n[k];
    // The reference always evaluates the 13-point level before its first convergence test
    // (phiaction.hpp:175-240), so levels 0 and 1 are swept as ONE batch: the 13 nodes of the
    // 13-point rule (= 25-rule nodes 0, 2, ..., 24) into pool slots 0..12.  Per-node results do
    // not depend on the batch they are computed in, so this is bit-identical to two sweeps.
    int half = 3;
    const NodesWeights* rule = &memo_rule(kClenshaw, 2 * half + 1);
    std::vector<int> slot_of(static_cast<size_t>(rule->size()));
    for (int i = 0; i < rule->size(); ++i) slot_of[static_cast<size_t>(i)] = 2 * i;  // 7-rule i = 13-rule 2i
    int used = 13;
    double* pool = ws(c, "ccpool", static_cast<size_t>(used) * nb * N);
    {
        const double* E[3];
        long long Es[3];
        for (int k = 0; k < op.d; ++k) {
            E[k] = px25.node[k];
            Es[k] = 2 * nn[k];
        }
        node_sweep(c, op, E, Es, 13, nb, bs, p, nullptr, nullptr, 0, pool, 0, px25.node_band);
        run_deferred(c);  // the late exponentials' side-stream work, now that the sweep is enqueued
    }
    double* accs[2] = {out, ws(c, "ccacc", col)};
    int cur = 0;
    auto combine_all = [&](const NodesWeights& r, const std::vector<int>& slots, double* acc) {
        std::vector<int> idx(static_cast<size_t>(r.size()));
        std::iota(idx.begin(), idx.end(), 0);
        std::vector<double> coef;
        node_coefs(r, idx, p, coef);
        const double* coef_dev = static_cast<const double*>(arena_push(c, coef.data(), coef.size() * sizeof(double)));
        const int* sl_dev = static_cast<const int*>(arena_push(c, slots.data(), slots.size() * sizeof(int)));
        arena_flush(c);
        for (int m = 0; m < nb; ++m) {
            KernelProbe kp(c, "k_combine", 8.0 * N * (r.size() + p));
            launch_combine(N, p, r.size(), pool + static_cast<long long>(m) * N, static_cast<long long>(nb) * N, sl_dev,
                           coef_dev, acc + static_cast<long long>(m) * p * N, N, 1, c.stream);
            count_launch(c);
        }
    };
    // p <= 8: each level is one fused pass (combination + coarse rule + error statistics); the
    // 7-point result is only ever compared against, so it never goes to memory
    const bool fused = p <= 8;
    if (!fused) combine_all(*rule, slot_of, accs[cur]);
    double* stats = ws(c, "ccstats", 2 * static_cast<size_t>(nb) * p);
    std::vector<double> hstats(2 * static_cast<size_t>(nb) * p);
    int level = 0;
    // Fresh (odd) nodes of ladder level L >= 2 live in pool slots [base[L], base[L] + fresh).
    std::map<int, int> level_base;
    // Sweeps the fresh nodes of `lev` (rule `rl`) into the next free pool slots.
    auto sweep_level = [&](int lev, const NodesWeights& rl) {
        const int fr = rl.size() / 2;
        {
            DevBuf& b = c.bufs["ccpool"];
            const size_t want = static_cast<size_t>(used + fr) * nb * N * sizeof(double);
            if (b.bytes < want) {
                double* np = static_cast<double*>(ws_alloc(c, want, "ccpool"));
                cuda_check(cudaMemcpyAsync(np, b.p, static_cast<size_t>(used) * nb * N * sizeof(double),
                                           cudaMemcpyDeviceToDevice, c.stream),
                           "pool copy");
                ws_retire(c, b.p);
                b.p = np;
                b.bytes = want;
            }
            pool = static_cast<double*>(b.p);
        }
        std::vector<int> odd(static_cast<size_t>(fr));
        for (int k = 0; k < fr; ++k) odd[static_cast<size_t>(k)] = 2 * k + 1;
        const double* E[3];
        const int2* B[3] = {nullptr, nullptr, nullptr};
        long long Es[3];
        PhiExps pxl;
        if (lev == 2) {
            // 25-rule odd nodes 2k+1, exponentiated in the call's expm batch
            for (int k = 0; k < op.d; ++k) {
                E[k] = px25.node[k] + nn[k];
                Es[k] = 2 * nn[k];
                B[k] = px25.node_band[k] ? px25.node_band[k] + band_row_blocks(op.n[k]) : nullptr;
            }
        } else {
            pxl = phi_exponentials(c, op, s, l, thetas_of(rl, odd), false, false, "ccE" + std::to_string(lev));
            for (int k = 0; k < op.d; ++k) {
                E[k] = pxl.node[k];
                Es[k] = nn[k];
                B[k] = pxl.node_band[k];
            }
        }
        level_base[lev] = used;
        node_sweep(c, op, E, Es, fr, nb, bs, p, nullptr, nullptr, 0, pool, used, B);
        used += fr;
    };
    if (!c.ev_cc) cuda_check(cudaEventCreateWithFlags(&c.ev_cc, cudaEventDisableTiming), "cc event");
    const bool pinned_stats = 2 * nb * p <= 1024;
    // Deferred checks: when the planner predicts the converging level (spec_points), every level up
    // to it is enqueued without a host round trip -- each level's statistics go to their own slot of
    // the mapped readback -- and the caller enqueues the squaring and phi_0 before it checks them
    // (cc_pending_holds); a wrong prediction re-runs the call with the checks inline.
    int spec_levels = 0;
    if (spec_points > 0)
        for (int pts = 13;; pts = 2 * pts - 1) {
            ++spec_levels;
            if (pts >= spec_points) break;
        }
    const bool defer = pend && cc_defer_enabled() && spec_points > 0 && 2 * nb * p * spec_levels <= 1024;
    int dlev = 0;
    // a level whose combination runs on c.sq2 (while the speculative sweep of the next level runs
    // on the main stream): the main stream joins on ev_cc before it reads that level's sums
    bool join_pending = false;
    const cudaStream_t main_stream = c.stream;
    struct RestoreStream {  // an exception thrown while a level runs on c.sq2 leaves c.stream intact
        pq_ctx& c;
        cudaStream_t s;
        ~RestoreStream() { c.stream = s; }
    } restore{c, main_stream};
    while (true) {
        const int half_next = 2 * half;
        if (half_next > (1 << 14)) throw ConvergenceFailure("phi_adaptive: no convergence within the node budget");
        const NodesWeights& fine = memo_rule(kClenshaw, 2 * half_next + 1);
        const int fresh = fine.size() / 2;
        ++level;
        const bool preswept = level == 1;  // 13-point nodes already in slots 0..12
        if (!preswept && !level_base.count(level)) sweep_level(level, fine);
        std::vector<int> fine_slot(static_cast<size_t>(fine.size()));
        for (int i = 0; i < rule->size(); ++i) fine_slot[static_cast<size_t>(2 * i)] = slot_of[static_cast<size_t>(i)];
        for (int k = 0; k < fresh; ++k)
            fine_slot[static_cast<size_t>(2 * k + 1)] = preswept ? 2 * k + 1 : level_base[level] + k;
        const int nxt = 1 - cur;
        const int next_points = 2 * fine.size() - 1;
        const bool will_spec =
            pinned_stats && spec_points > 0 && next_points <= spec_points && 2 * half_next <= (1 << 14);
        if (join_pending) {
            cuda_check(cudaStreamWaitEvent(main_stream, c.ev_cc, 0), "cc join");
            join_pending = false;
        }
        const bool offload = fused && will_spec && !c.profiling;
        if (offload) {
            ensure_ccs(c);
            cuda_check(cudaEventRecord(c.ev_ccfork, main_stream), "cc fork");
            cuda_check(cudaStreamWaitEvent(c.ccs, c.ev_ccfork, 0), "cc fork wait");
            c.stream = c.ccs;
        }
        // deferred ladder, predicted last level: the side stream's phi_0 may start now, so its DMMA
        // work overlaps this level's (HBM-bound) combination instead of the squaring
        if (defer && fork_ev && fine.size() == spec_points && !offload) {
            cuda_check(cudaEventRecord(fork_ev, c.stream), "phi_0 fork");
            pend->forked = true;
        }
        // phiaction.hpp:225-240: max over columns of ||y - y_prev||_inf / ||y||_inf
        if (fused) {
            std::vector<int> idx(static_cast<size_t>(fine.size()));
            std::iota(idx.begin(), idx.end(), 0);
            std::vector<double> cf, cc;
            node_coefs(fine, idx, p, cf);
            const double* cf_dev = static_cast<const double*>(arena_push(c, cf.data(), cf.size() * sizeof(double)));
            const double* cc_dev = nullptr;
            if (level == 1) {  // coarse rule node k = fine node 2k
                std::vector<int> cidx(static_cast<size_t>(rule->size()));
                std::iota(cidx.begin(), cidx.end(), 0);
                std::vector<double> c7;
                node_coefs(*rule, cidx, p, c7);
                cc.assign(cf.size(), 0.0);
                for (int k = 0; k < rule->size(); ++k)
                    for (int j = 0; j < p; ++j)
                        cc[static_cast<size_t>(2 * k) * p + j] = c7[static_cast<size_t>(k) * p + j];
                cc_dev = static_cast<const double*>(arena_push(c, cc.data(), cc.size() * sizeof(double)));
            }
            const int* sl_dev = static_cast<const int*>(arena_push(c, fine_slot.data(), fine_slot.size() * sizeof(int)));
            arena_flush(c);
            cuda_check(cudaMemsetAsync(stats, 0, sizeof(double) * 2 * nb * p, c.stream), "cc stats zero");
            for (int m = 0; m < nb; ++m) {
                KernelProbe kp(c, "k_node_combine_ring", 8.0 * N * (fine.size() + p + (level == 1 ? 0 : p)));
                launch_combine_stats(N, p, fine.size(), pool + static_cast<long long>(m) * N, static_cast<long long>(nb) * N,
                                     sl_dev, cf_dev, cc_dev,
                                     level == 1 ? nullptr : accs[cur] + static_cast<long long>(m) * p * N,
                                     accs[nxt] + static_cast<long long>(m) * p * N, N, stats + 2 * m * p, c.stream);
                count_launch(c);
            }
        } else {
            combine_all(fine, fine_slot, accs[nxt]);
            KernelProbe kp(c, "k_colstats", 16.0 * N * nb * p);
            launch_colstats(N, nb * p, accs[nxt], accs[cur], stats, c.stream);
            count_launch(c);
        }
        half = half_next;
        rule = &fine;
        slot_of = std::move(fine_slot);
        if (pinned_stats) {  // mapped: stored by a kernel, no copy engine
            launch_store_words(stats, c.h_small_d + (defer ? static_cast<size_t>(dlev) * hstats.size() : 0),
                               hstats.size(), c.stream);
            count_launch(c);
        } else {
            cuda_check(cudaMemcpyAsync(hstats.data(), stats, hstats.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                       c.stream),
                       "cc stats readback");
        }
        cuda_check(cudaEventRecord(c.ev_cc, c.stream), "cc record");
        if (offload) {
            c.stream = main_stream;
            join_pending = true;
        }
        mark(c, "cc_level_enqueued");
        // Speculation: when the planner predicts the next level is needed (its rule has at most
        // spec_points nodes), its node sweep is enqueued before the host waits for this level's
        // error, so the GPU never drains at the check (a wasted sweep if this level converges).
        if (will_spec) sweep_level(level + 1, memo_rule(kClenshaw, next_points));
        if (defer) {
            ++dlev;
            cur = nxt;
            if (fine.size() < spec_points) continue;
            pend->active = true;
            pend->levels = dlev;
            pend->nb = nb;
            pend->p = p;
            pend->eps = eps;
            break;
        }
        cuda_check(cudaEventSynchronize(c.ev_cc), "cc stats wait");
        mark(c, "cc_level_synced");
        cur = nxt;
        const volatile double* hs = pinned_stats ? c.h_small : hstats.data();
        double err = 0.0;
        for (int k = 0; k < nb * p; ++k) {
            const double diff = hs[2 * k], norm = hs[2 * k + 1];
            if (diff == 0.0) continue;
            err = std::max(err, norm == 0.0 ? std::numeric_limits<double>::infinity() : diff / norm);
        }
        if (err <= eps) break;
    }
    if (join_pending) cuda_check(cudaStreamWaitEvent(main_stream, c.ev_cc, 0), "cc join");
    if (accs[cur] != out)
        cuda_check(cudaMemcpyAsync(out, accs[cur], col * sizeof(double), cudaMemcpyDeviceToDevice, c.stream), "cc copy");
    if (points_used) *points_used = rule->size();
}

void phi_adaptive_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p, double eps, double* out,
                      int* points_used) {
    const NodesWeights& r25 = memo_rule(kClenshaw, 25);
    const PhiExps px = phi_exponentials(c, op, scale, 0, r25.x, false, false, "nodeE");
    phi_adaptive_shift(c, op, scale, 0, nb, bs, p, eps, px, out, points_used, 0);
}

// phiaction.hpp:255-272 + 290-301: l doubling steps with E_k (= expm(2^-l A_k) on entry),
// squared after each step but the last.  y [nb][p][N] holds phi_j(2^-l A) b on entry; the
// result lands in y when l is even and in `partner` when l is odd (ping-pong, no copy).
// With sq_len >= l, E_in[k] already holds the chain E, E^2, ..., E^(2^(l-1)) (phi_exponentials
// sq_chain) and no matrix squaring is issued here.
// host_out (pinned, two-stream path only): each column half is copied to the host as soon as its
// last step is done; *copied reports whether that happened.
static double* squaring_pingpong(pq_ctx& c, const DevOp& op, int l, int nb, int p, double* y, double* partner,
                                 const double* const* E_in, int sq_len = 1, const int2* const* band_in = nullptr,
                                 double* host_out = nullptr, bool* copied = nullptr) {
    if (l <= 0) return y;
    const long long N = op.N;
    const bool chain = sq_len >= l;
    // Distinct exponentials grouped by size, copied into contiguous ping-pong slots so each
    // step's E <- E E is one batched DMMA launch per size (dims sharing an exponential share it).
    struct Group {
        int n = 0;
        std::vector<int> dims;  // first dim of each distinct exponential
        double* buf = nullptr;  // [2][count][n*n]
    };
    std::vector<Group> groups;
    int slot_dim[3] = {-1, -1, -1};  // k -> (group, index)
    int slot_idx[3] = {0, 0, 0};
    for (int k = 0; k < op.d && !chain; ++k) {
        int same = -1;
        for (int j = 0; j < k; ++j)
            if (E_in[j] == E_in[k]) same = j;
        if (same >= 0) {
            slot_dim[k] = slot_dim[same];
            slot_idx[k] = slot_idx[same];
            continue;
        }
        int gi = -1;
        for (size_t g = 0; g < groups.size(); ++g)
            if (groups[g].n == op.n[k]) gi = static_cast<int>(g);
        if (gi < 0) {
            groups.push_back(Group{op.n[k], {}, nullptr});
            gi = static_cast<int>(groups.size()) - 1;
        }
        slot_dim[k] = gi;
        slot_idx[k] = static_cast<int>(groups[static_cast<size_t>(gi)].dims.size());
        groups[static_cast<size_t>(gi)].dims.push_back(k);
    }
    for (size_t g = 0; g < groups.size(); ++g) {
        Group& G = groups[g];
        const size_t nn = static_cast<size_t>(G.n) * G.n;
        G.buf = ws(c, "sqE" + std::to_string(g), 2 * G.dims.size() * nn);
        for (size_t i = 0; i < G.dims.size(); ++i) dev_copy(c, G.buf + i * nn, E_in[G.dims[i]], nn, c.stream);
    }
    int parity = 0;
    auto cur_E = [&](int k) {
        const Group& G = groups[static_cast<size_t>(slot_dim[k])];
        const size_t nn = static_cast<size_t>(G.n) * G.n;
        return G.buf + (static_cast<size_t>(parity) * G.dims.size() + slot_idx[k]) * nn;
    };
    // combination table: coef[i][j] = 2^-(i+1) / (i-j)!  (inverse_factorials, phiaction.hpp:58-66)
    std::vector<double> inv(static_cast<size_t>(p), 1.0);
    {
        double f = 1.0;
        for (int k = 1; k < p; ++k) {
            f *= k;
            inv[static_cast<size_t>(k)] = 1.0 / f;
        }
    }
    std::vector<double> coef(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j <= i; ++j)
            coef[static_cast<size_t>(i) * p + j] = std::ldexp(1.0, -(i + 1)) * inv[static_cast<size_t>(i - j)];
    const double* coef_dev = static_cast<const double*>(arena_push(c, coef.data(), coef.size() * sizeof(double)));
    const int Z1 = nb * p;
    // The combination fused into the last mode product's epilogue (PQ_SQ_FUSE=1; default off):
    // column z1 (i = z1 mod p) = 2^-(i+1) acc + sum_{j <= i} coef[i][j] b_j, with the same
    // roundings in the same order as k_sq_combine2 (bitwise identical results, checked with
    // tools/bitwise_env_ab.py).  Measured at config 2: 461.7 vs 461-471 actions/s -- the k-major
    // last-mode tiles (6 CTAs/SM, 80 registers) read the i + 1 addend columns term by term in
    // their epilogue (645 us per call vs 340 us + 237 us for the separate streaming combination,
    // which loads each b_j once for all columns i >= j).
    static const bool fuse = [] {
        const char* e = std::getenv("PQ_SQ_FUSE");
        return e && std::atoi(e) != 0;
    }();
    Epilogue fused{};
    if (fuse) {
        std::vector<double> alpha(static_cast<size_t>(Z1)), rows(static_cast<size_t>(Z1) * p, 0.0);
        std::vector<int> nterms(static_cast<size_t>(Z1));
        for (int z = 0; z < Z1; ++z) {
            const int i = z % p;
            alpha[static_cast<size_t>(z)] = std::ldexp(1.0, -(i + 1));
            nterms[static_cast<size_t>(z)] = i + 1;
            for (int j = 0; j <= i; ++j) rows[static_cast<size_t>(z) * p + j] = coef[static_cast<size_t>(i) * p + j];
        }
        fused.alpha_z = static_cast<const double*>(arena_push(c, alpha.data(), alpha.size() * sizeof(double)));
        fused.coef = static_cast<const double*>(arena_push(c, rows.data(), rows.size() * sizeof(double)));
        fused.nterms = static_cast<const int*>(arena_push(c, nterms.data(), nterms.size() * sizeof(int)));
        fused.cld = p;  // = ext_group: batch z1 reads addends (z1 / p) p + t, its own right-hand side's
        fused.ext_s = N;
    }
    auto fused_at = [&](const double* cur, int c0) {
        Epilogue e = fused;
        e.ext = cur;
        e.alpha_z += c0;
        e.coef += static_cast<size_t>(c0) * p;
        e.nterms += c0;
        return e;
    };
    arena_flush(c);
    long long Es[3] = {0, 0, 0};
    if (chain && squaring_split_ok(c, nb, p, N)) {
        // Column groups on their own streams, R rotating buffers b_s (step s reads b_s, writes
        // b_{s+1}).  Column i of step s needs columns j <= i of step s-1 (phiaction.hpp:260-268), so
        // group g's combination of step s waits for every lower group's combination of step s-1,
        // and group g's chain of step s overwrites b_{s+1} = b_{s+1-R}, last read by the higher
        // groups' combinations of step s+1-R.  Everything else is ordered within a stream, so one
        // group's bandwidth-bound combination runs under the others' DMMA chains.
        //  * device-resident: two halves, lower on the context stream, upper on c.sq2, R = 3;
        //  * pinned host results (squaring_ring > 3): groups on helper streams with descending
        //    priority and no buffer reuse, so the lowest columns finish first and their D2H runs
        //    under the later columns.  Two groups by default; PQ_SQ_GROUPS=3|4 splits further (one
        //    column per group at p = 4: same e2e within noise, twice the launches).
        const int R = squaring_ring(nb, p, N, l, host_out != nullptr);
        const bool cascade = host_out != nullptr && R > 3;
        static const int max_groups = [] {
            const char* e = std::getenv("PQ_SQ_GROUPS");
            return e ? std::max(2, std::min(4, std::atoi(e))) : 2;
        }();
        const int G = cascade ? std::min(p, max_groups) : 2;
        std::vector<int> lo(static_cast<size_t>(G) + 1);
        for (int g = 0; g <= G; ++g) lo[static_cast<size_t>(g)] = cascade ? (g * p) / G : (g == 0 ? 0 : g == 1 ? p / 2 : p);
        double* scratch = ws(c, "sq3", static_cast<size_t>(R - 2) * p * N);
        std::vector<double*> b(static_cast<size_t>(R), nullptr);
        b[0] = y;
        // b_(l mod R) is `partner` when l mod R != 0 (the caller's output then); for l mod R == 0
        // the result lands in y.  The other slots are scratch.
        const int fin = (l % R == 0) ? 1 : l % R;
        b[static_cast<size_t>(fin)] = partner;
        for (int r = 1, k = 0; r < R; ++r)
            if (r != fin) b[static_cast<size_t>(r)] = scratch + static_cast<size_t>(k++) * p * N;
        ensure_sq2(c);
        if (cascade) ensure_sq_cascade(c, G);
        while (static_cast<int>(c.ev_sqg.size()) < G * l) {
            cudaEvent_t e;
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "sq event");
            c.ev_sqg.push_back(e);
        }
        auto ev = [&](int g, int st) { return c.ev_sqg[static_cast<size_t>(st) * G + g]; };
        const cudaStream_t main_stream = c.stream;
        std::vector<cudaStream_t> gs(static_cast<size_t>(G));
        for (int g = 0; g < G; ++g)
            gs[static_cast<size_t>(g)] = cascade ? c.sqs[static_cast<size_t>(g)] : (g == 0 ? main_stream : c.sq2);
        cuda_check(cudaEventRecord(c.ev_sqfork, main_stream), "sq fork");
        for (int g = 0; g < G; ++g)
            if (gs[static_cast<size_t>(g)] != main_stream)
                cuda_check(cudaStreamWaitEvent(gs[static_cast<size_t>(g)], c.ev_sqfork, 0), "sq fork wait");
        static const char* tags[4] = {"sqch0", "sqch1", "sqch2", "sqch3"};
        try {
            for (int step = 0; step < l; ++step) {
                const double* E[3];
                const int2* Bd[3] = {nullptr, nullptr, nullptr};
                for (int k = 0; k < op.d; ++k) {
                    E[k] = E_in[k] + static_cast<size_t>(step) * op.n[k] * op.n[k];
                    if (band_in && band_in[k]) Bd[k] = band_in[k] + step * band_row_blocks(op.n[k]);
                }
                double* cur = b[static_cast<size_t>(step % R)];
                double* nxt = b[static_cast<size_t>((step + 1) % R)];
                for (int g = 0; g < G; ++g) {
                    const int c0 = lo[static_cast<size_t>(g)], c1 = lo[static_cast<size_t>(g) + 1];
                    c.stream = gs[static_cast<size_t>(g)];
                    if (step + 1 >= R)
                        for (int h = g + 1; h < G; ++h)
                            cuda_check(cudaStreamWaitEvent(c.stream, ev(h, step + 1 - R), 0), "sq wait (reuse)");
                    // the combination reads columns j < c0 of this step's input: the lower groups'
                    // results of the previous step
                    auto lower_done = [&] {
                        if (step >= 1)
                            for (int h = 0; h < g; ++h)
                                cuda_check(cudaStreamWaitEvent(c.stream, ev(h, step - 1), 0), "sq wait (columns)");
                    };
                    if (fuse) {
                        mode_chain(c, op.d, op.n, E, Es, cur + static_cast<size_t>(c0) * N, N,
                                   nxt + static_cast<size_t>(c0) * N, N, c1 - c0, fused_at(cur, c0), tags[g], Bd,
                                   lower_done);
                    } else {
                        mode_chain(c, op.d, op.n, E, Es, cur + static_cast<size_t>(c0) * N, N,
                                   nxt + static_cast<size_t>(c0) * N, N, c1 - c0, Epilogue{}, tags[g], Bd);
                        lower_done();
                        KernelProbe kp(c, "k_sq_combine2", 8.0 * N * (2 * (c1 - c0) + c1));
                        launch_sq_combine(N, p, 1, nxt, cur, coef_dev, c.stream, c0, c1);
                        count_launch(c);
                    }
                    cuda_check(cudaEventRecord(ev(g, step), c.stream), "sq rec");
                }
            }
        } catch (...) {
            c.stream = main_stream;
            throw;
        }
        c.stream = main_stream;
        const double* res = b[static_cast<size_t>(l % R)];
        for (int g = 0; g < G; ++g) {
            const int c0 = lo[static_cast<size_t>(g)], c1 = lo[static_cast<size_t>(g) + 1];
            const cudaStream_t st = gs[static_cast<size_t>(g)];
            c.stream = st;
            mark(c, "sq_group_done");
            if (host_out) {  // this group's columns are final on its stream now
                gate_point(c, st);
                cuda_check(cudaMemcpyAsync(host_out + static_cast<size_t>(c0) * N, res + static_cast<size_t>(c0) * N,
                                           sizeof(double) * (c1 - c0) * N, cudaMemcpyDeviceToHost, st),
                           "phi columns D2H");
                note_early_copy(c, st, host_out + static_cast<size_t>(c0) * N, static_cast<size_t>(c1 - c0) * N);
                mark(c, "sq_group_copied");
            }
            c.stream = main_stream;
            if (st != main_stream) {
                cuda_check(cudaEventRecord(ev(g, l - 1), st), "sq rec (final)");
                cuda_check(cudaStreamWaitEvent(main_stream, ev(g, l - 1), 0), "sq join");
            }
        }
        if (host_out && copied) *copied = true;
        if (host_out) c.gate_covered = true;  // (only copies follow on the context stream)
        check_launch(c);
        return b[static_cast<size_t>(l % R)];
    }
    double* cur = y;
    double* nxt = partner;
    for (int step = 0; step < l; ++step) {
        const double* E[3];
        const int2* Bd[3] = {nullptr, nullptr, nullptr};
        for (int k = 0; k < op.d; ++k) {
            E[k] = chain ? E_in[k] + static_cast<size_t>(step) * op.n[k] * op.n[k] : cur_E(k);
            if (chain && band_in && band_in[k]) Bd[k] = band_in[k] + step * band_row_blocks(op.n[k]);
        }
        if (fuse) {
            mode_chain(c, op.d, op.n, E, Es, cur, N, nxt, N, Z1, fused_at(cur, 0), "chain", Bd);
        } else {
            mode_chain(c, op.d, op.n, E, Es, cur, N, nxt, N, Z1, Epilogue{}, "chain", Bd);
            KernelProbe kp(c, "k_sq_combine2", 8.0 * N * nb * 3 * p);
            launch_sq_combine(N, p, nb, nxt, cur, coef_dev, c.stream);
            count_launch(c);
        }
        std::swap(cur, nxt);
        if (step < l - 1 && !chain) {
            for (const Group& G : groups) {
                const size_t nn = static_cast<size_t>(G.n) * G.n;
                const int cnt = static_cast<int>(G.dims.size());
                double* src = G.buf + static_cast<size_t>(parity) * cnt * nn;
                double* dst = G.buf + static_cast<size_t>(1 - parity) * cnt * nn;
                {
                    GemmArgs sb = square_batch(G.n, cnt, src, src, dst);
                    sb.tag = "sq_E^2";
                    gemm(c, sb);
                }
            }
            parity = 1 - parity;
        }
    }
    check_launch(c);
    return cur;
}

void squaring_steps_dev(pq_ctx& c, const DevOp& op, double scale, int nb, int p, int l, double* y,
                        const double* exps_override) {
    double* partner = ws(c, "sqT", static_cast<size_t>(nb) * p * op.N);
    const double* E[3] = {nullptr, nullptr, nullptr};
    if (exps_override) {
        size_t off = 0;
        for (int k = 0; k < op.d; ++k) {
            E[k] = exps_override + off;
            off += static_cast<size_t>(op.n[k]) * op.n[k];
        }
    } else {
        const PhiExps px = phi_exponentials(c, op, scale, l, {}, true, false, "sqE0");
        for (int k = 0; k < op.d; ++k) E[k] = px.sq[k];
    }
    double* res = squaring_pingpong(c, op, l, nb, p, y, partner, E);
    if (res != y)
        cuda_check(cudaMemcpyAsync(y, res, sizeof(double) * nb * p * op.N, cudaMemcpyDeviceToDevice, c.stream), "sq copy");
}

// phiaction.hpp:277-303, plus (when phi0_out) kron.hpp:123-128 phi_0 from the same expm batch.
static void phi_call_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p, int l, int n,
                         int kind, double eps, double* out, int* points_used, double* phi0_out,
                         double* phi0_host = nullptr, double* out_host = nullptr, bool* out_copied = nullptr,
                         bool allow_defer = true) {
    if (l < 0) throw std::invalid_argument("phi_with_plan: need l >= 0");
    if (p < 1) throw std::invalid_argument(kind == kGauss ? "phi_fixed: need p >= 1" : "phi_adaptive: need p >= 1");
    const NodesWeights& rule = kind == kGauss ? memo_rule(kGauss, n + 1) : memo_rule(kClenshaw, 25);
    CcPending pend;
    // squaring chain and phi_0 exponentials are finished on the side stream during the node sweep
    // (not while profiling, so per-launch events stay unambiguous)
    const PhiExps px = phi_exponentials(c, op, scale, l, rule.x, l > 0, phi0_out != nullptr, "nodeE", true,
                                        !c.profiling);
    mark(c, "exps");
    double* partner = l > 0 ? ws(c, "sqT", static_cast<size_t>(nb) * p * op.N) : nullptr;
    // the squaring then ends in `out`: ping-pong (l odd: start in partner), or the two-stream
    // three-buffer rotation (l mod 3 != 0: start in partner, squaring_pingpong rotates into out)
    const bool split_sq = l > 0 && px.sq_len >= l && squaring_split_ok(c, nb, p, op.N);
    const int ring = squaring_ring(nb, p, op.N, l, out_host != nullptr);
    double* first = split_sq ? ((l % ring == 0) ? out : partner) : ((l % 2 == 1) ? partner : out);
    if (kind == kGauss) {
        phi_fixed_shift(c, op, scale, l, nb, bs, p, rule, px, first);
        if (points_used) *points_used = rule.size();
    } else {
        // the planner's node parameter predicts the ladder level that converges: speculate up to
        // the first CC rule with at least n + 1 points (the plan's Gauss-equivalent count)
        int spec = 0;
        if (n > 0) {
            spec = 13;
            while (spec < n + 1 && spec < (1 << 15)) spec = 2 * spec - 1;
        }
        if (phi0_out && l > 0 && !c.profiling) ensure_side(c);
        phi_adaptive_shift(c, op, scale, l, nb, bs, p, eps, px, first, points_used, spec, allow_defer ? &pend : nullptr,
                           phi0_out && l > 0 && !c.profiling ? c.ev_fork : nullptr);
    }
    mark(c, "nodes");
    // phi_0 needs only its exponentials and b: run its mode chain on the side stream alongside the
    // last CC level's combination (deferred ladder) or the squaring chain, where its CTAs fill the
    // tails of the squaring GEMM waves (not while profiling, so per-launch events stay unambiguous)
    const bool side_phi0 = phi0_out && l > 0 && !c.profiling;
    if (side_phi0) {
        ensure_side(c);
        if (!pend.forked) cuda_check(cudaEventRecord(c.ev_fork, c.stream), "fork");
        cuda_check(cudaStreamWaitEvent(c.side, c.ev_fork, 0), "fork wait");
        cudaStream_t main_stream = c.stream;
        c.stream = c.side;
        try {
            apply_phi0(c, op, px, nb, bs, phi0_out);
            if (phi0_host) {  // pinned destination: the D2H overlaps the squaring
                gate_point(c, c.side);
                cuda_check(cudaMemcpyAsync(phi0_host, phi0_out, sizeof(double) * nb * op.N, cudaMemcpyDeviceToHost, c.side),
                           "phi_0 D2H");
                note_early_copy(c, c.side, phi0_host, static_cast<size_t>(nb) * op.N);
            }
        } catch (...) {
            c.stream = main_stream;
            throw;
        }
        c.stream = main_stream;
        cuda_check(cudaEventRecord(c.ev_join, c.side), "join record");
    }
    run_deferred(c);  // (no-op unless the node phase did not flush it)
    if (px.late) cuda_check(cudaStreamWaitEvent(c.stream, c.ev_late, 0), "late exps wait");
    if (l > 0) {
        double* res = squaring_pingpong(c, op, l, nb, p, first, first == out ? partner : out, px.sq, px.sq_len,
                                        px.sq_band, split_sq ? out_host : nullptr, out_copied);
        if (res != out)
            cuda_check(cudaMemcpyAsync(out, res, sizeof(double) * nb * p * op.N, cudaMemcpyDeviceToDevice, c.stream),
                       "plan copy");
    }
    mark(c, "squaring");
    if (side_phi0) {
        cuda_check(cudaStreamWaitEvent(c.stream, c.ev_join, 0), "join wait");
    } else if (phi0_out) {
        apply_phi0(c, op, px, nb, bs, phi0_out);
        if (phi0_host)
            cuda_check(cudaMemcpyAsync(phi0_host, phi0_out, sizeof(double) * nb * op.N, cudaMemcpyDeviceToHost, c.stream),
                       "phi_0 D2H");
    }
    if (pend.active) {
        // the ladder's deferred checks: everything above is enqueued, so the GPU keeps running
        // while the host reads the levels' statistics
        if (cc_pending_holds(c, pend)) {
            ++c.cc_defer_hits;
        } else {
            ++c.cc_defer_misses;
            // drain this run (its early host copies included) before the re-run writes the same buffers
            for (cudaStream_t st : {c.stream, c.side, c.sq2, c.ccs})
                if (st) cuda_check(cudaStreamSynchronize(st), "cc re-run drain");
            for (cudaStream_t st : c.sqs) cuda_check(cudaStreamSynchronize(st), "cc re-run drain");
            c.early.clear();  // this run's early host copies are superseded
            if (out_copied) *out_copied = false;
            phi_call_dev(c, op, scale, nb, bs, p, l, n, kind, eps, out, points_used, phi0_out, phi0_host, out_host,
                         out_copied, false);
        }
    }
}

void phi_with_plan_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p, int l, int n, int kind,
                       double eps, double* out, int* points_used) {
    phi_call_dev(c, op, scale, nb, bs, p, l, n, kind, eps, out, points_used, nullptr);
}

// phiaction.hpp:307-346 (+ phi_0 when phi0_out).
// beta = max ||b||_inf: reduced on the device and read back into pinned c.h_beta on ev_beta
// (nb <= 512); larger batches reduce synchronously and return beta directly (>= 0 then).
static double beta_enqueue(pq_ctx& c, const DevOp& op, int nb, const double* bs) {
    if (nb > 512) return max_inf_norm_dev(c, bs, op.N, nb);
    if (nb <= 0) return 0.0;
    double* stats = ws(c, "colstats", 2 * static_cast<size_t>(nb));
    launch_colstats(op.N, nb, bs, nullptr, stats, c.stream);
    count_launch(c);
    if (!c.ev_beta) cuda_check(cudaEventCreateWithFlags(&c.ev_beta, cudaEventDisableTiming), "beta event");
    launch_store_words(stats, c.h_beta_d, 2 * static_cast<size_t>(nb), c.stream);  // (mapped: no copy engine)
    count_launch(c);
    cuda_check(cudaEventRecord(c.ev_beta, c.stream), "beta record");
    return -1.0;
}

// waits for the readback (any thread) and reduces the per-column maxima
static double beta_collect(pq_ctx& c, int nb) {
    cuda_check(cudaEventSynchronize(c.ev_beta), "beta wait");
    double beta = 0.0;
    for (int m = 0; m < nb; ++m) beta = std::max(beta, c.h_beta[2 * m + 1]);
    return beta;
}

// phiaction.hpp:312-340 on the host: setup_quadrature (or quadnodes at a pinned l)
static PlanInfo plan_host(int d, double alpha, double beta, int p, double eps, int mode, bool has_l, int l, double c1,
                          double c2) {
    Cost cost{c1, c2, d};
    PlanInfo info;
    int n = 0;
    bool planned = false;
    double plan_cost = 0.0;
    if (has_l) {
        if (l < 0) throw std::invalid_argument("phiquadmv: need l >= 0");
        if (alpha > 0.0 && beta > 0.0)
            n = node_count(eps, p, std::ldexp(alpha, -l), beta, mode);
        else
            n = mode == kGauss ? 2 : 4;
        plan_cost = cost(n, l, p);
    } else if (alpha > 0.0 && beta > 0.0) {
        const Plan pl = plan_quadrature(eps, p, alpha, beta, mode, cost);
        l = pl.l;
        n = pl.n;
        plan_cost = pl.cost;
        planned = true;
    } else {
        l = 0;
        n = mode == kGauss ? 2 : 4;
        plan_cost = cost(n, l, p);
        planned = true;
    }
    info.l = l;
    info.n = n;
    info.mode = mode;
    info.planned = planned ? 1 : 0;
    info.alpha = alpha;
    info.beta = beta;
    info.cost = plan_cost;
    return info;
}

static double alpha_of(const DevOp& op) {
    double alpha = 0.0;
    for (int k = 0; k < op.d; ++k) alpha += op.inf_norm[k];
    return alpha;
}

PlanInfo plan_phi(pq_ctx& c, const DevOp& op, int nb, const double* bs, int p, double eps, int mode, bool has_l, int l,
                  double c1, double c2) {
    if (p < 1) throw std::invalid_argument("phiquadmv: need p >= 1");
    double beta = beta_enqueue(c, op, nb, bs);
    // the exponentials' shared Taylor powers do not depend on the plan: enqueue them before the
    // host waits for beta, so the GPU computes them while the host plans
    taylor_prefetch(c, op, 1.0);
    if (beta < 0.0) beta = beta_collect(c, nb);
    mark(c, "beta_ready");
    const PlanInfo info = plan_host(op.d, alpha_of(op), beta, p, eps, mode, has_l, l, c1, c2);
    mark(c, "planned");
    return info;
}

// ---- planner worker thread ----
void worker_submit(pq_ctx& c, std::function<void()> job) {
    if (!c.worker) {
        c.worker = std::make_unique<pq_ctx::Worker>();
        pq_ctx::Worker* w = c.worker.get();
        w->th = std::thread([w] {
            std::unique_lock<std::mutex> lk(w->mu);
            while (true) {
                w->cv.wait(lk, [w] { return w->has_job || w->stop; });
                if (w->stop) return;
                std::function<void()> f = std::move(w->job);
                w->has_job = false;
                lk.unlock();
                std::exception_ptr err;
                try {
                    f();
                } catch (...) {
                    err = std::current_exception();
                }
                lk.lock();
                w->err = err;
                w->busy = false;
                w->cv.notify_all();
            }
        });
    }
    pq_ctx::Worker* w = c.worker.get();
    std::lock_guard<std::mutex> lk(w->mu);
    w->job = std::move(job);
    w->has_job = true;
    w->busy = true;
    w->err = nullptr;
    w->cv.notify_all();
}

void worker_wait(pq_ctx& c) {
    if (!c.worker) return;
    pq_ctx::Worker* w = c.worker.get();
    std::unique_lock<std::mutex> lk(w->mu);
    w->cv.wait(lk, [w] { return !w->busy; });
    if (w->err) {
        std::exception_ptr e = w->err;
        w->err = nullptr;
        std::rethrow_exception(e);
    }
}

void worker_stop(pq_ctx& c) {
    if (!c.worker) return;
    {
        std::lock_guard<std::mutex> lk(c.worker->mu);
        c.worker->stop = true;
        c.worker->cv.notify_all();
    }
    if (c.worker->th.joinable()) c.worker->th.join();
    c.worker.reset();
}

static bool plan_spec_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PQ_PLAN_SPEC");
        return !(v && v[0] == '0');
    }();
    return on;
}

void phiquadmv_dev(pq_ctx& c, const DevOp& op, int nb, const double* bs, int p, double eps, int mode, bool has_l, int l,
                   double c1, double c2, double* out, PlanInfo* info, double* phi0_out, double* phi0_host,
                   double* out_host, bool* out_copied) {
    if (p < 1) throw std::invalid_argument("phiquadmv: need p >= 1");
    // the last plan for this operator (bit-identical factors share the cached host copy) and request
    pq_ctx::PlanMemo* memo = nullptr;
    for (auto& m : c.plan_memo)
        if (m.host == op.host && m.p == p && m.mode == mode && m.has_l == (has_l ? 1 : 0) && m.l_in == (has_l ? l : 0) &&
            m.eps == eps && m.c1 == c1 && m.c2 == c2)
            memo = &m;
    const bool spec = memo && plan_spec_enabled() && nb > 0 && nb <= 512 && !c.profiling;
    PlanInfo pi;
    int points = 0;
    if (!spec) {
        pi = plan_phi(c, op, nb, bs, p, eps, mode, has_l, l, c1, c2);
        phi_call_dev(c, op, 1.0, nb, bs, p, pi.l, pi.n, mode, eps, out, &points, phi0_out, phi0_host, out_host,
                     out_copied);
    } else {
        // speculation: the pipeline with the remembered plan is enqueued while the worker thread
        // waits for beta and plans; the GPU never idles for the host planner
        const int sl = memo->l, sn = memo->n;
        beta_enqueue(c, op, nb, bs);
        mark(c, "beta_enqueued");
        const double alpha = alpha_of(op);
        const int d = op.d;
        worker_submit(c, [&c, &pi, nb, d, alpha, p, eps, mode, has_l, l, c1, c2] {
            pi = plan_host(d, alpha, beta_collect(c, nb), p, eps, mode, has_l, l, c1, c2);
        });
        // the shared Taylor powers depend on the operator only: enqueue them before the host builds
        // the rest of the call (phi_exponentials finds them cached); after the planner job, which
        // is on the critical path of latency-bound calls (config 1)
        taylor_prefetch(c, op, 1.0);
        try {
            phi_call_dev(c, op, 1.0, nb, bs, p, sl, sn, mode, eps, out, &points, phi0_out, phi0_host, out_host,
                         out_copied);
        } catch (...) {
            try {
                worker_wait(c);
            } catch (...) {
            }
            throw;
        }
        worker_wait(c);
        mark(c, "planned");
        // for the adaptive CC rule n only sets the ladder speculation depth, not the result
        if (pi.l != sl || (mode == kGauss && pi.n != sn)) {
            ++c.plan_spec_misses;
            c.early.clear();  // the speculative run's early host copies are superseded
            if (out_copied) *out_copied = false;
            phi_call_dev(c, op, 1.0, nb, bs, p, pi.l, pi.n, mode, eps, out, &points, phi0_out, phi0_host, out_host,
                         out_copied);
        } else {
            ++c.plan_spec_hits;
        }
    }
    if (!memo) {
        c.plan_memo.push_back({});
        memo = &c.plan_memo.back();
        if (c.plan_memo.size() > 16) {
            c.plan_memo.erase(c.plan_memo.begin());
            memo = &c.plan_memo.back();
        }
    }
    *memo = pq_ctx::PlanMemo{op.host, p, mode, has_l ? 1 : 0, has_l ? l : 0, eps, c1, c2, pi.l, pi.n};
    pi.points = points;
    if (info) *info = pi;
}

// phiaction.hpp:355-389: one sweep of the combined integrand sum_j theta^{j-1}/(j-1)! b_j.
void phi_lincomb_dev(pq_ctx& c, const DevOp& op, double scale, int p, const double* bs, const NodesWeights& rule,
                     double* out) {
    if (p < 1) throw std::invalid_argument("phi_lincomb: need at least one vector");
    const int q = rule.size();
    const long long N = op.N;
    const PhiExps px = phi_exponentials(c, op, scale, 0, rule.x, false, false, "lincE");
    long long Es[3];
    for (int k = 0; k < op.d; ++k) Es[k] = static_cast<long long>(op.n[k]) * op.n[k];
    // mixing coefficients per node (coeff = 1, coeff *= theta/j) and final weights
    std::vector<double> mix(static_cast<size_t>(q) * p), wts(static_cast<size_t>(q));
    for (int i = 0; i < q; ++i) {
        double coeff = 1.0;
        for (int j = 1; j <= p; ++j) {
            mix[static_cast<size_t>(i) * p + j - 1] = coeff;
            coeff *= rule.x[static_cast<size_t>(i)] / j;
        }
        wts[static_cast<size_t>(i)] = rule.w[static_cast<size_t>(i)];
    }
    std::vector<int> bslots(static_cast<size_t>(p)), vslots(static_cast<size_t>(q));
    std::iota(bslots.begin(), bslots.end(), 0);
    std::iota(vslots.begin(), vslots.end(), 0);
    const double* mix_dev = static_cast<const double*>(arena_push(c, mix.data(), mix.size() * sizeof(double)));
    const double* w_dev = static_cast<const double*>(arena_push(c, wts.data(), wts.size() * sizeof(double)));
    const int* bsl = static_cast<const int*>(arena_push(c, bslots.data(), bslots.size() * sizeof(int)));
    const int* vsl = static_cast<const int*>(arena_push(c, vslots.data(), vslots.size() * sizeof(int)));
    arena_flush(c);
    const int qc = node_chunk(c, N, q, 4);
    double* M = ws(c, "lincMix", static_cast<size_t>(qc) * N);
    double* V = ws(c, "lincV", static_cast<size_t>(qc) * N);
    // mixing coefficients transposed per group of <= 8 nodes: input j, output node a -> [j][a - g0]
    constexpr int kMixOut = 8;
    std::vector<double> mixT;
    std::vector<size_t> mix_off;
    for (int g0 = 0; g0 < q; g0 += kMixOut) {
        const int gc = std::min(kMixOut, q - g0);
        mix_off.push_back(mixT.size());
        for (int j = 0; j < p; ++j)
            for (int a = 0; a < gc; ++a) mixT.push_back(mix[static_cast<size_t>(g0 + a) * p + j]);
    }
    const double* mixT_dev = static_cast<const double*>(arena_push(c, mixT.data(), mixT.size() * sizeof(double)));
    arena_flush(c);
    for (int a0 = 0; a0 < q; a0 += qc) {
        const int cnt = std::min(qc, q - a0);
        // mix_a = sum_j c_aj b_j (ascending j) for up to 8 nodes per streaming pass: the p inputs
        // are read once per group instead of once per node
        for (int a = 0; a < cnt;) {
            const int node = a0 + a, g = node / kMixOut, in_g = node % kMixOut;
            const int gc = std::min(kMixOut, q - g * kMixOut);
            const int take = std::min(gc - in_g, cnt - a);
            if (in_g == 0 && take == gc) {
                KernelProbe kp(c, "k_combine(lincomb mix)", 8.0 * N * (p + gc));
                launch_combine(N, gc, p, bs, N, bsl, mixT_dev + mix_off[static_cast<size_t>(g)], M + static_cast<long long>(a) * N,
                               N, 1, c.stream);
                count_launch(c);
            } else {
                for (int t = 0; t < take; ++t) {  // a chunk boundary inside a group: one node at a time
                    KernelProbe kp(c, "k_combine(lincomb mix)", 8.0 * N * (p + 1));
                    launch_combine(N, 1, p, bs, N, bsl, mix_dev + static_cast<size_t>(node + t) * p,
                                   M + static_cast<long long>(a + t) * N, N, 1, c.stream);
                    count_launch(c);
                }
            }
            a += take;
        }
        const double* Ec[3];
        const int2* Bc[3];
        for (int k = 0; k < op.d; ++k) {
            Ec[k] = px.node[k] + a0 * Es[k];
            Bc[k] = px.node_band[k] ? px.node_band[k] + a0 * band_row_blocks(op.n[k]) : nullptr;
        }
        mode_chain(c, op.d, op.n, Ec, Es, M, N, V, N, cnt, Epilogue{}, "chain", Bc);
        KernelProbe kp(c, "k_combine(lincomb nodes)", 8.0 * N * (cnt + 1 + (a0 == 0 ? 0 : 1)));
        launch_combine(N, 1, cnt, V, N, vsl, w_dev + a0, out, N, a0 == 0 ? 1 : 0, c.stream);
        count_launch(c);
    }
    check_launch(c);
}

}  // namespace pqb
