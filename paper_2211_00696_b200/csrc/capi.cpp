// The extern "C" boundary (include/pq_b200.h): argument checks with the reference's messages,
// host<->device staging for PQ_HOST calls, and exception -> return-code mapping.  No entry point
// has a CPU fallback; without an sm_100 device, context creation fails.
#include "pq_b200.h"

#include <cmath>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

using namespace pqb;

namespace pqb {
std::string& last_error_slot() {
    thread_local std::string msg;
    return msg;
}
}  // namespace pqb

namespace {

void need(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(what);
}

void need_ctx(pq_ctx* c) {
    if (!c) throw std::invalid_argument("pq: null context");
    cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
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

// Pageable host results go through context-owned pinned buffers: the engine's early, overlapped
// result copies (phi_0 during the squaring, the run-ahead column half) need pinned destinations, and
// a pageable cudaMemcpy is a staged synchronous copy after the compute.  The bounce is copied to the
// caller's memory by several host threads once the call has finished.
constexpr size_t kBounceMin = size_t(1) << 20;  // doubles (8 MB)

static double* pinned_bounce(pq_ctx& c, const std::string& name, size_t count) {
    auto& slot = c.pin_bounce[name];
    const size_t bytes = count * sizeof(double);
    if (slot.second < bytes) {
        if (slot.first) cuda_check(cudaFreeHost(slot.first), "cudaFreeHost(bounce)");
        slot = {nullptr, 0};
        cuda_check(cudaMallocHost(reinterpret_cast<void**>(&slot.first), bytes), "cudaMallocHost(bounce)");
        slot.second = bytes;
    }
    return slot.first;
}

// Persistent helper threads for the host copies below (creating and joining 7 std::threads per
// copy cost ~0.1 ms, several times per drop-in call).  One job at a time; a caller that finds the
// pool busy (another thread's call) runs its copy with its own temporary threads.
class CopyPool {
public:
    static constexpr size_t kWorkers = 7;
    // f(w, nw) for w = 0 .. nw-1, nw = workers + 1, the caller running w = 0; false if busy
    bool try_run(const std::function<void(size_t, size_t)>& f) {
        std::unique_lock<std::mutex> own(busy_, std::try_to_lock);
        if (!own.owns_lock()) return false;
        start();
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &f;
            pending_ = kWorkers;
            ++gen_;
        }
        cv_.notify_all();
        f(0, kWorkers + 1);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
        job_ = nullptr;
        return true;
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }

private:
    void start() {
        if (!th_.empty()) return;
        for (size_t w = 1; w <= kWorkers; ++w)
            th_.emplace_back([this, w] {
                uint64_t seen = 0;
                while (true) {
                    const std::function<void(size_t, size_t)>* f = nullptr;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                        if (stop_) return;
                        seen = gen_;
                        f = job_;
                    }
                    (*f)(w, kWorkers + 1);
                    std::lock_guard<std::mutex> lk(mu_);
                    if (--pending_ == 0) done_.notify_all();
                }
            });
    }
    std::mutex busy_, mu_;
    std::condition_variable cv_, done_;
    std::vector<std::thread> th_;
    const std::function<void(size_t, size_t)>* job_ = nullptr;
    size_t pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Runs work(t0, step) over `total` pieces on up to 8 threads (the pool, else temporary threads).
static void host_parallel(size_t total, const std::function<void(size_t, size_t)>& work) {
    if (total <= 1) {
        work(0, 1);
        return;
    }
    static CopyPool pool;
    if (total >= 4 && pool.try_run(work)) return;
    const size_t threads = std::min<size_t>(8, total);
    std::vector<std::thread> team;
    for (size_t w = 1; w < threads; ++w) team.emplace_back(work, w, threads);
    work(0, threads);
    for (auto& t : team) t.join();
}

// dst[k] <- src + k*count for each k, split over up to 8 host threads in 512 KB pieces
static void host_scatter(double* const* dst, const double* src, int parts, size_t count) {
    const size_t piece = size_t(1) << 16;  // doubles (512 KB)
    const size_t per = (count + piece - 1) / piece, total = per * static_cast<size_t>(parts);
    auto work = [&](size_t t0, size_t step) {
        for (size_t t = t0; t < total; t += step) {
            const size_t k = t / per, o = (t % per) * piece, len = std::min(piece, count - o);
            std::memcpy(dst[k] + o, src + k * count + o, len * sizeof(double));
        }
    };
    host_parallel(total, work);
}

static bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    const bool yes = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();  // a pageable pointer is not an error
    return yes;
}

// dst + k*count <- src[k] for each k (the inverse of host_scatter), same thread split
static void host_gather(double* dst, const double* const* src, int parts, size_t count) {
    const size_t piece = size_t(1) << 16;
    const size_t per = (count + piece - 1) / piece, total = per * static_cast<size_t>(parts);
    auto work = [&](size_t t0, size_t step) {
        for (size_t t = t0; t < total; t += step) {
            const size_t k = t / per, o = (t % per) * piece, len = std::min(piece, count - o);
            std::memcpy(dst + k * count + o, src[k] + o, len * sizeof(double));
        }
    };
    host_parallel(total, work);
}

// Device view of a caller vector: device pointers pass through; host data is staged.  Pageable
// inputs of 8 MB and more are first copied into a pinned bounce by several host threads: the
// driver's own staging of a pageable H2D runs at a fraction of the pinned PCIe rate.
const double* stage_in(pq_ctx& c, const double* p, size_t count, int space, const char* slot) {
    if (space == PQ_DEVICE || count == 0) return p;
    double* d = ws(c, slot, count);
    const double* src = p;
    if (count >= kBounceMin && !host_pinned(p)) {
        // four chunks: each chunk's H2D runs while the host threads fill the next one
        double* bnc = pinned_bounce(c, std::string("in:") + slot, count);
        const size_t chunk = (count / 4 + 1023) & ~size_t(1023);
        for (size_t o = 0; o < count; o += chunk) {
            const size_t len = std::min(chunk, count - o);
            double* dst = bnc + o;
            host_scatter(&dst, p + o, 1, len);
            cuda_check(cudaMemcpyAsync(d + o, bnc + o, len * sizeof(double), cudaMemcpyHostToDevice, c.stream), "H2D");
        }
        return d;
    }
    cuda_check(cudaMemcpyAsync(d, src, count * sizeof(double), cudaMemcpyHostToDevice, c.stream), "H2D");
    return d;
}
double* stage_out(pq_ctx& c, double* p, size_t count, int space, const char* slot) {
    if (space == PQ_DEVICE) return p;
    return ws(c, slot, count);
}
// Result to the caller's memory.  Pageable results of 8 MB and more: D2H into a pinned bounce at
// the full PCIe rate, wait, then several host threads copy it out (the call waits for its results
// anyway, so the wait here only moves the synchronisation earlier).
void finish_out(pq_ctx& c, double* host, const double* dev, size_t count, int space) {
    if (space == PQ_DEVICE || count == 0) return;
    if (count >= kBounceMin && !host_pinned(host)) {
        double* bnc = pinned_bounce(c, "out", count);
        cuda_check(cudaMemcpyAsync(bnc, dev, count * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "D2H (bounce)");
        cuda_check(cudaStreamSynchronize(c.stream), "D2H (bounce) wait");
        host_scatter(&host, bnc, 1, count);
        return;
    }
    cuda_check(cudaMemcpyAsync(host, dev, count * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "D2H");
}
void finish(pq_ctx& c, int space) {
    if (space == PQ_HOST) cuda_check(cudaStreamSynchronize(c.stream), "stream sync");
    int err = 0;
    // singular LU flag (dense.hpp:167) -- checked whenever the host already waits
    if (space == PQ_HOST) {
        err = *static_cast<volatile int*>(c.h_err);  // mapped: visible once the stream has drained
        if (err) {
            *c.h_err = 0;
            throw std::runtime_error("lu_solve: singular matrix");
        }
    }
}

// Caller vectors at their own addresses (the drop-in headers' std::vectors): gathered into one
// contiguous device buffer, and results scattered back -- pageable results of 8 MB and more
// through the context's pinned bounce, moved by several host threads.
const double* gather_cols(pq_ctx& c, const double* const* v, int count, long long N, int space, const char* slot) {
    need(v != nullptr, "null vector list");
    for (int k = 0; k < count; ++k) need(v[k] != nullptr, "null vector");
    if (space == PQ_DEVICE && count == 1) return v[0];
    double* g = ws(c, slot, static_cast<size_t>(count) * N);
    const size_t total = static_cast<size_t>(count) * N;
    if (space == PQ_HOST && total >= kBounceMin) {
        bool all_pinned = true;
        for (int k = 0; k < count && all_pinned; ++k) all_pinned = host_pinned(v[k]);
        if (!all_pinned) {  // pageable: several host threads fill a pinned bounce, then one H2D
            double* bnc = pinned_bounce(c, std::string("in:") + slot, total);
            host_gather(bnc, v, count, static_cast<size_t>(N));
            cuda_check(cudaMemcpyAsync(g, bnc, total * sizeof(double), cudaMemcpyHostToDevice, c.stream), "gather H2D");
            return g;
        }
    }
    for (int k = 0; k < count; ++k)
        cuda_check(cudaMemcpyAsync(g + static_cast<size_t>(k) * N, v[k], N * sizeof(double),
                                   space == PQ_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c.stream),
                   "gather vectors");
    return g;
}

void scatter_cols(pq_ctx& c, const double* dout, double* const* cols, int count, long long N, int space) {
    need(cols != nullptr, "null output list");
    for (int k = 0; k < count; ++k) need(cols[k] != nullptr, "null output vector");
    const size_t total = static_cast<size_t>(count) * N;
    if (space == PQ_HOST && total >= kBounceMin) {
        double* bnc = pinned_bounce(c, "cols", total);
        cuda_check(cudaMemcpyAsync(bnc, dout, total * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "D2H");
        finish(c, space);
        host_scatter(cols, bnc, count, static_cast<size_t>(N));
        return;
    }
    for (int k = 0; k < count; ++k)
        cuda_check(cudaMemcpyAsync(cols[k], dout + static_cast<size_t>(k) * N, N * sizeof(double),
                                   space == PQ_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c.stream),
                   "scatter columns");
    finish(c, space);
}

NodesWeights rule_from(int m, const double* nodes, const double* weights) {
    need(m >= 1 && nodes && weights, "phi_fixed: rule needs at least one point");
    NodesWeights r;
    r.x.assign(nodes, nodes + m);
    r.w.assign(weights, weights + m);
    return r;
}

int check_kind(int kind) {
    need(kind == PQ_GAUSS_LEGENDRE || kind == PQ_CLENSHAW_CURTIS, "pq: unknown quadrature kind");
    return kind;
}

}  // namespace

extern "C" {

const char* pq_version(void) { return "phiquad-b200 0.1 (sm_100a, FP64 DMMA)"; }
const char* pq_last_error(void) { return last_error_slot().c_str(); }

int pq_ctx_create(int device, pq_ctx** out) {
    return guarded([&] {
        need(out != nullptr, "pq_ctx_create: null out");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            throw CudaError("pq_ctx_create: no CUDA device (the engine has no CPU fallback)");
        }
        need(device >= 0 && device < count, "pq_ctx_create: device index out of range");
        cudaDeviceProp prop{};
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10)
            throw CudaError("pq_ctx_create: kernels are built for sm_100a; device is sm_" + std::to_string(prop.major) +
                            std::to_string(prop.minor));
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        auto* c = new pq_ctx();
        c->device = device;
        cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        c->own_stream = true;
        const char* tr = std::getenv("PQ_TRACE");
        c->trace = tr && tr[0] == '1';
        // small flags and readbacks in mapped pinned memory: kernels store into them directly, so
        // they never wait on the copy engines behind MB-sized transfers
        const unsigned mapped = cudaHostAllocMapped | cudaHostAllocPortable;
        cuda_check(cudaHostAlloc(&c->h_err, sizeof(int), mapped), "cudaHostAlloc(err)");
        *c->h_err = 0;
        cuda_check(cudaHostGetDevicePointer(&c->d_err, c->h_err, 0), "err device view");
        cuda_check(cudaMalloc(&c->d_int, 64 * sizeof(int)), "cudaMalloc(int)");
        cuda_check(cudaMalloc(&c->d_small, 1024 * sizeof(double)), "cudaMalloc(small)");
        cuda_check(cudaHostAlloc(&c->h_small, 1024 * sizeof(double), mapped), "cudaHostAlloc(small)");
        cuda_check(cudaHostGetDevicePointer(&c->h_small_d, c->h_small, 0), "small device view");
        cuda_check(cudaHostAlloc(&c->h_beta, 1024 * sizeof(double), mapped), "cudaHostAlloc(beta)");
        cuda_check(cudaHostGetDevicePointer(&c->h_beta_d, c->h_beta, 0), "beta device view");
        *out = c;
    });
}

int pq_ctx_destroy(pq_ctx* c) {
    return guarded([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        gate_forget(*c);
        for (auto& kv : c->bufs) ws_free_now(*c, kv.second.p);
        for (void* p : c->graveyard) cudaFree(p);
        trim_pool(*c);
        if (c->arena.host) cudaFreeHost(c->arena.host);
        if (c->arena.dev) cudaFree(c->arena.dev);
        if (c->arena.done) cudaEventDestroy(c->arena.done);
        cudaFreeHost(c->h_err);
        cudaFree(c->d_int);
        cudaFree(c->d_small);
        if (c->d_flops) cudaFree(c->d_flops);
        worker_stop(*c);
        cudaFreeHost(c->h_small);
        cudaFreeHost(c->h_beta);
        for (auto e : c->ev_pool) cudaEventDestroy(e);
        if (c->side) {
            cudaStreamSynchronize(c->side);
            cudaStreamDestroy(c->side);
            cudaEventDestroy(c->ev_fork);
            cudaEventDestroy(c->ev_join);
        }
        if (c->ev_late) cudaEventDestroy(c->ev_late);
        if (c->sq2) {
            cudaStreamSynchronize(c->sq2);
            cudaStreamDestroy(c->sq2);
            cudaEventDestroy(c->ev_sqfork);
        }
        if (c->ccs) {
            cudaStreamSynchronize(c->ccs);
            cudaStreamDestroy(c->ccs);
        }
        if (c->ev_ccfork) cudaEventDestroy(c->ev_ccfork);
        for (auto s : c->sqs) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
        for (auto e : c->ev_sqg) cudaEventDestroy(e);
        for (auto e : c->ev_early) cudaEventDestroy(e);
        for (auto& m : c->marks) cudaEventDestroy(m.ev);
        for (auto& r : c->krecs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        if (c->ev_latefork) cudaEventDestroy(c->ev_latefork);
        if (c->ev_beta) cudaEventDestroy(c->ev_beta);
        if (c->ev_cc) cudaEventDestroy(c->ev_cc);
        if (c->ev_fac) cudaEventDestroy(c->ev_fac);
        if (c->pin_fac) cudaFreeHost(c->pin_fac);
        for (auto& kv : c->pin_bounce) cudaFreeHost(kv.second.first);
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

int pq_ctx_set_stream(pq_ctx* c, void* stream) {
    return guarded([&] {
        need_ctx(c);
        cuda_check(cudaStreamSynchronize(c->stream), "sync old stream");
        if (c->own_stream) cudaStreamDestroy(c->stream);
        if (stream) {
            c->stream = static_cast<cudaStream_t>(stream);
            c->own_stream = false;
        } else {
            cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            c->own_stream = true;
        }
        if (c->arena.done) {
            cudaEventDestroy(c->arena.done);
            cuda_check(cudaEventCreateWithFlags(&c->arena.done, cudaEventDisableTiming), "event");
            cuda_check(cudaEventRecord(c->arena.done, c->stream), "record");
        }
        // helper streams follow the new stream's priority: recreated on next use
        for (cudaStream_t s : c->sqs) {
            cuda_check(cudaStreamSynchronize(s), "sync helper stream");
            cudaStreamDestroy(s);
        }
        c->sqs.clear();
        for (cudaStream_t* h : {&c->side, &c->sq2, &c->ccs}) {
            if (*h) {
                cuda_check(cudaStreamSynchronize(*h), "sync helper stream");
                cudaStreamDestroy(*h);
                *h = nullptr;
            }
        }
    });
}

void* pq_ctx_stream(const pq_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int pq_ctx_synchronize(pq_ctx* c) {
    return guarded([&] {
        need_ctx(c);
        finish(*c, PQ_HOST);
    });
}

uint64_t pq_ctx_launches(const pq_ctx* c) { return c ? c->launches : 0; }

int pq_ctx_set_workspace_limit(pq_ctx* c, uint64_t bytes) {
    return guarded([&] {
        need_ctx(c);
        c->ws_limit = bytes;
    });
}

int pq_ctx_release_workspace(pq_ctx* c) {
    return guarded([&] {
        need_ctx(c);
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        free_graveyard(*c);
        for (auto& kv : c->bufs) ws_free_now(*c, kv.second.p);
        c->bufs.clear();
        c->band_packs.clear();  // the fragment-major copies went with the workspace
        c->fac_cache.clear();
        trim_pool(*c);
    });
}

int pq_ctx_set_profiling(pq_ctx* c, int on) {
    return guarded([&] {
        need_ctx(c);
        c->profiling = on != 0;
    });
}

int pq_ctx_gemm_stats(pq_ctx* c, int reset, uint64_t* launches, double* ms, double* flops) {
    return guarded([&] {
        need_ctx(c);
        prof_collect(*c);
        if (launches) *launches = c->prof_launches;
        if (ms) *ms = c->prof_ms;
        if (flops) *flops = c->prof_flops;
        if (reset) {
            c->prof_launches = 0;
            c->prof_ms = c->prof_flops = 0.0;
        }
    });
}

int pq_ctx_gemm_dense_flops(pq_ctx* c, int reset, double* flops) {
    return guarded([&] {
        need_ctx(c);
        prof_collect(*c);
        if (flops) *flops = c->prof_flops_dense;
        if (reset) c->prof_flops_dense = 0.0;
    });
}

int pq_ctx_timeline(pq_ctx* c, const char** json) {
    return guarded([&] {
        need_ctx(c);
        cuda_check(cudaStreamSynchronize(c->stream), "timeline sync");
        std::string s = "[";
        for (size_t i = 0; i < c->marks.size(); ++i) {
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, c->marks[0].ev, c->marks[i].ev), "timeline elapsed");
            char buf[256];
            std::snprintf(buf, sizeof buf, "%s{\"mark\":\"%s\",\"gpu_us\":%.1f,\"host_us\":%.1f}", i ? "," : "",
                          c->marks[i].name.c_str(), ms * 1000.0, c->marks[i].host_us - c->marks[0].host_us);
            s += buf;
        }
        s += "]";
        for (auto& m : c->marks) cudaEventDestroy(m.ev);
        c->marks.clear();
        c->marks_json = s;
        *json = c->marks_json.c_str();
    });
}

int pq_ctx_gemm_breakdown(pq_ctx* c, int reset, const char** json) {
    return guarded([&] {
        need_ctx(c);
        prof_collect(*c);
        std::string s = "{";
        bool first = true;
        for (const auto& kv : c->gstats) {
            char buf[400];
            std::snprintf(buf, sizeof buf, "%s\"%s\":{\"launches\":%llu,\"ms\":%.6f,\"flops\":%.17g,\"dense\":%.17g}",
                          first ? "" : ",", kv.first.c_str(), static_cast<unsigned long long>(kv.second.launches),
                          kv.second.ms, kv.second.flops, kv.second.dense);
            s += buf;
            first = false;
        }
        s += "}";
        if (reset) c->gstats.clear();
        c->marks_json = s;
        if (json) *json = c->marks_json.c_str();
    });
}

int pq_ctx_check_guards(pq_ctx* c, int* damaged) {
    return guarded([&] {
        need_ctx(c);
        std::string names;
        const int bad = check_guards(*c, &names);
        if (damaged) *damaged = bad;
        last_error_slot() = bad ? "damaged workspace guards: " + names : std::string();
    });
}

int pq_ctx_kernel_stats(pq_ctx* c, int reset, const char** json) {
    return guarded([&] {
        need_ctx(c);
        prof_collect(*c);
        std::string s = "{";
        bool first = true;
        for (const auto& kv : c->kstats) {
            char buf[320];
            std::snprintf(buf, sizeof buf, "%s\"%s\":{\"launches\":%llu,\"ms\":%.6f,\"bytes\":%.17g}", first ? "" : ",",
                          kv.first.c_str(), static_cast<unsigned long long>(kv.second.launches), kv.second.ms,
                          kv.second.bytes);
            s += buf;
            first = false;
        }
        s += "}";
        if (reset) c->kstats.clear();
        c->marks_json = s;
        if (json) *json = c->marks_json.c_str();
    });
}

int pq_ctx_phase_times(pq_ctx* c, double* ms6) {
    return guarded([&] {
        need_ctx(c);
        need(ms6 != nullptr, "pq_ctx_phase_times: null out");
        for (int i = 0; i < 6; ++i) ms6[i] = c->phase_ms[i];
    });
}

// ---------------------------------------------------------------- host estimator -----------

int pq_gauss_legendre(int m, double* nodes, double* weights) {
    return guarded([&] {
        const NodesWeights r = gauss_legendre01(m);
        std::memcpy(nodes, r.x.data(), sizeof(double) * m);
        std::memcpy(weights, r.w.data(), sizeof(double) * m);
    });
}

int pq_clenshaw_curtis(int m, double* nodes, double* weights) {
    return guarded([&] {
        const NodesWeights r = clenshaw_curtis01(m);
        std::memcpy(nodes, r.x.data(), sizeof(double) * m);
        std::memcpy(weights, r.w.data(), sizeof(double) * m);
    });
}

int pq_cached_rule(int kind, int m, const double** nodes, const double** weights) {
    return guarded([&] {
        const NodesWeights& r = memo_rule(check_kind(kind), m);
        *nodes = r.x.data();
        *weights = r.w.data();
    });
}

int pq_quartic_roots(const double* c4, double* roots8) {
    return guarded([&] {
        auto z = quartic_zeros(Quartic{c4[0], c4[1], c4[2], c4[3]});
        for (int k = 0; k < 4; ++k) {
            roots8[2 * k] = z[static_cast<size_t>(k)].real();
            roots8[2 * k + 1] = z[static_cast<size_t>(k)].imag();
        }
    });
}

int pq_real_roots_greater_one(const double* c4, double* roots4, int* count) {
    return guarded([&] {
        auto r = real_zeros_above_one(Quartic{c4[0], c4[1], c4[2], c4[3]});
        *count = static_cast<int>(r.size());
        for (size_t i = 0; i < r.size(); ++i) roots4[i] = r[i];
    });
}

int pq_log_bound_at_rho(double n, int p, double alpha, double beta, int kind, double rho, double* out) {
    return guarded([&] { *out = log_bound_rho(BoundArgs{n, p, alpha, beta, check_kind(kind)}, rho); });
}

int pq_bound_quartic(double n, int p, double alpha, double beta, int kind, double* c4) {
    return guarded([&] {
        const Quartic q = stationary_quartic(BoundArgs{n, p, alpha, beta, check_kind(kind)});
        for (int k = 0; k < 4; ++k) c4[k] = q[static_cast<size_t>(k)];
    });
}

int pq_theorem_bound(double n, int p, double alpha, double beta, int kind, double* out) {
    return guarded([&] { *out = log_theorem_bound(BoundArgs{n, p, alpha, beta, check_kind(kind)}); });
}

int pq_corollary_bound(double n, int p, double alpha, double beta, int kind, double* out) {
    return guarded([&] { *out = log_corollary_bound(BoundArgs{n, p, alpha, beta, check_kind(kind)}); });
}

int pq_quaderr(double n, int p, double alpha, double beta, int kind, double* out) {
    return guarded([&] { *out = log_quaderr(n, p, alpha, beta, check_kind(kind)); });
}

int pq_quadnodes(double eps, int p, double alpha, double beta, int kind, int* n) {
    return guarded([&] { *n = node_count(eps, p, alpha, beta, check_kind(kind)); });
}

int pq_setup_quadrature(double eps, int p, double alpha, double beta, int kind, double c1, double c2, int d, int* l,
                        int* n, double* cost) {
    return guarded([&] {
        const Plan pl = plan_quadrature(eps, p, alpha, beta, check_kind(kind), Cost{c1, c2, d});
        *l = pl.l;
        *n = pl.n;
        *cost = pl.cost;
    });
}

int pq_infnorm_bound(int d, const int* shape, const double* factors, double* out) {
    return guarded([&] {
        dim_of(d, shape);
        double s = 0.0;
        size_t off = 0;
        for (int k = 0; k < d; ++k) {
            const int n = shape[k];
            double best = 0.0;
            for (int i = 0; i < n; ++i) {
                double rs = 0.0;
                for (int j = 0; j < n; ++j) rs += std::abs(factors[off + static_cast<size_t>(i) * n + j]);
                if (rs > best) best = rs;
            }
            s += best;
            off += static_cast<size_t>(n) * n;
        }
        *out = s;
    });
}

// ---------------------------------------------------------------- device primitives --------

int pq_expm(pq_ctx* c, int n, int batch, const double* a, const double* scale, double* out, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_expm");
        need_ctx(c);
        need(n >= 0 && batch >= 0, "expm: bad extent");
        if (n == 0 || batch == 0) return;
        const size_t nn = static_cast<size_t>(n) * n;
        if (space == PQ_HOST)
            for (size_t e = 0; e < nn; ++e)
                if (!std::isfinite(a[e])) throw std::invalid_argument("DenseMatrix: non-finite entry");
        const double* da = stage_in(*c, a, nn, space, "hin_a");
        double* dout = stage_out(*c, out, nn * batch, space, "hout");
        std::vector<double> sc(static_cast<size_t>(batch), 1.0);
        if (scale) {
            if (space == PQ_HOST) {
                std::memcpy(sc.data(), scale, sizeof(double) * batch);
            } else {
                cuda_check(cudaMemcpy(sc.data(), scale, sizeof(double) * batch, cudaMemcpyDeviceToHost), "scale");
            }
        }
        arena_begin(*c);
        double one_norm = -1.0;  // unknown for device input: counts are read back
        if (space == PQ_HOST) {
            std::vector<double> col(static_cast<size_t>(n), 0.0);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) col[static_cast<size_t>(j)] += std::abs(a[static_cast<size_t>(i) * n + j]);
            one_norm = 0.0;
            for (double v : col) one_norm = std::max(one_norm, v);
        }
        expm_batch(*c, n, batch, da, 0, sc, one_norm, dout);
        finish_out(*c, out, dout, nn * batch, space);
        finish(*c, space);
    });
}

int pq_mode_apply(pq_ctx* c, int d, const int* shape, const double* mats, const double* x, double* y, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_mode_apply");
        need_ctx(c);
        const long long N = dim_of(d, shape);
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, mats, "mats");
        const double* dx = stage_in(*c, x, N, space, "hin_x");
        double* dy = stage_out(*c, y, N, space, "hout");
        const double* E[3] = {op.F[0], op.F[1], op.F[2]};
        long long Es[3] = {0, 0, 0};
        mode_chain(*c, d, op.n, E, Es, dx, N, dy, N, 1, Epilogue{});
        finish_out(*c, y, dy, N, space);
        finish(*c, space);
    });
}

int pq_kron_matvec(pq_ctx* c, int d, const int* shape, const double* factors, const double* x, double* y, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_kron_matvec");
        need_ctx(c);
        const long long N = dim_of(d, shape);
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* dx = stage_in(*c, x, N, space, "hin_x");
        double* dy = stage_out(*c, y, N, space, "hout");
        kron_matvec_dev(*c, op, 1.0, dx, dy);
        finish_out(*c, y, dy, N, space);
        finish(*c, space);
    });
}

int pq_exp_action(pq_ctx* c, int d, const int* shape, const double* factors, const double* b, double* y, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_exp_action");
        need_ctx(c);
        const long long N = dim_of(d, shape);
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* db = stage_in(*c, b, N, space, "hin_b");
        double* dy = stage_out(*c, y, N, space, "hout0");
        exp_action_dev(*c, op, 1.0, 1, db, dy);
        finish_out(*c, y, dy, N, space);
        finish(*c, space);
    });
}

// ---------------------------------------------------------------- phi engine ---------------

int pq_phi_fixed(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs, int p, int m,
                 const double* nodes, const double* weights, double* out, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_fixed");
        need_ctx(c);
        need(p >= 1, "phi_fixed: need p >= 1");
        need(nb >= 0, "phi_fixed: need nb >= 0");
        const long long N = dim_of(d, shape);
        const NodesWeights rule = rule_from(m, nodes, weights);
        if (nb == 0) return;
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* db = stage_in(*c, bs, static_cast<size_t>(nb) * N, space, "hin_b");
        double* dout = stage_out(*c, out, static_cast<size_t>(nb) * p * N, space, "hout");
        phi_fixed_dev(*c, op, 1.0, nb, db, p, rule, dout);
        finish_out(*c, out, dout, static_cast<size_t>(nb) * p * N, space);
        finish(*c, space);
    });
}

int pq_phi_adaptive(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs, int p,
                    double eps, double* out, int* points_used, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_adaptive");
        need_ctx(c);
        need(p >= 1, "phi_adaptive: need p >= 1");
        need(eps > 0.0, "phi_adaptive: need eps > 0");
        need(nb >= 0, "phi_adaptive: need nb >= 0");
        const long long N = dim_of(d, shape);
        if (nb == 0) {  // the reference still climbs to the 13-point rule (phiaction.hpp:175-240)
            if (points_used) *points_used = 13;
            return;
        }
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* db = stage_in(*c, bs, static_cast<size_t>(nb) * N, space, "hin_b");
        double* dout = stage_out(*c, out, static_cast<size_t>(nb) * p * N, space, "hout");
        phi_adaptive_dev(*c, op, 1.0, nb, db, p, eps, dout, points_used);
        finish_out(*c, out, dout, static_cast<size_t>(nb) * p * N, space);
        finish(*c, space);
    });
}

int pq_phi_fixed_cols(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* const* bs,
                      int p, int m, const double* nodes, const double* weights, double* const* cols, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_fixed_cols");
        need_ctx(c);
        need(p >= 1, "phi_fixed: need p >= 1");
        need(nb >= 0, "phi_fixed: need nb >= 0");
        const long long N = dim_of(d, shape);
        const NodesWeights rule = rule_from(m, nodes, weights);
        if (nb == 0) return;
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* db = gather_cols(*c, bs, nb, N, space, "hin_b");
        double* dout = ws(*c, "hout", static_cast<size_t>(nb) * p * N);
        phi_fixed_dev(*c, op, 1.0, nb, db, p, rule, dout);
        scatter_cols(*c, dout, cols, nb * p, N, space);
    });
}

int pq_phi_adaptive_cols(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* const* bs,
                         int p, double eps, double* const* cols, int* points_used, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_adaptive_cols");
        need_ctx(c);
        need(p >= 1, "phi_adaptive: need p >= 1");
        need(eps > 0.0, "phi_adaptive: need eps > 0");
        need(nb >= 0, "phi_adaptive: need nb >= 0");
        const long long N = dim_of(d, shape);
        if (nb == 0) {
            if (points_used) *points_used = 13;
            return;
        }
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* db = gather_cols(*c, bs, nb, N, space, "hin_b");
        double* dout = ws(*c, "hout", static_cast<size_t>(nb) * p * N);
        phi_adaptive_dev(*c, op, 1.0, nb, db, p, eps, dout, points_used);
        scatter_cols(*c, dout, cols, nb * p, N, space);
    });
}

int pq_squaring_step_cols(pq_ctx* c, int d, const int* shape, const double* exps, int p, double* const* cols,
                          int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_squaring_step_cols");
        need_ctx(c);
        need(p >= 1, "squaring_step: need p >= 1");
        const long long N = dim_of(d, shape);
        arena_begin(*c);
        DevOp ex = upload_op(*c, d, shape, exps, "exps");
        need(cols != nullptr, "null vector list");
        double* dy = ws(*c, "hio_y", static_cast<size_t>(p) * N);
        for (int k = 0; k < p; ++k) {
            need(cols[k] != nullptr, "null vector");
            cuda_check(cudaMemcpyAsync(dy + static_cast<size_t>(k) * N, cols[k], N * sizeof(double),
                                       space == PQ_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                                       c->stream),
                       "gather columns");
        }
        squaring_steps_dev(*c, ex, 1.0, 1, p, 1, dy, ex.F[0]);
        scatter_cols(*c, dy, cols, p, N, space);
    });
}

int pq_squaring_step(pq_ctx* c, int d, const int* shape, const double* exps, int p, double* y, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_squaring_step");
        need_ctx(c);
        need(p >= 1, "squaring_step: need p >= 1");
        const long long N = dim_of(d, shape);
        arena_begin(*c);
        DevOp ex = upload_op(*c, d, shape, exps, "exps");
        // exps are already exponentials: pass them as the override of the step's E
        double* dy = space == PQ_DEVICE ? y : ws(*c, "hio_y", static_cast<size_t>(p) * N);
        if (space == PQ_HOST)
            cuda_check(cudaMemcpyAsync(dy, y, sizeof(double) * p * N, cudaMemcpyHostToDevice, c->stream), "H2D");
        size_t total = 0;
        for (int k = 0; k < d; ++k) total += static_cast<size_t>(shape[k]) * shape[k];
        squaring_steps_dev(*c, ex, 1.0, 1, p, 1, dy, ex.F[0]);
        (void)total;
        finish_out(*c, y, dy, static_cast<size_t>(p) * N, space);
        finish(*c, space);
    });
}

// phi_with_plan's argument checks in the reference's order (phiaction.hpp:277-290 -> cached_rule
// -> phi_fixed_multi :134-139 / phi_adaptive_multi :156-166)
static void plan_checks(int l, int n, int p, int kind, double eps) {
    need(l >= 0, "phi_with_plan: need l >= 0");
    check_kind(kind);
    if (kind == PQ_GAUSS_LEGENDRE) {
        need(n + 1 >= 1, "gauss_legendre: need at least one point");
        need(p >= 1, "phi_fixed: need p >= 1");
    } else {
        need(p >= 1, "phi_adaptive: need p >= 1");
        need(eps > 0.0, "phi_adaptive: need eps > 0");
    }
}

int pq_phi_with_plan(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs, int p, int l,
                     int n, int kind, double eps, double* out, int* points_used, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_with_plan");
        need_ctx(c);
        plan_checks(l, n, p, kind, eps);
        const long long N = dim_of(d, shape);
        if (nb == 0) {  // the reference still reports the rule size (phiaction.hpp:282-290)
            if (points_used) *points_used = kind == PQ_GAUSS_LEGENDRE ? n + 1 : 13;
            return;
        }
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* db = stage_in(*c, bs, static_cast<size_t>(nb) * N, space, "hin_b");
        double* dout = stage_out(*c, out, static_cast<size_t>(nb) * p * N, space, "hout");
        phi_with_plan_dev(*c, op, 1.0, nb, db, p, l, n, kind, eps, dout, points_used);
        finish_out(*c, out, dout, static_cast<size_t>(nb) * p * N, space);
        finish(*c, space);
    });
}

int pq_phi_with_plan_cols(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* const* bs,
                          int p, int l, int n, int kind, double eps, double* const* cols, int* points_used, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_with_plan_cols");
        need_ctx(c);
        plan_checks(l, n, p, kind, eps);
        const long long N = dim_of(d, shape);
        if (nb == 0) {  // the reference still reports the rule size (phiaction.hpp:282-290)
            if (points_used) *points_used = kind == PQ_GAUSS_LEGENDRE ? n + 1 : 13;
            return;
        }
        need(bs != nullptr && cols != nullptr, "phi_with_plan: null vector list");
        for (int m = 0; m < nb; ++m) need(bs[m] != nullptr, "phi_with_plan: null right-hand side");
        for (int k = 0; k < nb * p; ++k) need(cols[k] != nullptr, "phi_with_plan: null output column");
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        double* db = ws(*c, "hin_b", static_cast<size_t>(nb) * N);
        for (int m = 0; m < nb; ++m)
            cuda_check(cudaMemcpyAsync(db + static_cast<size_t>(m) * N, bs[m], N * sizeof(double),
                                       space == PQ_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream),
                       "gather b");
        double* dout = ws(*c, "hout", static_cast<size_t>(nb) * p * N);
        phi_with_plan_dev(*c, op, 1.0, nb, db, p, l, n, kind, eps, dout, points_used);
        const size_t total = static_cast<size_t>(nb) * p * N;
        if (space == PQ_HOST && total >= kBounceMin) {  // one D2H into a pinned bounce, host threads fill the columns
            double* bnc = pinned_bounce(*c, "cols", total);
            cuda_check(cudaMemcpyAsync(bnc, dout, total * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
            finish(*c, space);
            host_scatter(cols, bnc, nb * p, static_cast<size_t>(N));
        } else {
            for (int k = 0; k < nb * p; ++k)
                cuda_check(cudaMemcpyAsync(cols[k], dout + static_cast<size_t>(k) * N, N * sizeof(double),
                                           space == PQ_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                           c->stream),
                           "scatter columns");
            finish(*c, space);
        }
    });
}

// b_list / col_list (pq_phiquadmv_cols): RHS m at b_list[m], phi_{j+1} of RHS m to col_list[m p + j]
// instead of the contiguous bs / out
static void run_phiquadmv_impl(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs,
                               const pq_phi_request* req, double* out0, double* out, pq_phi_info* info, int space,
                               const double* const* b_list, double* const* col_list);

// PQ_SLOWLOG=<ms>: every phiquadmv-family call records its phase marks (device events + host
// clock, like PQ_TRACE); a call whose host wall time exceeds <ms> prints its timeline to stderr
// (diagnostics for latency outliers such as the acceptance gate's criterion 7).
static double slowlog_ms() {
    static const double v = [] {
        const char* e = std::getenv("PQ_SLOWLOG");
        return e ? std::atof(e) : 0.0;
    }();
    return v;
}

static void run_phiquadmv(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs,
                          const pq_phi_request* req, double* out0, double* out, pq_phi_info* info, int space,
                          const double* const* b_list = nullptr, double* const* col_list = nullptr) {
    const double thr = slowlog_ms();
    if (thr <= 0.0 || !c) {
        run_phiquadmv_impl(c, d, shape, factors, nb, bs, req, out0, out, info, space, b_list, col_list);
        return;
    }
    const bool was = c->trace;
    c->trace = true;
    for (auto& m : c->marks) cudaEventDestroy(m.ev);
    c->marks.clear();
    const auto t0 = std::chrono::steady_clock::now();
    try {
        run_phiquadmv_impl(c, d, shape, factors, nb, bs, req, out0, out, info, space, b_list, col_list);
    } catch (...) {
        c->trace = was;
        throw;
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    c->trace = was;
    if (ms > thr && !c->marks.empty()) {
        cudaStreamSynchronize(c->stream);
        std::string s;
        for (size_t i = 0; i < c->marks.size(); ++i) {
            float g = 0.f;
            cudaEventElapsedTime(&g, c->marks[0].ev, c->marks[i].ev);
            char buf[200];
            std::snprintf(buf, sizeof buf, " %s@gpu%.0fus/host%.0fus", c->marks[i].name.c_str(), g * 1000.0,
                          c->marks[i].host_us - c->marks[0].host_us);
            s += buf;
        }
        std::fprintf(stderr, "[pq slow call] %.2f ms (N=%lld, nb=%d, p=%d):%s\n", ms, dim_of(d, shape), nb,
                     req ? req->p : 0, s.c_str());
    }
    if (!was) {
        for (auto& m : c->marks) cudaEventDestroy(m.ev);
        c->marks.clear();
    }
}

static void run_phiquadmv_impl(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs,
                               const pq_phi_request* req, double* out0, double* out, pq_phi_info* info, int space,
                               const double* const* b_list, double* const* col_list) {
    need_ctx(c);
    need(req != nullptr, "phiquadmv: null request");
    need(req->p >= 1, "phiquadmv: need p >= 1");
    check_kind(req->mode);
    const long long N = dim_of(d, shape);
    need(nb >= 0, "phiquadmv: negative right-hand-side count");
    const int p = req->p;
    if (nb == 0) {  // reference: beta = 0 plans l = 0 (or the pinned l) and returns no columns
        double alpha = 0.0;
        if (pq_infnorm_bound(d, shape, factors, &alpha) != PQ_OK) throw std::invalid_argument(last_error_slot());
        int l = 0, n = req->mode == PQ_GAUSS_LEGENDRE ? 2 : 4;
        if (req->has_l) {
            need(req->l >= 0, "phiquadmv: need l >= 0");
            l = req->l;
        }
        plan_checks(l, n, p, req->mode, req->eps);
        if (info) {
            info->l = l;
            info->n = n;
            info->points = req->mode == PQ_GAUSS_LEGENDRE ? n + 1 : 13;
            info->mode = req->mode;
            info->planned = req->has_l ? 0 : 1;
            info->alpha = alpha;
            info->beta = 0.0;
            info->plan_cost = pqb::Cost{req->c1, req->c2, d}(n, l, p);
        }
        return;
    }
    mark(*c, "call");
    arena_begin(*c);
    DevOp op = upload_op(*c, d, shape, factors, "factors");
    const double* db = nullptr;
    if (b_list) {
        for (int m = 0; m < nb; ++m) need(b_list[m] != nullptr, "phiquadmv: null right-hand side");
        if (space == PQ_DEVICE && nb == 1) {
            db = b_list[0];
        } else if (space == PQ_HOST && nb == 1) {
            db = stage_in(*c, b_list[0], static_cast<size_t>(N), space, "hin_b");
        } else {
            db = gather_cols(*c, b_list, nb, N, space, "hin_b");
        }
    } else {
        db = stage_in(*c, bs, static_cast<size_t>(nb) * N, space, "hin_b");
    }
    if (col_list)
        for (int k = 0; k < nb * p; ++k) need(col_list[k] != nullptr, "phiquadmv: null output column");
    double* dout = col_list ? ws(*c, "hout", static_cast<size_t>(nb) * p * N)
                            : stage_out(*c, out, static_cast<size_t>(nb) * p * N, space, "hout");
    mark(*c, "uploaded");
    PlanInfo pi;
    double* d0 = out0 ? stage_out(*c, out0, static_cast<size_t>(nb) * N, space, "hout0") : nullptr;
    // pinned host phi_0 buffer: copied out by the engine as soon as phi_0 exists (overlaps the squaring)
    auto pinned = [&](double* ptr) {
        if (!ptr || space != PQ_HOST) return false;
        cudaPointerAttributes at{};
        const bool yes = cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeHost;
        cudaGetLastError();  // a pageable pointer is not an error
        return yes;
    };
    double* h0 = pinned(out0) ? out0 : nullptr;
    double* hc = pinned(out) ? out : nullptr;
    double* bounce0 = nullptr;
    double* bounce = nullptr;
    // (only for results of 8 MB and more: below that the direct copies cost less than the bounce's
    // host threads and first-use cudaMallocHost)
    if (space == PQ_HOST && static_cast<size_t>(nb) * p * N >= kBounceMin) {
        if (out0 && !h0) h0 = bounce0 = pinned_bounce(*c, "phi0", static_cast<size_t>(nb) * N);
        if (col_list || (out && !hc)) hc = bounce = pinned_bounce(*c, "cols", static_cast<size_t>(nb) * p * N);
    }
    bool cols_copied = false;
    c->early.clear();
    // several host callers: this call's compute waits for the previous caller's compute, not for its
    // result copies (engine.hpp gate_acquire)
    struct GateHold {
        pq_ctx* c = nullptr;
        void done() {
            if (c) gate_enqueued(*c);
            c = nullptr;
        }
        ~GateHold() { done(); }
    } gate;
    if (space == PQ_HOST && gate_wanted(static_cast<size_t>(nb) * (p + (out0 ? 1 : 0)) * N * sizeof(double))) {
        gate_acquire(*c);
        gate.c = c;
    }
    phiquadmv_dev(*c, op, nb, db, p, req->eps, req->mode, req->has_l != 0, req->l, req->c1, req->c2, dout, &pi, d0, h0,
                  hc, &cols_copied);
    gate.done();
    // bounced results that are already on their way: move each to the caller's memory as soon as
    // its copy lands, while the device finishes the rest of the call
    bool done0 = false;
    std::vector<char> done_col(static_cast<size_t>(nb) * p, 0);
    auto drain = [&](const pq_ctx::EarlyCopy& e) {
        if (bounce0 && e.host == bounce0) {
            cuda_check(cudaEventSynchronize(e.ev), "early copy wait");
            host_scatter(&out0, bounce0, 1, static_cast<size_t>(nb) * N);
            done0 = true;
        } else if (bounce && e.host >= bounce && e.host < bounce + static_cast<size_t>(nb) * p * N) {
            const size_t k0 = static_cast<size_t>(e.host - bounce) / N, kc = e.count / N;
            if (k0 * N != static_cast<size_t>(e.host - bounce) || kc * N != e.count) return;  // not whole columns
            cuda_check(cudaEventSynchronize(e.ev), "early copy wait");
            if (col_list) {
                host_scatter(col_list + k0, bounce + k0 * N, static_cast<int>(kc), static_cast<size_t>(N));
            } else {
                double* dst = out + k0 * N;
                host_scatter(&dst, bounce + k0 * N, 1, kc * N);
            }
            for (size_t k = k0; k < k0 + kc; ++k) done_col[k] = 1;
        }
    };
    if (bounce0 || bounce)
        for (size_t i = 0; i + 1 < c->early.size(); ++i) drain(c->early[i]);  // the last one ends the call anyway
    mark(*c, "computed");
    if (out0 && !h0) finish_out(*c, out0, d0, static_cast<size_t>(nb) * N, space);
    if (bounce && !cols_copied)
        cuda_check(cudaMemcpyAsync(bounce, dout, static_cast<size_t>(nb) * p * N * sizeof(double), cudaMemcpyDeviceToHost,
                                   c->stream),
                   "D2H (bounce)");
    if (col_list && !bounce) {
        for (int k = 0; k < nb * p; ++k)
            cuda_check(cudaMemcpyAsync(col_list[k], dout + static_cast<size_t>(k) * N, N * sizeof(double),
                                       space == PQ_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream),
                       "scatter columns");
    } else if (!bounce && !cols_copied) {
        finish_out(*c, out, dout, static_cast<size_t>(nb) * p * N, space);
    }
    finish(*c, space);
    if (bounce0 && !done0) host_scatter(&out0, bounce0, 1, static_cast<size_t>(nb) * N);
    if (bounce) {
        for (int k = 0; k < nb * p; ++k) {
            if (done_col[static_cast<size_t>(k)]) continue;
            int k1 = k;
            while (k1 + 1 < nb * p && !done_col[static_cast<size_t>(k1) + 1]) ++k1;
            if (col_list) {
                host_scatter(col_list + k, bounce + static_cast<size_t>(k) * N, k1 - k + 1, static_cast<size_t>(N));
            } else {
                double* dst = out + static_cast<size_t>(k) * N;
                host_scatter(&dst, bounce + static_cast<size_t>(k) * N, 1, static_cast<size_t>(k1 - k + 1) * N);
            }
            k = k1;
        }
    }
    mark(*c, "returned");
    if (info) {
        info->l = pi.l;
        info->n = pi.n;
        info->points = pi.points;
        info->mode = pi.mode;
        info->planned = pi.planned;
        info->alpha = pi.alpha;
        info->beta = pi.beta;
        info->plan_cost = pi.cost;
    }
}

int pq_phiquadmv(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs,
                 const pq_phi_request* req, double* out, pq_phi_info* info, int space) {
    return guarded([&] { run_phiquadmv(c, d, shape, factors, nb, bs, req, nullptr, out, info, space); });
        NvtxRange nvtx("pq_phiquadmv");
}

int pq_phiquadmv_cols(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* const* bs,
                      const pq_phi_request* req, double* const* cols, pq_phi_info* info, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phiquadmv_cols");
        need(nb == 0 || (bs != nullptr && cols != nullptr), "phiquadmv: null vector list");
        run_phiquadmv(c, d, shape, factors, nb, nullptr, req, nullptr, nullptr, info, space, bs, cols);
    });
}

int pq_phi_0p(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs,
              const pq_phi_request* req, double* out0, double* out, pq_phi_info* info, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_0p");
        need(out0 != nullptr, "phi_0p: null phi_0 output");
        run_phiquadmv(c, d, shape, factors, nb, bs, req, out0, out, info, space);
    });
}

int pq_phi_lincomb(pq_ctx* c, int d, const int* shape, const double* factors, int p, const double* bs, int m,
                   const double* nodes, const double* weights, double* out, int space) {
    return guarded([&] {
        NvtxRange nvtx("pq_phi_lincomb");
        need_ctx(c);
        need(p >= 1, "phi_lincomb: need at least one vector");
        const long long N = dim_of(d, shape);
        const NodesWeights rule = rule_from(m, nodes, weights);
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        const double* db = stage_in(*c, bs, static_cast<size_t>(p) * N, space, "hin_b");
        double* dout = stage_out(*c, out, N, space, "hout");
        phi_lincomb_dev(*c, op, 1.0, p, db, rule, dout);
        finish_out(*c, out, dout, N, space);
        finish(*c, space);
    });
}

int pq_phi_nodes_partial(pq_ctx* c, int d, const int* shape, const double* factors, int nb, const double* bs, int p,
                         int l, int m, const double* nodes, const double* weights, int rank, int world, int zero,
                         double* acc) {
    return guarded([&] {
        need_ctx(c);
        need(p >= 1, "phi_fixed: need p >= 1");
        need(l >= 0, "phi_with_plan: need l >= 0");
        need(world >= 1 && rank >= 0 && rank < world, "phi_nodes_partial: bad rank/world");
        dim_of(d, shape);
        const NodesWeights rule = rule_from(m, nodes, weights);
        std::vector<int> mine;
        for (int i = rank; i < m; i += world) mine.push_back(i);
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        // nodes on 2^-l A: fold the exact power of two into the operator scale
        phi_nodes_partial_dev(*c, op, std::ldexp(1.0, -l), nb, bs, p, rule, mine, zero, acc);
    });
}

int pq_mode_product(pq_ctx* c, int d, const int* shape, int mode, const double* E, int nb, const double* x, double* y) {
    return guarded([&] {
        need_ctx(c);
        const long long N = dim_of(d, shape);
        need(mode >= 0 && mode < d, "mode_product: mode out of range");
        need(nb >= 1, "mode_product: need at least one column");
        need(E && x && y && x != y, "mode_product: null or aliased pointers");
        int n[3] = {1, 1, 1};
        for (int k = 0; k < d; ++k) n[k] = shape[k];
        gemm(*c, mode_gemm_public(d, n, mode, E, x, y, nb, N));
        check_launch(*c);
    });
}

int pq_squaring_combine(pq_ctx* c, long long n, int p, int nb, double* t, const double* y) {
    return guarded([&] {
        need_ctx(c);
        need(n >= 1 && p >= 1 && nb >= 1, "squaring_combine: bad extents");
        need(t && y, "squaring_combine: null pointers");
        std::vector<double> inv(static_cast<size_t>(p), 1.0);
        double f = 1.0;
        for (int k = 1; k < p; ++k) {
            f *= k;
            inv[static_cast<size_t>(k)] = 1.0 / f;
        }
        std::vector<double> coef(static_cast<size_t>(p) * p, 0.0);
        for (int i = 0; i < p; ++i)
            for (int j = 0; j <= i; ++j)
                coef[static_cast<size_t>(i) * p + j] = std::ldexp(1.0, -(i + 1)) * inv[static_cast<size_t>(i - j)];
        arena_begin(*c);
        const double* cd = static_cast<const double*>(arena_push(*c, coef.data(), coef.size() * sizeof(double)));
        arena_flush(*c);
        launch_sq_combine(n, p, nb, t, y, cd, c->stream);
        count_launch(*c);
    });
}

int pq_squaring_chain(pq_ctx* c, int d, const int* shape, const double* factors, int nb, int p, int l, double* y) {
    return guarded([&] {
        need_ctx(c);
        need(l >= 0, "phi_with_plan: need l >= 0");
        need(p >= 1, "squaring_step: need p >= 1");
        dim_of(d, shape);
        arena_begin(*c);
        DevOp op = upload_op(*c, d, shape, factors, "factors");
        squaring_steps_dev(*c, op, 1.0, nb, p, l, y, nullptr);
    });
}

}  // extern "C"
