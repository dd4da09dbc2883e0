// Internal host-side engine: context, device workspace and the phi pipeline built from the
// kernels in kernels.cu.  Everything here is stream-ordered on ctx.stream; the only host syncs
// are the ones a host decision needs (beta for the planner, the adaptive CC error per level,
// expm squaring counts for standalone pq_expm) and the final copy-out of PQ_HOST calls.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "estimator.hpp"
#include "kernels.hpp"

namespace pqb {

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
void cuda_check(cudaError_t e, const char* what);

// A device buffer that only grows (cudaMalloc is a device-wide sync; steady state never reallocates).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

// Pinned staging arena for small per-call parameter tables (rule coefficients, epilogue tables).
struct ParamArena {
    char* host = nullptr;
    char* host_d = nullptr;  // device view of the mapped pinned staging buffer
    char* dev = nullptr;
    size_t cap = 0, used = 0, flushed = 0;
    cudaEvent_t done = nullptr;
};

struct Engine;

}  // namespace pqb

struct pq_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t launches = 0;
    uint64_t ws_limit = 0;
    std::map<std::string, pqb::DevBuf> bufs;
    // workspace buffers replaced by a larger one: freed only when the context releases its workspace
    // (or an allocation fails), never inside a call -- cudaFree of a large buffer is a device-wide
    // synchronisation that took 20-60 ms on the B200 (the acceptance gate's criterion-7 outlier)
    std::vector<void*> graveyard;
    // PQ_WS_GUARD=1 (debug, the memcheck substitute on pools where compute-sanitizer is closed):
    // every workspace buffer carries 4 KB canary regions before and after it; user pointer -> base
    struct Guarded {
        void* base;
        size_t bytes;
        std::string name;
    };
    std::map<void*, Guarded> guards;
    pqb::ParamArena arena;
    int* d_err = nullptr;        // error flag (singular LU): mapped pinned host memory, device view
    int* h_err = nullptr;        //   ... and its host view
    double* h_small = nullptr;   // mapped pinned readback scratch (host view)
    double* h_small_d = nullptr; //   ... device view (launch_store_words target)
    double* h_beta = nullptr;    // mapped pinned readback of the planner's beta (read by the planner thread)
    double* h_beta_d = nullptr;  //   ... device view
    double* d_small = nullptr;   // device scratch for reductions
    int* d_int = nullptr;        // device int scratch (expm squaring counts)
    bool profiling = false;
    bool trace = false;  // PQ_TRACE=1: phase marks without profiling's stream serialisation
    // side stream for work independent of the node sweep (phi_0), joined back before returning
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_late = nullptr;  // late exponentials (squaring chain, phi_0) finished on `side`
    cudaEvent_t ev_latefork = nullptr;  // main-stream point the late exponentials depend on
    // side-stream work enqueued only after the first node sweep is on the main stream (so the
    // host's enqueue time for it does not delay the sweep); run_deferred() flushes it
    std::vector<std::function<void()>> deferred;
    // two-stream squaring (engine.cpp squaring_pingpong): second stream, fork event, per-step events
    cudaStream_t sq2 = nullptr;
    // a CC ladder level's combination offloaded under the next level's node sweep: one priority
    // step above the main stream, so its (HBM-bound) CTAs interleave with the sweep's DMMA tiles
    cudaStream_t ccs = nullptr;
    cudaEvent_t ev_ccfork = nullptr;
    // per-column squaring streams when the results go to pinned host memory (descending priority:
    // column 1 runs ahead and its D2H overlaps the later columns) and their per-(group, step) events
    std::vector<cudaStream_t> sqs;
    std::vector<cudaEvent_t> ev_sqg;
    cudaEvent_t ev_sqfork = nullptr;
    // Taylor powers of the current call's factors (engine.cpp taylor_powers), per factor size;
    // valid only for the DevOp serial they were computed for (never reused across calls)
    struct PowCache {
        const double* P = nullptr;
        const double* base = nullptr;
        std::vector<long long> foff;
        double scale = 0.0;
        uint64_t serial = 0;
    };
    std::map<int, PowCache> pow_cache;
    uint64_t op_serial = 0;  // incremented per operator upload (one per API call)
    // negligible-block tables of the operator's own factors (kron_matvec), per upload serial
    uint64_t fac_band_serial = 0;
    // fragment-major copies of exponential batches (kernels.hpp launch_band_ranges pack), found from
    // the batch's band-table pointer: records [lo, lo + recs) <-> pack + record_index * per-matrix size
    struct BandPack {
        const int2* lo = nullptr;
        size_t recs = 0;
        double* pack = nullptr;
        int n = 0;
    };
    std::vector<BandPack> band_packs;
    uint64_t tri_serial = 0;  // operator upload whose factors were checked for tridiagonality
    bool tri = false;
    const int2* fac_band[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev_beta = nullptr;  // beta readback (phiquadmv) completes
    // Plan speculation (engine.cpp phiquadmv_dev): the last plan per operator/request; a call on
    // the same operator enqueues its pipeline with that plan while a host worker thread reads beta
    // back and runs the planner; a different plan re-runs the pipeline (results depend only on
    // (l, n), so a confirmed speculation returns exactly the non-speculative result)
    struct PlanMemo {
        std::shared_ptr<const std::vector<double>> host;
        int p = 0, mode = 0, has_l = 0, l_in = 0;
        double eps = 0.0, c1 = 0.0, c2 = 0.0;
        int l = 0, n = 0;
    };
    std::vector<PlanMemo> plan_memo;
    uint64_t plan_spec_hits = 0, plan_spec_misses = 0;
    // deferred CC convergence checks (engine.cpp phi_call_dev): confirmed / re-run calls
    uint64_t cc_defer_hits = 0, cc_defer_misses = 0;
    struct Worker {
        std::thread th;
        std::mutex mu;
        std::condition_variable cv;
        std::function<void()> job;
        bool has_job = false, busy = false, stop = false;
        std::exception_ptr err;
    };
    std::unique_ptr<Worker> worker;
    cudaEvent_t ev_cc = nullptr;    // adaptive CC error readback completes
    // factor uploads: pinned staging (no implicit stream sync) + per-slot cache of the last
    // operator (reused when the caller passes bit-identical factors again)
    double* pin_fac = nullptr;
    size_t pin_fac_cap = 0;
    // result copies into pinned host memory issued before the end of a call, each followed by an
    // event (note_early_copy): a caller bouncing pageable results can consume them while the device
    // still computes the rest
    struct EarlyCopy {
        cudaEvent_t ev;
        double* host;
        size_t count;
    };
    std::vector<EarlyCopy> early;
    std::vector<cudaEvent_t> ev_early;
    // compute gate (gate_acquire .. gate_enqueued): this call's compute-done events
    std::vector<cudaEvent_t> gate_ev;
    size_t gate_used = 0;
    bool gate_held = false;
    bool gate_covered = false;  // the points cover every stream's compute (else one on c.stream)
    // pinned bounce buffers for pageable host results (capi.cpp run_phiquadmv): name -> (ptr, bytes)
    std::map<std::string, std::pair<double*, size_t>> pin_bounce;
    cudaEvent_t ev_fac = nullptr;
    // slot -> the last uploaded operator: validated host copy, device pointer, norms, canonical map
    struct FacCache {
        int d = 0;
        int n[3] = {0, 0, 0};
        std::shared_ptr<const std::vector<double>> host;
        const double* dev = nullptr;
        double one_norm[3] = {0, 0, 0}, inf_norm[3] = {0, 0, 0};
        int canon[3] = {0, 1, 2};
    };
    std::map<std::string, FacCache> fac_cache;
    // timeline marks while profiling: name, device event, host time (us since first mark)
    struct Mark {
        std::string name;
        cudaEvent_t ev;
        double host_us;
    };
    std::vector<Mark> marks;
    std::string marks_json;
    double phase_ms[6] = {0, 0, 0, 0, 0, 0};
    // GEMM (DMMA) launch records while profiling: (start, stop) events + algorithmic flops
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<double> ev_flops;
    std::vector<std::string> ev_keys;  // launch signature per recorded GEMM (breakdown)
    struct GStat {
        uint64_t launches = 0;
        double ms = 0.0, flops = 0.0, dense = 0.0;
    };
    std::map<std::string, GStat> gstats;
    double prof_ms = 0.0, prof_flops = 0.0;  // prof_flops: executed (negligible blocks skipped)
    double prof_flops_dense = 0.0;            // 2 M N K Z of the same launches
    unsigned long long* d_flops = nullptr;    // per-launch executed-flop counters (profiling)
    uint64_t prof_launches = 0;
    // streaming (HBM-bound) kernel launches while profiling: tag, events around the launch on its
    // stream, algorithmic bytes (every vector read / written once); folded into kstats on collect
    struct KRec {
        const char* tag;
        cudaEvent_t a, b;
        double bytes;
    };
    std::vector<KRec> krecs;
    struct KStat {
        uint64_t launches = 0;
        double ms = 0.0, bytes = 0.0;
    };
    std::map<std::string, KStat> kstats;
};

namespace pqb {

// The Kronecker-sum operator resident on the device.  `scale` multiplies every factor lazily
// (the reference's KroneckerSum::scaled, kron.hpp:44-49, one rounding per entry) -- expm and
// kron_matvec apply it on the fly, so ETD stages never re-upload factors.
struct DevOp {
    int d = 0;
    int n[3] = {1, 1, 1};
    long long N = 1;
    const double* F[3] = {nullptr, nullptr, nullptr};  // device, row-major n_k x n_k (unscaled)
    double one_norm[3] = {0, 0, 0};                    // host: 1-norms of the unscaled factors
    double inf_norm[3] = {0, 0, 0};                    // host: inf-norms of the unscaled factors
    std::shared_ptr<const std::vector<double>> host;   // host copy (concatenated), for host math
    int canon[3] = {0, 1, 2};                          // first dim holding a bit-identical factor
    uint64_t serial = 0;                               // upload serial (per API call)
};

// Epilogue applied at the last mode of a mode chain (see GemmArgs).
struct Epilogue {
    const double* alpha_z = nullptr;
    const double* ext = nullptr;
    long long ext_s = 0;
    const double* coef = nullptr;
    int cld = 0;
    const int* nterms = nullptr;
    int accumulate = 0;
};

// The exponentials one phi call needs (engine.cpp phi_exponentials): per dimension k, the node
// matrices expm((1 - theta_a) 2^-l s A_k) (a < q, stride n_k^2), the squaring chain expm(2^(j-l) s A_k)
// (j < sq_len) and expm(s A_k) for phi_0, with their negligible-block tables.
struct PhiExps {
    const double* node[3] = {nullptr, nullptr, nullptr};
    const double* sq[3] = {nullptr, nullptr, nullptr};
    const double* phi0[3] = {nullptr, nullptr, nullptr};
    int sq_len = 1;
    bool late = false;
    // negligible-block tables parallel to node/sq/phi0 (band_row_blocks(n_k) entries per matrix)
    const int2* node_band[3] = {nullptr, nullptr, nullptr};
    const int2* sq_band[3] = {nullptr, nullptr, nullptr};
    const int2* phi0_band[3] = {nullptr, nullptr, nullptr};
};

// ---- C-ABI error plumbing (capi.cpp owns the thread-local message) ----
std::string& last_error_slot();
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConvergenceFailure& e) {
        last_error_slot() = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        last_error_slot() = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        last_error_slot() = e.what();
        return 4;
    } catch (const std::runtime_error& e) {
        last_error_slot() = e.what();
        return 3;
    } catch (const std::exception& e) {
        last_error_slot() = e.what();
        return 5;
    }
}

// ---- context helpers (engine.cpp) ----
double* ws(pq_ctx& c, const std::string& name, size_t count);          // device doubles
void* ws_bytes(pq_ctx& c, const std::string& name, size_t bytes);
void free_graveyard(pq_ctx& c);     // device-synchronising
void recycle_graveyard(pq_ctx& c);  // cudaFreeAsync on c.stream
void trim_pool(pq_ctx& c);          // returns the pool's unused memory to the driver
void* dev_alloc(pq_ctx& c, size_t bytes, const char* what);  // stream-ordered pool allocation on c.stream
// a workspace-sized allocation (canary-guarded under PQ_WS_GUARD=1) and its release
void* ws_alloc(pq_ctx& c, size_t bytes, const std::string& name);
void ws_retire(pq_ctx& c, void* p);     // into the graveyard (stream-ordered free at the next call)
void ws_free_now(pq_ctx& c, void* p);   // synchronous free (release / destroy)
// canary check of every guarded buffer (syncs); returns the number of damaged buffers, names in *what
int check_guards(pq_ctx& c, std::string* what);
void arena_begin(pq_ctx& c);
const void* arena_push(pq_ctx& c, const void* data, size_t bytes);     // returns device address
void arena_flush(pq_ctx& c);
void count_launch(pq_ctx& c, int n = 1);
// launch_gemm + launch counting + (when profiling) per-launch events and algorithmic flops
int gemm(pq_ctx& c, const GemmArgs& g);
void prof_collect(pq_ctx& c);  // syncs, folds recorded events into prof_ms/prof_flops (and kstats)
// Brackets one streaming-kernel launch on c.stream with events while profiling (no-op otherwise):
// `KernelProbe kp(c, "k_combine", bytes);` before the launch, the scope end records the stop.
struct KernelProbe {
    pq_ctx& c;
    cudaStream_t s = nullptr;
    cudaEvent_t a = nullptr;
    const char* tag;
    double bytes;
    KernelProbe(pq_ctx& ctx, const char* t, double b);
    ~KernelProbe();
    KernelProbe(const KernelProbe&) = delete;
    KernelProbe& operator=(const KernelProbe&) = delete;
};
void note_early_copy(pq_ctx& c, cudaStream_t s, double* host, size_t count);  // after an early D2H on s
// Compute gate: several host-buffer callers on one device compute one after the other, each call's
// kernels queued behind the previous call's compute (device-side event waits, no host blocking on
// the GPU) but not behind its result copies, which drain under the next call's kernels.
// gate_acquire takes the device's gate (host mutex, held while this call enqueues) and makes
// c.stream wait for the last holder's compute-done events; gate_point(c, s) records one on stream s
// (s has only this call's result copies left); gate_enqueued publishes them (plus one on c.stream
// unless c.gate_covered) and passes the gate on; gate_forget drops a context being destroyed.
void dev_copy(pq_ctx& c, double* dst, const double* src, size_t count, cudaStream_t s);  // small D2D on the SMs
void gate_acquire(pq_ctx& c);
void gate_point(pq_ctx& c, cudaStream_t s);
void gate_enqueued(pq_ctx& c);
void gate_forget(pq_ctx& c);
bool gate_wanted(size_t result_bytes);  // PQ_COMPUTE_GATE=1 (default off) and a result of >= 8 MB
void mark(pq_ctx& c, const char* name);  // NVTX marker; timeline mark (device event + host clock) when profiling / tracing
// NVTX range over one C-ABI call (visible under nsys / ncu --nvtx; a few ns when no tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
void check_launch(pq_ctx& c);
void ensure_side(pq_ctx& c);  // creates the side stream and its fork/join events on first use
void run_deferred(pq_ctx& c);

// ---- device building blocks ----
DevOp upload_op(pq_ctx& c, int d, const int* shape, const double* factors, const std::string& slot);
// E[i] = expm(scale[i] * base) for i < count; base is one device n x n matrix (or a strided batch).
void expm_batch(pq_ctx& c, int n, int count, const double* base, long long base_stride,
                const std::vector<double>& scales, double base_one_norm, double* out);
// y[z1] = (E_0[z1] (x) ... (x) E_{d-1}[z1]) x[z1] for z1 < Z1, epilogue fused into the last mode.
// band (nullable, per dim): negligible-block tables of E[k]'s matrices (launch_band_ranges),
// matrix a of E[k] at band[k] + a (E_stride[k]/n_k^2) ceil(n_k/64).
// before_last (optional) runs on the host right before the last mode's GEMM is enqueued (e.g. a
// stream wait that only the epilogue's extra addends need).
void mode_chain(pq_ctx& c, int d, const int* n, const double* const* E, const long long* E_stride,
                const double* x, long long x_stride, double* y, long long y_stride, int Z1, const Epilogue& ep,
                const char* tmp_tag = "chain", const int2* const* band = nullptr,
                const std::function<void()>& before_last = {});
void kron_matvec_dev(pq_ctx& c, const DevOp& op, double scale, const double* x, double* y);
// one mode product of nb columns (no band table): the GEMM the mode chain issues for `mode`
GemmArgs mode_gemm_public(int d, const int* n, int mode, const double* E, const double* x, double* y, int nb,
                          long long N);
void exp_action_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* b, double* y);
double max_inf_norm_dev(pq_ctx& c, const double* v, long long N, int ncols);  // syncs

// phi pipeline on device pointers.  `scale` multiplies the operator (e.g. -sigma*tau).
void phi_fixed_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p,
                   const NodesWeights& rule, double* out);
void phi_adaptive_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p, double eps,
                      double* out, int* points_used);
void squaring_steps_dev(pq_ctx& c, const DevOp& op, double scale, int nb, int p, int l, double* y,
                        const double* exps_override = nullptr);
void phi_with_plan_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p, int l, int n,
                       int kind, double eps, double* out, int* points_used);
struct PlanInfo {
    int l = 0, n = 0, points = 0, mode = 0, planned = 0;
    double alpha = 0, beta = 0, cost = 0;
};
// phiquadmv's planner (phiaction.hpp:307-340): alpha from the factor norms, beta = max ||b||_inf
// read back from the device (one sync), then setup_quadrature / quadnodes.  points is left 0.
PlanInfo plan_phi(pq_ctx& c, const DevOp& op, int nb, const double* bs, int p, double eps, int mode, bool has_l, int l,
                  double c1, double c2);
// The planner on a host worker thread of the context (one job at a time): submit, then wait
// (rethrows the job's exception).  worker_stop joins the thread (pq_ctx_destroy).
void worker_submit(pq_ctx& c, std::function<void()> job);
void worker_wait(pq_ctx& c);
void worker_stop(pq_ctx& c);
// Enqueues the Taylor powers of op's factors at `scale` (they do not depend on the plan), so they
// run while the host waits for beta and plans; phi_exponentials of the same call reuses them.
void taylor_prefetch(pq_ctx& c, const DevOp& op, double scale);
// phi0_host (optional, pinned host memory): phi_0 is also copied there as soon as it is computed,
// on the side stream while the squaring runs (joined before the call returns).  out_host
// (optional, pinned): the phi columns are copied there per column half as each half finishes
// (two-stream squaring only; *out_copied says whether it happened).
void phiquadmv_dev(pq_ctx& c, const DevOp& op, int nb, const double* bs, int p, double eps, int mode, bool has_l,
                   int l, double c1, double c2, double* out, PlanInfo* info, double* phi0_out = nullptr,
                   double* phi0_host = nullptr, double* out_host = nullptr, bool* out_copied = nullptr);
void phi_nodes_partial_dev(pq_ctx& c, const DevOp& op, double scale, int nb, const double* bs, int p,
                           const NodesWeights& rule, const std::vector<int>& nodes, int zero, double* acc);
PhiExps phi_exponentials(pq_ctx& c, const DevOp& op, double s, int l, const std::vector<double>& thetas,
                         bool want_sq, bool want_phi0, const std::string& tag, bool sq_chain = false,
                         bool late_async = false);
void apply_phi0(pq_ctx& c, const DevOp& op, const PhiExps& px, int nb, const double* b, double* y);
// phiaction.hpp:102-107 coefficients w_i theta_i^(j-1)/(j-1)! of the nodes idx, [a][p]
void node_coefs(const NodesWeights& r, const std::vector<int>& idx, int p, std::vector<double>& out);
std::vector<double> thetas_of(const NodesWeights& r, const std::vector<int>& idx);
// q node vectors v_a = (E_a0 (x) E_a1 (x) E_a2) b_m (E[k] + a*Es[k]): combined into acc [nb][p][N]
// with coef [q][p], or (pool != null) stored at pool + ((slot0 + a)*nb + m)*N
void node_sweep(pq_ctx& c, const DevOp& op, const double* const* E, const long long* Es, int q, int nb,
                const double* bs, int p, const std::vector<double>* coef, double* acc, int zero, double* pool,
                int slot0, const int2* const* band = nullptr);
// one mode-k product of Z1 tensors of shape n[0..d) (x[z] at x + z*x_stride, y[z] likewise) with
// ONE matrix E (band: its negligible-block table or null): y[z] = (I (x) .. E .. (x) I) x[z]
// remote (device table, nullable): the outputs go to other ranks' buffers (dist.cpp peer transport)
void mode_product_dev(pq_ctx& c, int d, const int* n, int k, const double* E, const int2* band, const double* x,
                      long long x_stride, double* y, long long y_stride, int Z1, const RemoteMap* remote = nullptr);
void phi_lincomb_dev(pq_ctx& c, const DevOp& op, double scale, int p, const double* bs, const NodesWeights& rule,
                     double* out);

}  // namespace pqb
