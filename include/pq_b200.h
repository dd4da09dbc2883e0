/*
 * pq_b200.h — the C-ABI boundary of the B200-native phi-function action engine.
 *
 * The reference (arXiv 2211.00696, `phiquad`) is a header-only C++20 library; its "FFI" for
 * the hot path is the C++ API in proj/include/phiquad/*.hpp.  This header is the flat C layer
 * under our drop-in copy of that API (include/phiquad/*.hpp, same names and signatures):
 * every C++ entry point there is a thin wrapper that calls exactly one function below and
 * rethrows the return code as the reference's exception type.  Plain pointers and sizes only,
 * no torch or CUDA types: a `void*` stream is a cudaStream_t.
 *
 * Conventions (same as the reference unless stated):
 *  - vectors are in vec order: row-major over `shape`, leftmost factor slowest
 *    (reference kron.hpp:13-15);
 *  - a Kronecker-sum argument is (d, shape[d], factors) where `factors` is the HOST
 *    concatenation of d row-major shape[k] x shape[k] blocks (reference KroneckerSum,
 *    kron.hpp:16-53); factors are validated (finite, 1..3 square factors);
 *  - `space` says where every vector argument of the call lives: PQ_HOST (pageable or pinned
 *    host memory; the call stages copies and synchronises) or PQ_DEVICE (device pointers on the
 *    context's GPU; the call is stream-ordered on the context stream and returns once the work
 *    is enqueued, except where a host decision needs device data — noted per function);
 *  - phi outputs are laid out [nb][p][N]: right-hand side m, column j (phi_{j+1}).
 *  - return codes map 1:1 to the reference's exceptions (see PQ_E*); the message of the last
 *    failure on the calling thread is pq_last_error().
 *  - there is NO CPU fallback: without a usable sm_100 device every device entry point fails
 *    with PQ_ERUNTIME.
 */
#ifndef PQ_B200_H
#define PQ_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define PQ_API __attribute__((visibility("default")))
#else
#define PQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* return codes ------------------------------------------------------------------------------ */
enum {
    PQ_OK = 0,
    PQ_EINVAL = 1,        /* std::invalid_argument            (shape, p, l, eps, guards)    */
    PQ_ECONVERGENCE = 2,  /* phiquad::ConvergenceError         (util.hpp:11-14)              */
    PQ_ERUNTIME = 3,      /* std::runtime_error                (singular LU, CUDA failures)  */
    PQ_ERANGE = 4,        /* std::out_of_range                 (PhiColumns::col)             */
    PQ_EINTERNAL = 5
};

enum { PQ_GAUSS_LEGENDRE = 0, PQ_CLENSHAW_CURTIS = 1 }; /* reference QuadKind, quadrature.hpp:14 */
enum { PQ_HOST = 0, PQ_DEVICE = 1 };

typedef struct pq_ctx pq_ctx;

PQ_API const char* pq_version(void);
PQ_API const char* pq_last_error(void);

/* context: one device, one stream, a growable device workspace --------------------------- */
PQ_API int pq_ctx_create(int device, pq_ctx** out);
PQ_API int pq_ctx_destroy(pq_ctx* ctx);
/* Use an external stream (e.g. torch.cuda.current_stream().cuda_stream); NULL = own stream;
 * the legacy default stream is (void*)1 (cudaStreamLegacy), not NULL. */
PQ_API int pq_ctx_set_stream(pq_ctx* ctx, void* cuda_stream);
PQ_API void* pq_ctx_stream(const pq_ctx* ctx);
PQ_API int pq_ctx_synchronize(pq_ctx* ctx);
/* Number of kernels this context has launched so far (evidence for bench.py gpu_launches). */
PQ_API uint64_t pq_ctx_launches(const pq_ctx* ctx);
/* Device memory budget for the workspace in bytes (0 = 85% of free memory at first use). */
PQ_API int pq_ctx_set_workspace_limit(pq_ctx* ctx, uint64_t bytes);
PQ_API int pq_ctx_release_workspace(pq_ctx* ctx);
/* Device time (ms) spent in each phase of the last phi call: [0] planner+setup (host, wall),
 * [1] batched expm, [2] node sweep (mode products), [3] node combine, [4] squaring,
 * [5] phi_0 exp-action.  Only filled when profiling is on (adds events, no syncs). */
PQ_API int pq_ctx_set_profiling(pq_ctx* ctx, int on);
PQ_API int pq_ctx_phase_times(pq_ctx* ctx, double* ms6);
/* With profiling on, every DMMA GEMM launch (mode products and expm products) is bracketed by
 * CUDA events on the context stream.  Returns (synchronising) the number of such launches, their
 * summed device time in ms and the FLOPs their CTAs executed (negligible exponential blocks
 * skipped; counted on the device). */
PQ_API int pq_ctx_gemm_stats(pq_ctx* ctx, int reset, uint64_t* launches, double* ms, double* flops);
/* Same launches: 2*M*N*K per batch entry, i.e. the dense mode-product work of the reference's
 * algorithm (kron.hpp:65-108) without any block skipped. */
PQ_API int pq_ctx_gemm_dense_flops(pq_ctx* ctx, int reset, double* flops);
/* With profiling on, every streaming (HBM-bound) kernel launch -- node combines, squaring
 * combinations, column statistics, ETD stage kernels -- is bracketed by events on its stream.
 * Returns (synchronising) a JSON object {"<kernel>": {"launches", "ms", "bytes"}} with the summed
 * device time and ALGORITHMIC bytes (each vector read / written once) per kernel tag. */
PQ_API int pq_ctx_kernel_stats(pq_ctx* ctx, int reset, const char** json);
/* The profiled DMMA GEMM launches grouped by call site and shape: JSON {"<site> M.. N.. K.. Z..":
 * {"launches", "ms", "flops" (executed), "dense"}} (synchronising). */
PQ_API int pq_ctx_gemm_breakdown(pq_ctx* ctx, int reset, const char** json);
/* Debug (environment PQ_WS_GUARD=1 at first use): every workspace buffer is allocated with 4 KB
 * canary regions before and after it.  Synchronises and counts the buffers whose canaries were
 * overwritten (*damaged; their names in pq_last_error()) -- an out-of-bounds-write check that needs
 * no compute-sanitizer. */
PQ_API int pq_ctx_check_guards(pq_ctx* ctx, int* damaged);
/* With profiling on, phase boundaries are marked (device event + host clock).  Returns (and
 * clears, synchronising) a JSON array [{"mark","gpu_us","host_us"}] relative to the first mark. */
PQ_API int pq_ctx_timeline(pq_ctx* ctx, const char** json);

/* host estimator: rules, roots, bounds, planner (no GPU) --------------------------------- */
/* quadrature.hpp:31 gauss_legendre, :67 clenshaw_curtis — ascending nodes on [0,1]. */
PQ_API int pq_gauss_legendre(int m, double* nodes, double* weights);
PQ_API int pq_clenshaw_curtis(int m, double* nodes, double* weights);
/* quadrature.hpp:90 cached_rule — pointers stay valid for the process lifetime. */
PQ_API int pq_cached_rule(int kind, int m, const double** nodes, const double** weights);
/* roots.hpp:34 quartic_roots: coeffs = {a3, a2, a1, a0}; roots = 4 x (re, im). */
PQ_API int pq_quartic_roots(const double* coeffs4, double* roots8);
/* roots.hpp:88 real_roots_greater_one: up to 4 ascending roots, *count of them. */
PQ_API int pq_real_roots_greater_one(const double* coeffs4, double* roots4, int* count);
/* bounds.hpp:71 / :88 / :107 / :122 / :146 — log-domain bounds. */
PQ_API int pq_log_bound_at_rho(double n, int p, double alpha, double beta, int kind, double rho, double* out);
PQ_API int pq_bound_quartic(double n, int p, double alpha, double beta, int kind, double* coeffs4);
PQ_API int pq_theorem_bound(double n, int p, double alpha, double beta, int kind, double* out);
PQ_API int pq_corollary_bound(double n, int p, double alpha, double beta, int kind, double* out);
PQ_API int pq_quaderr(double n, int p, double alpha, double beta, int kind, double* out);
/* bounds.hpp:159 quadnodes, :185 setup_quadrature (CostModel {c1, c2, d}). */
PQ_API int pq_quadnodes(double eps, int p, double alpha, double beta, int kind, int* n);
PQ_API int pq_setup_quadrature(double eps, int p, double alpha, double beta, int kind, double c1, double c2,
                        int d, int* l, int* n, double* cost);
/* kron.hpp:131 infnorm_bound (host, exact sum of factor inf-norms). */
PQ_API int pq_infnorm_bound(int d, const int* shape, const double* factors, double* out);

/* dense / Kronecker primitives on the device ---------------------------------------------- */
/* dense.hpp:194 expm for a batch: out[i] = expm(scale[i] * a) (scale NULL = 1). a and out are
 * in `space`; a is ONE n x n matrix shared by the batch. */
PQ_API int pq_expm(pq_ctx* ctx, int n, int batch, const double* a, const double* scale, double* out, int space);
/* kron.hpp:92 mode_apply: y = (M_0 (x) ... (x) M_{d-1}) x; mats host-side like factors. */
PQ_API int pq_mode_apply(pq_ctx* ctx, int d, const int* shape, const double* mats, const double* x, double* y,
                  int space);
/* kron.hpp:111 kron_matvec: y = A x without assembly. */
PQ_API int pq_kron_matvec(pq_ctx* ctx, int d, const int* shape, const double* factors, const double* x,
                   double* y, int space);
/* kron.hpp:123 exp_action (phi_0): y = e^A b. */
PQ_API int pq_exp_action(pq_ctx* ctx, int d, const int* shape, const double* factors, const double* b,
                  double* y, int space);

/* phi engine (phiaction.hpp) -------------------------------------------------------------- */
typedef struct {
    int p;          /* PhiRequest::p                                      */
    double eps;     /* PhiRequest::eps (reference default 1e-14)          */
    int mode;       /* PQ_GAUSS_LEGENDRE / PQ_CLENSHAW_CURTIS             */
    int has_l;      /* PhiRequest::l engaged?                             */
    int l;
    double c1, c2;  /* CostModel weights (reference defaults 0, 1)        */
    int threads;    /* accepted for API parity; results never depend on it */
} pq_phi_request;

typedef struct {
    int l, n, points, mode, planned;
    double alpha, beta, plan_cost;
} pq_phi_info; /* PhiInfo, phiaction.hpp:45-54 */

/* phiaction.hpp:134 phi_fixed_multi on an explicit rule (m ascending nodes/weights, host). */
PQ_API int pq_phi_fixed(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb, const double* bs,
                 int p, int m, const double* nodes, const double* weights, double* out, int space);
/* phiaction.hpp:156 phi_adaptive_multi (CC ladder 7 -> 13 -> 25 ...). Synchronises once per level. */
PQ_API int pq_phi_adaptive(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb,
                    const double* bs, int p, double eps, double* out, int* points_used, int space);
/* The same with the caller's vectors as they are (the drop-in headers' phi_fixed(_multi) /
 * phi_adaptive(_multi)): RHS m at bs[m], phi_{j+1} of RHS m to cols[m*p + j] (N doubles each). */
PQ_API int pq_phi_fixed_cols(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb,
                             const double* const* bs, int p, int m, const double* nodes, const double* weights,
                             double* const* cols, int space);
PQ_API int pq_phi_adaptive_cols(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb,
                                const double* const* bs, int p, double eps, double* const* cols, int* points_used,
                                int space);
/* phiaction.hpp:255 squaring_step: y [p][N] rewritten in place to phi_j(2A). exps host-side. */
PQ_API int pq_squaring_step(pq_ctx* ctx, int d, const int* shape, const double* exps, int p, double* y,
                     int space);
/* squaring_step on the caller's column vectors in place (cols[j], N doubles each). */
PQ_API int pq_squaring_step_cols(pq_ctx* ctx, int d, const int* shape, const double* exps, int p,
                                 double* const* cols, int space);
/* phiaction.hpp:277 phi_with_plan. */
PQ_API int pq_phi_with_plan(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb,
                     const double* bs, int p, int l, int n, int kind, double eps, double* out,
                     int* points_used, int space);
/* phiaction.hpp:277 phi_with_plan with the caller's vectors as they are: RHS m at bs[m], phi_{j+1}
 * of RHS m to cols[m*p + j] (the drop-in headers' phi_with_plan and PhiEngine::apply). */
PQ_API int pq_phi_with_plan_cols(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb,
                                 const double* const* bs, int p, int l, int n, int kind, double eps,
                                 double* const* cols, int* points_used, int space);
/* phiaction.hpp:307 phiquadmv_multi (plans from alpha = infnorm_bound, beta = max ||b||_inf;
 * reads beta back from the device, i.e. synchronises once before planning). */
PQ_API int pq_phiquadmv(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb, const double* bs,
                 const pq_phi_request* req, double* out, pq_phi_info* info, int space);
/* phiaction.hpp:307 phiquadmv_multi with the caller's vectors as they are: RHS m at bs[m], and
 * phi_{j+1}(A) b_m written to cols[m*p + j] (each N doubles).  The drop-in headers call this so a
 * std::vector RHS and the PhiColumns vectors are read / written in place (no flattening copies). */
PQ_API int pq_phiquadmv_cols(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb,
                             const double* const* bs, const pq_phi_request* req, double* const* cols,
                             pq_phi_info* info, int space);
/* phiquadmv plus phi_0 = exp_action for every RHS: out0 [nb][N], out [nb][p][N] — the
 * "phi_0..phi_p action" the benchmark counts. */
PQ_API int pq_phi_0p(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb, const double* bs,
              const pq_phi_request* req, double* out0, double* out, pq_phi_info* info, int space);
/* phiaction.hpp:355 phi_lincomb: y = sum_j phi_j(A) b_j on an explicit rule (no squaring). */
PQ_API int pq_phi_lincomb(pq_ctx* ctx, int d, const int* shape, const double* factors, int p, const double* bs,
                   int m, const double* nodes, const double* weights, double* out, int space);

/* Node-sharded partial sums for multi-GPU runs (one process per GPU): accumulates, into
 * acc [nb][p][N] (zeroed first when `zero` != 0), the weighted node vectors of the GL rule
 * nodes i with i % world == rank, on 2^-l A, in ascending i.  Summing the ranks' acc in rank
 * order and then applying pq_squaring_chain reproduces pq_phi_with_plan up to rounding.
 * Device pointers only. */
PQ_API int pq_phi_nodes_partial(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb,
                         const double* bs, int p, int l, int m, const double* nodes,
                         const double* weights, int rank, int world, int zero, double* acc);
/* l modified-squaring steps on y [nb][p][N] with E = expm(2^-l A_k) (phiaction.hpp:290-301). */
PQ_API int pq_squaring_chain(pq_ctx* ctx, int d, const int* shape, const double* factors, int nb, int p, int l,
                      double* y);
/* Building blocks of the distributed squaring (paper_2211_00696_b200/sharded.py):
 * one mode product y[b] = (I (x) .. E .. (x) I) x[b] along `mode` of a d-way tensor of the given
 * shape, for nb columns of length prod(shape) (kron.hpp:65-87 accumulate_mode_apply, one mode),
 * and one modified-squaring combination in place, T_i <- 2^-i (T_i + sum_{j<=i} Y_j/(i-j)!) for
 * the p columns of each of nb right-hand sides laid out [nb][p][N] (phiaction.hpp:260-268; T holds
 * E y_i on entry, Y the old y).  Device pointers only. */
PQ_API int pq_mode_product(pq_ctx* ctx, int d, const int* shape, int mode, const double* E, int nb,
                           const double* x, double* y);
PQ_API int pq_squaring_combine(pq_ctx* ctx, long long n, int p, int nb, double* t, const double* y);

/* multi-GPU (one process per GPU; paper_2211_00696_b200/csrc/dist.cpp) ------------ */
/* The reference's node loop (phiaction.hpp:85 parallel_for, util.hpp:24-39) and its serial
 * squaring (phiaction.hpp:255-272, 293-301), partitioned over the ranks of a communicator:
 * quadrature nodes dealt round-robin (i % world == rank; each adaptive-CC level's fresh nodes
 * likewise), ONE all-to-all moving each node vector's x-slab to its owner (rank r owns the
 * x-indices [floor(n0 r/G), floor(n0 (r+1)/G)), a contiguous range of every vector, see
 * pq_dist_slab), the weighted node sums formed per slab in ascending node order (the node phase is
 * bitwise independent of the rank count), the adaptive-CC error as one exact all-reduce(max) of
 * 2 nb p scalars per level, and the modified squaring + phi_0 on slabs (modes 1..d-1 in the slab,
 * slab <-> pencil all-to-alls around mode 0).  Every rank passes the SAME inputs (factors, b, request). */
enum { PQ_COMM_NCCL = 0, PQ_COMM_HOST = 1, PQ_COMM_PEER = 2 };
typedef struct pq_comm pq_comm;
/* Host transport: collectives on pinned HOST buffers, e.g. torch.distributed over gloo, so several
 * processes can share one GPU in tests (no kernel ever waits on another process).  alltoallv sends
 * send_counts[h] doubles (consecutive, in rank order) to rank h and receives recv_counts[h] doubles
 * from rank h into recv (consecutive, in rank order); allreduce_max is an in-place elementwise max
 * over ranks.  Return 0 on success. */
typedef struct {
    void* user;
    int (*alltoallv)(void* user, const double* send, const int64_t* send_counts, double* recv,
                     const int64_t* recv_counts);
    int (*allreduce_max)(void* user, double* buf, int64_t n);
} pq_host_transport;
/* NCCL (loaded at run time: the libnccl.so.2 already mapped in the process, else the system one,
 * or $PQ_NCCL_LIB): rank 0 makes the 128-byte id, every rank passes it (broadcast by any means). */
PQ_API int pq_nccl_unique_id(char* out128);
PQ_API int pq_comm_create_nccl(pq_ctx* ctx, int world, int rank, const char* id128, pq_comm** out);
PQ_API int pq_comm_create_host(int world, int rank, const pq_host_transport* transport, pq_comm** out);
/* Peer transport: the squaring's slab <-> pencil flips are fused into the mode products -- their
 * epilogues store each output row straight into the owning rank's buffer through CUDA IPC mappings
 * (NVLink between the GPUs of a node; processes sharing one GPU in the tests), no pack / unpack
 * kernels and no staging.  The host transport carries the IPC-handle exchange and the per-flip
 * barrier (each rank drains its stream, then the allreduce acts as the barrier) and the remaining
 * exchanges.  Applies to 3-D operators whose second extent the world size divides; other shapes
 * fall back to the host transport's packed exchanges. */
PQ_API int pq_comm_create_peer(pq_ctx* ctx, int world, int rank, const pq_host_transport* transport, pq_comm** out);
PQ_API int pq_comm_destroy(pq_comm* comm);
/* Bytes this rank sent to other ranks and exchanges issued since the last reset. */
PQ_API int pq_comm_stats(pq_comm* comm, int reset, double* bytes_sent, uint64_t* exchanges);
/* [begin, end) of rank's x-slab inside a vector of the given shape. */
PQ_API int pq_dist_slab(int d, const int* shape, int world, int rank, int64_t* begin, int64_t* end);
/* phiquadmv_multi (+ phi_0 when out0 != NULL) across the communicator.  gather != 0: out [nb][p][N]
 * and out0 [nb][N] hold full vectors on every rank; gather == 0: this rank's slabs, out
 * [nb][p][end-begin], out0 [nb][end-begin].  The plan is computed identically on every rank. */
PQ_API int pq_phiquadmv_dist(pq_ctx* ctx, pq_comm* comm, int d, const int* shape, const double* factors, int nb,
                             const double* bs, const pq_phi_request* req, double* out0, double* out,
                             pq_phi_info* info, int space, int gather);
/* phi_with_plan (phiaction.hpp:277) across the communicator, layouts as pq_phiquadmv_dist. */
PQ_API int pq_phi_with_plan_dist(pq_ctx* ctx, pq_comm* comm, int d, const int* shape, const double* factors,
                                 int nb, const double* bs, int p, int l, int n, int kind, double eps, double* out,
                                 int* points_used, int space, int gather);

/* exponential integrators (integrators.hpp) ----------------------------------------------- */
/* Increment-form tableau (ExpRKTableau, integrators.hpp:32-38) flattened into terms: a term
 * with row >= 1 is a_{row,col} += coef * phi_k, row == -1 is b_col += coef * phi_k. */
typedef struct {
    int stages, order;
    const double* c;  /* stages */
    int nterms;
    const int* row;
    const int* col;
    const int* k;
    const double* coef;
} pq_tableau;

enum {
    PQ_SOURCE_ZERO = 0,       /* f = 0                                         */
    PQ_SOURCE_CUBIC = 1,      /* f(t,u) = s1*u + s3*u^3 (Allen-Cahn: s1=1, s3=-1), device kernel */
    PQ_SOURCE_CONSTANT = 2,   /* f = given vector (space of the call)          */
    PQ_SOURCE_CALLBACK = 3    /* host callback, vectors staged through host     */
};
typedef int (*pq_source_cb)(double t, const double* u, double* f, int64_t n, void* user);
typedef struct {
    int kind;
    double s1, s3;
    const double* vec;
    pq_source_cb cb;
    void* user;
} pq_source;

/* integrators.hpp:41-76 and our ETDRK4: id 0 exp_euler, 1 exp_rk2(c2), 2 exp_rk3(c2), 3 etdrk4.
 * Fills a static tableau (pointers valid for the process lifetime). */
PQ_API int pq_builtin_tableau(int id, double c2, pq_tableau* out);
/* integrators.hpp:193 integrate: m steps of erk_step with a PhiEngine (plans per (sigma,p), beta = 1). */
PQ_API int pq_integrate(pq_ctx* ctx, int d, const int* shape, const double* factors, const pq_source* f,
                 const double* u0, double t0, double t_end, int m, const pq_tableau* tab,
                 const pq_phi_request* base, double* u_out, int* phi_calls, int space);
/* integrators.hpp:160 erk_step with a fresh engine for step size tau. */
PQ_API int pq_erk_step(pq_ctx* ctx, int d, const int* shape, const double* factors, const pq_source* f,
                double tau, double t, const double* u, const pq_tableau* tab,
                const pq_phi_request* base, double* u_out, int* phi_calls, int space);

#ifdef __cplusplus
}
#endif
#endif /* PQ_B200_H */
