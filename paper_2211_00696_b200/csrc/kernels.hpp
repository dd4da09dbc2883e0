// Device kernels of the phi engine and their host-side launchers (all stream-ordered, no syncs).
#pragma once
#include <cstdlib>

#include <cuda_runtime.h>
#include <cstdint>

namespace pqb {

// Batched FP64 GEMM on the DMMA tensor pipe, the engine's only FLOP sink:
//   C[z][m][n] = alpha(z1) * sum_k A[z][m][k] B[z][k][n]  (+ C_old if accumulate)
//                + sum_{t < nterms(z1)} coef[z1*cld + t] * ext[t*ext_s + z2*sC2 + m*ldc + n]
// A is row-major (k contiguous).  B is row-major K x N ("n contiguous") or, when b_kmajor, stored
// as N x K rows ("k contiguous").  z = z1*zdiv + z2 indexes a two-level batch with independent
// strides, which maps every mode product of the engine (node-batched, column-batched, shared
// inputs with stride 0) onto one launch.
// Remote-store epilogue of the multi-GPU peer transport (dist.cpp): output rows go straight to
// other ranks' buffers (CUDA IPC mappings; NVLink stores between GPUs) instead of C.
//   mode 1, slab -> pencil (the last slab mode, rows m = r*n1 + i1 of column z1): rank h = owner of the
//     trailing index i1*n2; destination base[h] + (z1*n0 + s[me] + r)*(cb[h+1]-cb[h]) + i1*n2 - cb[h];
//   mode 2, pencil -> slab (mode 0 on the pencil, rows i0 of column z1): rank h = owner of i0;
//     destination base[h] + (z1*(s[h+1]-s[h]) + i0 - s[h])*rest + cb[me].
struct RemoteMap {
    int mode = 0, G = 1, me = 0, n0 = 1, n1 = 1, n2 = 1;
    long long rest = 1;
    int s[17] = {0};
    long long cb[17] = {0};
    double* base[16] = {nullptr};
};

struct GemmArgs {
    const double* A = nullptr;
    const double* B = nullptr;
    double* C = nullptr;
    int M = 0, N = 0, K = 0;
    long long lda = 0, ldb = 0, ldc = 0;
    int b_kmajor = 0;
    int Z = 1, zdiv = 1, z_off = 0;
    long long sA1 = 0, sA2 = 0, sB1 = 0, sB2 = 0, sC1 = 0, sC2 = 0;
    double alpha = 1.0;
    const double* alpha_z = nullptr;  // per z1 (device)
    const double* ext = nullptr;      // extra addends (device)
    long long ext_s = 0;              // stride between addend vectors
    int ext_group = 1;                // batch z1 reads addends (z1/ext_group)*ext_group + t
    const double* coef = nullptr;     // per z1 rows of cld coefficients (device)
    int cld = 0;
    const int* nterms = nullptr;      // per z1 (device)
    int accumulate = 0;
    const int* sq_count = nullptr;    // expm squaring: z with sq_round >= sq_count[z] copies A
    int sq_round = 0;
    // Negligible-block skip for mode products (the 32x128x16 / 64x32x16 band tiles, launch_gemm
    // shapes 6 / 7): band[e*band_stride + rb] =
    // {first, last+1} 8-wide k-slices of 32-row block rb of exponential e that hold any entry above
    // 2^-64 max|E| (launch_band_ranges).  The CTA streams the union of the 32-row blocks it covers; each
    // warp issues DMMAs only inside its own block's range.  band_mode 1: A = exponentials stacked
    // along M (e = m0 / band_rows); 2: A = exponential z1; 3: B (k-major) = exponential z1, rows
    // from n0.
    const int2* band = nullptr;
    long long band_stride = 0;
    int band_mode = 0, band_rows = 0;
    // profiling: every CTA adds the flops it actually executed (2 rows cols k) here
    unsigned long long* flop_counter = nullptr;
    const char* tag = nullptr;  // call site, for the profiling breakdown only
    const RemoteMap* remote = nullptr;  // device table: remote-store epilogue (plain stores only)
};
int launch_gemm(const GemmArgs& g, cudaStream_t s);  // returns number of kernel launches
// Fused last two modes of a 3-D apply with n1 = n2 = 128 (slab12.cu): for every x-slab
// X_s = X[z1][i0] (128 x 128), Y_s = (E1 X_s) E2^T, bitwise the two separate band tiles.
// Batch entry z1 < Z1 uses E1 + z1*sE1, E2 + z1*sE2, band tables band1 + z1*sband1 (4 int2,
// null = full K), X + z1*sX, Y + z1*sY; n0 slabs per entry.
struct Slab12Args {
    const double* E1 = nullptr;
    long long sE1 = 0;
    const double* E2 = nullptr;
    long long sE2 = 0;
    const int2* band1 = nullptr;
    long long sband1 = 0;
    const int2* band2 = nullptr;
    long long sband2 = 0;
    // fragment-major copies of the E2 matrices (launch_band_ranges pack; null = read E2 row-major)
    const double* E2p = nullptr;
    long long sE2p = 0;
    const double* X = nullptr;
    long long sX = 0;
    double* Y = nullptr;
    long long sY = 0;
    int n0 = 1, Z1 = 1;
    long long z_off = 0;
    unsigned long long* flop_counter = nullptr;
};
bool slab12_supported(int n1, int n2);
int launch_slab12(const Slab12Args& g, cudaStream_t s);  // returns number of kernel launches
// `count` dependent batched GEMM levels (plain products, row-major B, 16-byte aligned) in ONE
// cooperative launch with a grid barrier between levels; bar = one device unsigned (zeroed by
// the launcher).  Returns 1, or 0 when the chain does not qualify (the caller launches per level).
int launch_gemm_chain(const GemmArgs* levels, int count, unsigned* bar, cudaStream_t s);

// ---- batched Pade-13 expm building blocks (dense.hpp:194-228) ----
// X[z] = (scale[z] * (op_scale * base)) * 2^-s_z  (each product rounded, as the reference's
// KroneckerSum::scaled then DenseMatrix scaled), s_z from the 1-norm of the rounded argument.
// base_off (device, nullable) gives each batch entry its own base matrix offset.
void launch_expm_prep(int n, int count, const double* base, long long base_stride, const long long* base_off,
                      double op_scale, const double* scale, double* X, int* s_out, cudaStream_t s);
// ---- shared-power Taylor exponentials (engine.cpp expm_taylor) ----
constexpr int kTaylorChunk = 8;  // entries per combination block (same factor)
// P[f*m*n^2 ...] = f_pow2[f] * fl(op_scale * base[f_off[f] ...]) for f < nf (first power, normalised)
void launch_taylor_base(int n, int nf, int m, const double* base, const long long* f_off, double op_scale,
                        const double* f_pow2, double* P, cudaStream_t s);
// chunks: nchunks x int4 {factor, first entry, entry count, 0}; coef: [entry][m+1] Taylor weights;
// P: [factor][power 1..m][n x n]; out[entry] = sum_k coef[entry][k] P_factor^k (P^0 = I).
// m in {16, 18, 20, 24, 28, 32}.
void launch_taylor_combine(int n, int m, int nchunks, const int* chunks, const double* coef, const double* P, double* out,
                           cudaStream_t s);
// out = op_scale * a (elementwise, rounded once)
void launch_scale_copy(long long total, double op_scale, const double* a, double* out, cudaStream_t s);
void launch_pade_mid(int n, int count, const double* A2, const double* A4, const double* A6, double* T1,
                     double* Zc, cudaStream_t s);
void launch_pade_fin(int n, int count, const double* W, const double* Z, const double* A2, const double* A4,
                     const double* A6, double* W2, double* V, cudaStream_t s);
void launch_pade_pq(long long total, const double* V, const double* U, double* P, double* Q, cudaStream_t s);
// Solves P X = Q in place (X -> Q) with partial pivoting, one CTA per matrix; err[0] = 1 on a zero pivot.
void launch_lu_solve(int n, int count, double* P, double* Q, int* err, cudaStream_t s);
// n <= 128: shared-memory factorisation of P (L\U over P, pivots in piv[count*n]) + a batched
// triangular solve of Q over 32-column slices.  Q <- P^{-1} Q.
void launch_lu_factor_solve(int n, int count, double* P, double* Q, int* piv, int* err, cudaStream_t s);
// Per matrix z < count (n x n, stride n*n) a record of band_row_blocks(n) int2 (RB = ceil(n/32)):
//  rec[rb], rb < RB: {first, last+1} of the 8-wide column slices of 32-row block rb whose max |E|
//    exceeds 2^-64 x the row block's max (<= max|E_z|; NaN/Inf count as needed; an all-zero row
//    block gives an empty range) -- the k-slices a tile streams;
//  rec[RB + g], g < 4 RB: {first, last+1} of the 4-wide column chunks (DMMA k4 steps) of 8-row
//    group g whose max |E| exceeds 2^-64 x the group's max -- the k4 steps a DMMA row (or column,
//    for a k-major exponential) fragment issues.
// Dropping the rest changes a mode product by at most n 2^-64 of its max-norm -- below half an ulp
// in practice.
void launch_band_ranges(int n, int count, const double* E, int2* out, cudaStream_t s, double* pack = nullptr);
// doubles per matrix of the fragment-major copy launch_band_ranges writes into `pack` (k_slab12 phase 2)
inline long long band_pack_doubles(int n) { return static_cast<long long>((n + 7) / 8) * ((n + 3) / 4) * 32; }
inline int band_row_blocks(int n) { return 5 * ((n + 31) / 32); }  // record length (int2)
// max over z of s_z -> *out (device int)
void launch_imax(const int* v, int count, int* out, cudaStream_t s);

// ---- HBM-bound helpers ----
// acc[j][t] = (zero ? 0 : acc[j][t]) + sum_{i ascending} coef[i*p + j] * V[slot[i]][t]
// (exact reference order: separate multiply and add per node, phiaction.hpp:96-111).
void launch_combine(long long N, int p, int q, const double* V, long long vstride, const int* slots,
                    const double* coef, double* acc, long long acc_stride, int zero, cudaStream_t s);
// In-place doubling combination of a squaring step: T_i <- 2^-i T_i + sum_{j<=i} coef[i*p+j] Y_j
// (coef[i][j] = 2^-(i+1)/(i-j)!), columns laid out [nb][p][N].
// Columns i0 <= i < i1 only (default: all p); T_i reads Y_j for j <= i only.
void launch_sq_combine(long long N, int p, int nb, double* T, const double* Y, const double* coef, cudaStream_t s,
                       int i0 = 0, int i1 = -1);
// Fused adaptive-CC level (k_combine + coarse rule + k_colstats): acc[j] = sum_i cf[i][j] V[slots[i]];
// coarse = sum_i cc[i][j] V[slots[i]] (cc != null) or prev[j] (prev != null); stats[2j] max|acc_j -
// coarse_j|, stats[2j+1] max|acc_j| (atomic max: zero stats first).  False when p > 8.
bool launch_combine_stats(long long N, int p, int q, const double* V, long long vstride, const int* slots,
                          const double* cf, const double* cc, const double* prev, double* acc, long long acc_stride,
                          double* stats, cudaStream_t s);
// per column c < ncols: out[2c] = max|y_c - yp_c| (yp may be null -> max|y_c|), out[2c+1] = max|y_c|.
void launch_colstats(long long N, int ncols, const double* y, const double* yp, double* out, cudaStream_t s);
// copy `words` 8-byte words from device memory into mapped pinned host memory with one small kernel
void launch_store_words(const void* src, void* dst_mapped, size_t words, cudaStream_t s);
// copy vec4s 16-byte words (both pointers 16-byte aligned; either side may be mapped host memory)
void launch_copy_vec4(const void* src, void* dst, size_t vec4s, cudaStream_t s);
// out = s1*u + s3*u^3 - au   (Allen-Cahn source minus A u)
void launch_cubic_minus(long long N, double s1, double s3, const double* u, const double* au, double* out,
                        cudaStream_t s);
// y = y + c * x
void launch_axpy(long long N, double c, const double* x, double* y, cudaStream_t s);
// y = x - au  (generic source already evaluated)
void launch_sub(long long N, const double* x, const double* au, double* y, cudaStream_t s);

// kron_matvec with every factor tridiagonal (a 3-point stencil per mode, the reference's term order):
// y = sum_k (I (x) .. fl(scale A_k) .. (x) I) x, F[k] row-major n[k] x n[k]
// diag_scratch: 9 * max(n) doubles (the scaled diagonals, recomputed per call)
void launch_kron_tridiag(int d, const int* n, long long N, const double* const* F, double scale, const double* x,
                         double* y, double* diag_scratch, cudaStream_t s);

// ---- distributed squaring layout flips (dist.cpp) ----
// Trailing-index cuts of a slab: rank h's pencil owns t in [cb[h], cb[h+1]), cb[0] = 0, cb[G] = rest.
struct SlabCuts {
    int G = 1;
    long long ncols = 1;
    long long cb[17] = {0};
};
// pack: slab [col][row][t] (t < rest) -> blocks, block h at ncols*rows*cb[h] laid out
// [col][row][t - cb[h]] (contiguous per (h, col)); !pack: blocks -> slab.
void launch_slab_blocks(bool pack, int rows, long long rest, const SlabCuts& cuts, const double* src, double* dst,
                        cudaStream_t s);

}  // namespace pqb
