// FP64 DMMA mode-product GEMM template (see kernels.cu header comment); instantiated in
// gemm_nk.cu (B row-major, "n contiguous") and gemm_kk.cu (B stored k-contiguous).
//
// Structure: ST-stage cp.async pipeline (16-byte LDGSTS, zero-fill predicates) into padded
// shared-memory tiles; each warp owns a WM x WN register tile of m8n8k4 accumulators; one
// barrier per BK slice.  Per-thread global source pointers are computed once (no per-stage
// 64-bit address arithmetic) and the epilogue is compact (the extra-addend loop is not
// unrolled) so the whole kernel stays inside the instruction cache.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "kernels.hpp"

#ifndef PQ_GEMM_AFFINE
#define PQ_GEMM_AFFINE 1
#endif

namespace pqb {

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int VEC>
__device__ __forceinline__ void cp_async(unsigned dst, const double* src, bool ok) {
    const int bytes = ok ? 8 * VEC : 0;  // 0 -> zero-fill, nothing read
    if constexpr (VEC == 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Fine-gated DMMAs: only the fragment rows (ROWS) or columns whose bit is set in MASK.  Dispatched
// through a switch on the run-time mask (dmma_gated), so skipped DMMAs are not issued at all -- a
// plain `if` is if-converted into predicated DMMAs, which still occupy the tensor pipe.
template <int MI, int NI, bool ROWS, int MASK>
__device__ __forceinline__ void dmma_masked(double (&acc)[MI][NI][2], const double (&a)[MI], const double (&b)[NI]) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
            if ((MASK >> (ROWS ? i : j)) & 1) dmma_8x8x4(acc[i][j], a[i], b[j]);
}
template <int MI, int NI, bool ROWS, int M>
__device__ __forceinline__ void dmma_case(double (&acc)[MI][NI][2], const double (&a)[MI], const double (&b)[NI]) {
    if constexpr (M < (1 << (ROWS ? MI : NI))) dmma_masked<MI, NI, ROWS, M>(acc, a, b);
}
template <int MI, int NI, bool ROWS>
__device__ __forceinline__ void dmma_gated(unsigned mask, double (&acc)[MI][NI][2], const double (&a)[MI],
                                           const double (&b)[NI]) {
    static_assert((ROWS ? MI : NI) <= 4, "fine gating over at most 4 fragment groups");
    switch (mask) {
        case 1: dmma_case<MI, NI, ROWS, 1>(acc, a, b); break;
        case 2: dmma_case<MI, NI, ROWS, 2>(acc, a, b); break;
        case 3: dmma_case<MI, NI, ROWS, 3>(acc, a, b); break;
        case 4: dmma_case<MI, NI, ROWS, 4>(acc, a, b); break;
        case 5: dmma_case<MI, NI, ROWS, 5>(acc, a, b); break;
        case 6: dmma_case<MI, NI, ROWS, 6>(acc, a, b); break;
        case 7: dmma_case<MI, NI, ROWS, 7>(acc, a, b); break;
        case 8: dmma_case<MI, NI, ROWS, 8>(acc, a, b); break;
        case 9: dmma_case<MI, NI, ROWS, 9>(acc, a, b); break;
        case 10: dmma_case<MI, NI, ROWS, 10>(acc, a, b); break;
        case 11: dmma_case<MI, NI, ROWS, 11>(acc, a, b); break;
        case 12: dmma_case<MI, NI, ROWS, 12>(acc, a, b); break;
        case 13: dmma_case<MI, NI, ROWS, 13>(acc, a, b); break;
        case 14: dmma_case<MI, NI, ROWS, 14>(acc, a, b); break;
        case 15: dmma_case<MI, NI, ROWS, 15>(acc, a, b); break;
        default: break;
    }
}

// destination row of the remote-store epilogue (kernels.hpp RemoteMap)
__device__ __forceinline__ double* remote_row(const RemoteMap& rm, int z1, int m) {
    if (rm.mode == 1) {
        const int r = m / rm.n1, i1 = m - r * rm.n1;
        const long long t0 = (long long)i1 * rm.n2;
        int h = 0;
        while (h + 1 < rm.G && t0 >= rm.cb[h + 1]) ++h;
        const long long ch = rm.cb[h + 1] - rm.cb[h];
        return rm.base[h] + ((long long)z1 * rm.n0 + rm.s[rm.me] + r) * ch + (t0 - rm.cb[h]);
    }
    int h = 0;
    while (h + 1 < rm.G && m >= rm.s[h + 1]) ++h;
    return rm.base[h] + ((long long)z1 * (rm.s[h + 1] - rm.s[h]) + (m - rm.s[h])) * rm.rest + rm.cb[rm.me];
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM>
struct TileCfg {
    static constexpr int NWM = BM / WM, NWN = BN / WN, NT = NWM * NWN * 32;
    // Row strides padded to 4 (mod 16) doubles: the m8n8k4 fragment reads (row = lane/4,
    // k = lane%4) then hit 16 distinct 8-byte bank pairs per half-warp.
    static constexpr int SA = BK + 4;
    static constexpr int SB = BKM ? BK + 4 : BN + 4;
    static constexpr int ASZ = BM * SA;
    static constexpr int BSZ = BKM ? BN * SB : BK * SB;
    static constexpr int SMEM = ST * (ASZ + BSZ) * 8;
    static constexpr int MI = WM / 8, NI = WN / 8;
};

// One output tile (bx, by, bz) of a GemmArgs launch; the body of k_gemm and of the chained
// persistent kernel k_gemm_chain.  pdl: the programmatic-dependent-launch wait / trigger (plain
// stream launches only).
template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC>
__device__ __forceinline__ void gemm_tile(const GemmArgs& g, int bx, int by, int bz, double* smem, bool pdl) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    constexpr int NT = T::NT;
    double* sA = smem;
    double* sB = smem + ST * T::ASZ;

    const int z = bz + g.z_off;
    const int z1 = z / g.zdiv, z2 = z - z1 * g.zdiv;
    const double* __restrict__ A = g.A + z1 * g.sA1 + z2 * g.sA2;
    const double* __restrict__ B = g.B + z1 * g.sB1 + z2 * g.sB2;
    double* C = g.C + z1 * g.sC1 + z2 * g.sC2;
    const int m0 = bx * BM, n0 = by * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / T::NWN, wn = warp % T::NWN;
    const int gid = lane >> 2, tig = lane & 3;

    // programmatic dependent launch: everything above is index math; global data written by the
    // preceding kernel (operands, band tables, squaring counts) is read only after this wait
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (g.sq_count && g.sq_round >= g.sq_count[z]) {
        // expm squaring already finished for this matrix: carry it through unchanged.
        for (int e = tid; e < BM * BN; e += NT) {
            const int m = m0 + e / BN, n = n0 + e % BN;
            // __ldcg: in a chained launch A may have been written by other CTAs since this SM last
            // read it (L1 is not coherent across SMs; the operand tiles use cp.async.cg, L2 only)
            if (m < g.M && n < g.N) C[(long long)m * g.ldc + n] = __ldcg(&A[(long long)m * g.lda + n]);
        }
        return;
    }

    // ---- per-thread load descriptors (fixed across k slices) ----
    constexpr int KV = BK / VEC;
    constexpr int A_CH = BM * KV, A_IT = (A_CH + NT - 1) / NT;
    constexpr int B_CH = BKM ? BN * KV : BK * (BN / VEC), B_IT = (B_CH + NT - 1) / NT;
    const unsigned sA_base = static_cast<unsigned>(__cvta_generic_to_shared(sA));
    const unsigned sB_base = static_cast<unsigned>(__cvta_generic_to_shared(sB));
    // Affine descriptors: when every thread's chunks sit at a fixed row stride (NT a multiple of
    // the chunks per row), a thread keeps ONE source pointer per operand and walks it by that
    // stride -- ~14 registers instead of ~45 for per-chunk pointer / destination / bound arrays.
#if PQ_GEMM_AFFINE
    constexpr bool AFF = (A_CH % NT == 0) && (B_CH % NT == 0) && (NT % KV == 0) && (BKM || NT % (BN / VEC) == 0);
#else
    constexpr bool AFF = false;
#endif
    constexpr int NVB = BN / VEC;
    constexpr int RA = NT / KV;                  // A rows between a thread's chunks
    constexpr int RB = BKM ? NT / KV : NT / NVB;  // B rows (n for k-major, k otherwise) between chunks
    const double* a_p = nullptr;
    const double* b_p = nullptr;
    long long a_rowstep = 0, b_rowstep = 0;
    unsigned a_mask = 0, b_mask = 0, a_dst0 = 0, b_dst0 = 0;
    int a_kc = 0, b_r0 = 0;
    const double* a_src[AFF ? 1 : A_IT];
    unsigned a_dst[AFF ? 1 : A_IT];
    int a_k[AFF ? 1 : A_IT];
    bool a_ok[AFF ? 1 : A_IT];
    const double* b_src[AFF ? 1 : B_IT];
    unsigned b_dst[AFF ? 1 : B_IT];
    int b_k[AFF ? 1 : B_IT];
    bool b_ok[AFF ? 1 : B_IT];
    const long long b_kstep = BKM ? 1 : g.ldb;  // global stride of one k row of B
    if constexpr (AFF) {
        const int ra0 = tid / KV;
        a_kc = (tid % KV) * VEC;
        a_p = A + (long long)min(m0 + ra0, g.M - 1) * g.lda + a_kc;
        a_rowstep = (long long)RA * g.lda;
        a_dst0 = sA_base + 8u * (ra0 * T::SA + a_kc);
#pragma unroll
        for (int it = 0; it < A_IT; ++it)
            if (m0 + ra0 + it * RA < g.M) a_mask |= 1u << it;
        if constexpr (BKM) {
            const int rb0 = tid / KV, kc = (tid % KV) * VEC;  // rows = n, kc = k
            b_r0 = kc;
            b_p = B + (long long)min(n0 + rb0, g.N - 1) * g.ldb + kc;
            b_dst0 = sB_base + 8u * (rb0 * T::SB + kc);
#pragma unroll
            for (int it = 0; it < B_IT; ++it)
                if (n0 + rb0 + it * RB < g.N) b_mask |= 1u << it;
        } else {
            const int rb0 = tid / NVB, nc = (tid % NVB) * VEC;  // rows = k, nc = n
            b_r0 = rb0;
            b_p = B + (long long)rb0 * g.ldb + (n0 + nc < g.N ? n0 + nc : 0);
            b_dst0 = sB_base + 8u * (rb0 * T::SB + nc);
            b_mask = n0 + nc < g.N ? ~0u : 0u;
        }
        b_rowstep = (long long)RB * g.ldb;
    } else {
#pragma unroll
        for (int it = 0; it < A_IT; ++it) {
            const int c = tid + it * NT;
            const int r = c / KV, kc = (c % KV) * VEC;
            a_ok[it] = c < A_CH && m0 + r < g.M;
            a_src[it] = A + (long long)(a_ok[it] ? m0 + r : 0) * g.lda + kc;
            a_dst[it] = sA_base + 8u * (r * T::SA + kc);
            a_k[it] = kc;
        }
#pragma unroll
        for (int it = 0; it < B_IT; ++it) {
            const int c = tid + it * NT;
            if constexpr (BKM) {
                const int r = c / KV, kc = (c % KV) * VEC;  // r = n, kc = k
                b_ok[it] = c < B_CH && n0 + r < g.N;
                b_src[it] = B + (long long)(b_ok[it] ? n0 + r : 0) * g.ldb + kc;
                b_dst[it] = sB_base + 8u * (r * T::SB + kc);
                b_k[it] = kc;
            } else {
                const int r = c / NVB, nc = (c % NVB) * VEC;  // r = k, nc = n
                b_ok[it] = c < B_CH && n0 + nc < g.N;
                b_src[it] = B + (long long)r * g.ldb + (b_ok[it] ? n0 + nc : 0);
                b_dst[it] = sB_base + 8u * (r * T::SB + nc);
                b_k[it] = r;
            }
        }
    }

    // consecutive k slices are loaded in order: the source pointers advance by one slice per call
    // (no per-slice 64-bit multiply in the issue path)
    const long long b_step = static_cast<long long>(BK) * b_kstep;
    int k_next = 0;
    auto load_next = [&](int stage) {
        const int k0 = k_next;
        if constexpr (AFF) {
            const double* p = a_p;
            const bool kok = k0 + a_kc < g.K;
#pragma unroll
            for (int it = 0; it < A_IT; ++it) {
                const bool ok = kok && ((a_mask >> it) & 1u);
                cp_async<VEC>(a_dst0 + 8u * (it * RA * T::SA + stage * T::ASZ), ok ? p : A, ok);
                p += a_rowstep;
            }
            a_p += BK;
            p = b_p;
#pragma unroll
            for (int it = 0; it < B_IT; ++it) {
                const bool ok = ((b_mask >> (BKM ? it : 0)) & 1u) && (BKM ? k0 + b_r0 < g.K : k0 + b_r0 + it * RB < g.K);
                cp_async<VEC>(b_dst0 + 8u * (it * RB * T::SB + stage * T::BSZ), ok ? p : B, ok);
                p += b_rowstep;
            }
            b_p += b_step;
        } else {
#pragma unroll
            for (int it = 0; it < A_IT; ++it) {
                if (A_CH % NT != 0 && tid + it * NT >= A_CH) continue;
                const bool ok = a_ok[it] && k0 + a_k[it] < g.K;
                cp_async<VEC>(a_dst[it] + 8u * stage * T::ASZ, ok ? a_src[it] : A, ok);
                a_src[it] += BK;
            }
#pragma unroll
            for (int it = 0; it < B_IT; ++it) {
                if (B_CH % NT != 0 && tid + it * NT >= B_CH) continue;
                const bool ok = b_ok[it] && k0 + b_k[it] < g.K;
                cp_async<VEC>(b_dst[it] + 8u * stage * T::BSZ, ok ? b_src[it] : B, ok);
                b_src[it] += b_step;
            }
        }
        k_next += BK;
    };

    double acc[T::MI][T::NI][2];
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    int kt_lo = 0, KT = (g.K + BK - 1) / BK;
    int w_lo = 0, w_hi = KT;  // this warp's DMMA slices (absolute)
    // Fine gating: per 8-row group of the exponential covered by this warp's fragments (rows i for
    // an A exponential, columns j for a k-major B exponential), the k4 steps [lo, lo + len) its DMMAs
    // issue, packed lo | len << 16 (kernels.hpp launch_band_ranges).  Default: every step.
    constexpr int FG = BKM ? T::NI : T::MI;
    // every tile that can take a band table gates per group (the same executed k4 steps whichever
    // tile shape a mode product lands on: the fused and separate mode chains agree bitwise)
    constexpr bool GATE = (BK == 8 || BK == 16) && FG <= 4;
    unsigned fine[FG];
#pragma unroll
    for (int f = 0; f < FG; ++f) fine[f] = 0xffffu << 16;
    if constexpr (BK == 8 || BK == 16) {
        // negligible-block skip: the CTA streams the union of the 32-row exponential blocks its
        // tile covers, each warp multiplies only inside its own block's slices
        if (g.band) {
            int e, r0, te, wr, we;
            if (g.band_mode == 3) {  // exponential = B (k-major): its rows are the tile's columns
                e = z1;
                r0 = n0;
                te = BN;
                wr = n0 + wn * WN;
                we = WN;
            } else {
                e = g.band_mode == 1 ? m0 / g.band_rows : z1;
                r0 = g.band_mode == 1 ? m0 % g.band_rows : m0;
                te = BM;
                wr = r0 + wm * WM;
                we = WM;
            }
            const int2* br = g.band + (long long)e * g.band_stride;
            const int nb = (g.band_rows + 31) >> 5;
            int lo = 1 << 30, hi = 0;
            for (int b = r0 >> 5; b < min((r0 + te + 31) >> 5, nb); ++b) {
                const int2 v = br[b];
                if (v.y > v.x) {
                    lo = min(lo, v.x);
                    hi = max(hi, v.y);
                }
            }
            // the table counts 8-column slices; a BK-wide stage covers BK/8 of them
            constexpr int SH = BK == 16 ? 1 : 0;
            kt_lo = hi > lo ? (lo >> SH) : 0;
            KT = min(KT, hi > lo ? ((hi + (1 << SH) - 1) >> SH) : 0);
            if (we <= 32) {  // the warp lies in one 32-row block: multiply only inside its range
                const int wb = wr >> 5;
                const int2 mine = wb < nb ? br[wb] : make_int2(0, 0);
                w_lo = mine.x >> SH;
                w_hi = (mine.y + (1 << SH) - 1) >> SH;
            } else {
                w_lo = kt_lo;
                w_hi = KT;
            }
#pragma unroll
            for (int f = 0; f < FG; ++f) {
                if (!GATE) break;
                const int grp = (wr >> 3) + f;
                const int2 v = grp < 4 * nb ? br[nb + grp] : make_int2(0, 0);
                fine[f] = v.y > v.x ? static_cast<unsigned>(v.x) | (static_cast<unsigned>(v.y - v.x) << 16) : 0u;
            }
        }
    }
    const int NKT = KT > kt_lo ? KT - kt_lo : 0;
    if (g.flop_counter && lane == 0) {
        // executed DMMA work: per fragment row (column) group, its k4 steps inside the warp's slices
        const int lo = max(kt_lo, w_lo), hi = min(KT, w_hi);
        const int q0 = lo * (BK / 4), q1 = hi > lo ? (min(hi * BK, g.K) + 3) / 4 : q0;
        unsigned long long f_exec = 0;
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int j = 0; j < T::NI; ++j) {
                const unsigned fr = fine[BKM ? j : i];
                const int flo = static_cast<int>(fr & 0xffffu), fhi = flo + static_cast<int>(fr >> 16);
                const int steps = max(0, min(q1, fhi) - max(q0, flo));
                const long long rows = max(0, min(8, g.M - (m0 + wm * WM + i * 8)));
                const long long cols = max(0, min(8, g.N - (n0 + wn * WN + j * 8)));
                f_exec += static_cast<unsigned long long>(2 * rows * cols * 4 * steps);
            }
        atomicAdd(g.flop_counter, f_exec);
    }
    k_next = kt_lo * BK;
    if constexpr (AFF) {
        a_p += k_next;
        b_p += static_cast<long long>(k_next) * b_kstep;
    } else {
#pragma unroll
        for (int it = 0; it < A_IT; ++it) a_src[it] += k_next;
#pragma unroll
        for (int it = 0; it < B_IT; ++it) b_src[it] += static_cast<long long>(k_next) * b_kstep;
    }
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < NKT) load_next(s);
        cp_commit();
    }
    const double* tA0 = sA + (wm * WM + gid) * T::SA + tig;
    const double* tB0 = BKM ? sB + (wn * WN + gid) * T::SB + tig : sB + tig * T::SB + wn * WN + gid;
#pragma unroll 1
    for (int kt = 0; kt < NKT; ++kt) {
        cp_wait<ST - 2>();
        __syncthreads();
        {
            const int nk = kt + ST - 1;
            if (nk < NKT) load_next(nk % ST);
            cp_commit();
        }
        const int st = kt % ST;
        const int kabs = kt_lo + kt;
        if (kabs < w_lo || kabs >= w_hi) continue;  // warp-uniform: this warp's rows need no DMMA here
        const double* tA = tA0 + st * T::ASZ;
        const double* tB = tB0 + st * T::BSZ;
        // a slice every fragment group covers entirely runs the plain unrolled DMMA block; others
        // step through their k4 steps with the mask dispatch (kept out of the unrolled path, so the
        // kernel's hot loop stays small in the instruction cache)
        bool full = true;
        if constexpr (GATE) {
            const unsigned q0 = static_cast<unsigned>((kabs * BK) >> 2);
#pragma unroll
            for (int f = 0; f < FG; ++f)
                full = full && (fine[f] & 0xffffu) <= q0 && q0 + BK / 4 <= (fine[f] & 0xffffu) + (fine[f] >> 16);
        }
        if (full) {
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[T::MI], b[T::NI];
#pragma unroll
                for (int i = 0; i < T::MI; ++i) a[i] = tA[i * 8 * T::SA + kk];
#pragma unroll
                for (int j = 0; j < T::NI; ++j) b[j] = BKM ? tB[j * 8 * T::SB + kk] : tB[kk * T::SB + j * 8];
#pragma unroll
                for (int i = 0; i < T::MI; ++i)
#pragma unroll
                    for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
            }
        } else if constexpr (GATE) {
#pragma unroll 1
            for (int kk = 0; kk < BK; kk += 4) {
                const unsigned kq = static_cast<unsigned>((kabs * BK + kk) >> 2);
                unsigned mask = 0;
#pragma unroll
                for (int f = 0; f < FG; ++f) mask |= (kq - (fine[f] & 0xffffu) < (fine[f] >> 16) ? 1u : 0u) << f;
                if (mask == 0u) continue;
                double a[T::MI], b[T::NI];
#pragma unroll
                for (int i = 0; i < T::MI; ++i) a[i] = tA[i * 8 * T::SA + kk];
#pragma unroll
                for (int j = 0; j < T::NI; ++j) b[j] = BKM ? tB[j * 8 * T::SB + kk] : tB[kk * T::SB + j * 8];
                if (mask == (1u << FG) - 1u) {
#pragma unroll
                    for (int i = 0; i < T::MI; ++i)
#pragma unroll
                        for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
                } else {
                    dmma_gated<T::MI, T::NI, !BKM>(mask, acc, a, b);
                }
            }
        }
    }
    cp_wait<0>();
    // this CTA no longer needs the SM for DMMA work: let the next kernel in the stream launch its
    // CTAs (they stop at griddepcontrol.wait until this grid has completed)
    if (pdl) asm volatile("griddepcontrol.launch_dependents;");

    // ---- epilogue (registers -> global) ----
    const double alpha = g.alpha_z ? g.alpha_z[z1] : g.alpha;
    const int nt = g.nterms ? g.nterms[z1] : 0;
    const int mb = m0 + wm * WM + gid, nbase = n0 + wn * WN + 2 * tig;
    const double* crow = g.coef ? g.coef + (long long)z1 * g.cld : nullptr;
    const double* ext = g.ext ? g.ext + (long long)(z1 / g.ext_group) * g.ext_group * g.ext_s + z2 * g.sC2 : nullptr;
    // each thread owns 2 consecutive columns -> 16-byte accesses when everything is aligned
    const bool v2 = (g.ldc % 2 == 0) && (g.sC1 % 2 == 0) && (g.sC2 % 2 == 0) &&
                    ((reinterpret_cast<uintptr_t>(g.C) & 15) == 0) &&
                    (!ext || (g.ext_s % 2 == 0 && (reinterpret_cast<uintptr_t>(ext) & 15) == 0));
    // out = alpha*acc (+ C_old) + sum_t coef_t * ext_t  -- the reference's update order
    // (phiaction.hpp:260-268), applied term by term so each term's loads are independent.
    // integer test of the bit pattern: a DSETP here waits behind the other warps' DMMAs in the
    // shared FP64/tensor pipe (ncu source page: ~3% of the band kernel's stall samples)
    if (__double_as_longlong(alpha) != 0x3FF0000000000000LL) {
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int j = 0; j < T::NI; ++j) {
                acc[i][j][0] = __dmul_rn(alpha, acc[i][j][0]);
                acc[i][j][1] = __dmul_rn(alpha, acc[i][j][1]);
            }
    }
    auto add_term = [&](const double* src, double coef, bool plain) {
#pragma unroll
        for (int i = 0; i < T::MI; ++i) {
            const int m = mb + i * 8;
            if (m >= g.M) continue;
            const double* row = src + (long long)m * g.ldc;
#pragma unroll
            for (int j = 0; j < T::NI; ++j) {
                const int n = nbase + j * 8;
                double x0 = 0.0, x1 = 0.0;
                if (v2 && n + 1 < g.N) {
                    const double2 v = *reinterpret_cast<const double2*>(row + n);
                    x0 = v.x;
                    x1 = v.y;
                } else {
                    if (n < g.N) x0 = row[n];
                    if (n + 1 < g.N) x1 = row[n + 1];
                }
                if (plain) {  // accumulate: C_old + v
                    acc[i][j][0] = __dadd_rn(x0, acc[i][j][0]);
                    acc[i][j][1] = __dadd_rn(x1, acc[i][j][1]);
                } else {
                    acc[i][j][0] = __dadd_rn(acc[i][j][0], __dmul_rn(coef, x0));
                    acc[i][j][1] = __dadd_rn(acc[i][j][1], __dmul_rn(coef, x1));
                }
            }
        }
    };
    if (g.accumulate) add_term(C, 1.0, true);
#pragma unroll 1
    for (int t = 0; t < nt; ++t) add_term(ext + (long long)t * g.ext_s, crow[t], false);
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
        const int m = mb + i * 8;
        if (m >= g.M) continue;
        double* row = g.remote ? remote_row(*g.remote, z1, m) : C + (long long)m * g.ldc;
#pragma unroll
        for (int j = 0; j < T::NI; ++j) {
            const int n = nbase + j * 8;
            if (v2 && n + 1 < g.N) {
                *reinterpret_cast<double2*>(row + n) = make_double2(acc[i][j][0], acc[i][j][1]);
            } else {
                if (n < g.N) row[n] = acc[i][j][0];
                if (n + 1 < g.N) row[n + 1] = acc[i][j][1];
            }
        }
    }
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC, int MINB = 1>
__global__ void __launch_bounds__(TileCfg<BM, BN, BK, WM, WN, ST, BKM>::NT, MINB) k_gemm(const GemmArgs g) {
    extern __shared__ __align__(16) double smem[];
    gemm_tile<BM, BN, BK, WM, WN, ST, BKM, VEC>(g, blockIdx.x, blockIdx.y, blockIdx.z, smem, true);
}

// A chain of dependent batched GEMM levels in ONE cooperative launch (the Taylor powers
// P^(h+j) = P^h P^j of the shared-power exponentials and the expm squaring rounds): every CTA
// walks the tiles of a level (grid-stride), then the grid synchronises before the next level
// reads its results.  Replaces 5-7 short dependent launches per chain, each a fraction of a wave.
constexpr int kMaxChain = 12;
struct GemmChain {
    int levels = 0;
    GemmArgs g[kMaxChain];
};

__device__ __forceinline__ void chain_grid_sync(unsigned* bar, unsigned nblocks, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned target = (gen + 1) * nblocks;
        atomicAdd(bar, 1u);
        while (true) {
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v >= target) break;
            __nanosleep(32);
        }
    }
    ++gen;
    __syncthreads();
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC, int MINB>
__global__ void __launch_bounds__(TileCfg<BM, BN, BK, WM, WN, ST, BKM>::NT, MINB)
    k_gemm_chain(const __grid_constant__ GemmChain ch, unsigned* bar) {
    extern __shared__ __align__(16) double smem[];
    unsigned gen = 0;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int lv = 0; lv < ch.levels; ++lv) {
        const GemmArgs& g = ch.g[lv];
        const int gx = (g.M + BM - 1) / BM, gy = (g.N + BN - 1) / BN;
        const int tiles = gx * gy * g.Z;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            gemm_tile<BM, BN, BK, WM, WN, ST, BKM, VEC>(g, t % gx, (t / gx) % gy, t / (gx * gy), smem, false);
            __syncthreads();  // the next tile's prologue overwrites the stages this one read
        }
        if (lv + 1 < ch.levels) chain_grid_sync(bar, gridDim.x, gen);
    }
}

// Persistent variant for large launches: CTA c processes tiles c, c + grid, c + 2 grid, ...
// (tile = (z, n-tile, m-tile), m fastest) as ONE flattened (tile, k-slice) loop, so the cp.async
// pipeline runs across tile boundaries: the next tile's first slices are in flight while the
// current tile's epilogue stores.  Plain stores only (no fused epilogue terms, no squaring skip).
template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC>
__global__ void __launch_bounds__(TileCfg<BM, BN, BK, WM, WN, ST, BKM>::NT, 1)
    k_gemm_persist(const GemmArgs g, int tiles_m, int tiles_n, int total_tiles) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    constexpr int NT = T::NT;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + ST * T::ASZ;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / T::NWN, wn = warp % T::NWN;
    const int gid = lane >> 2, tig = lane & 3;
    const int KT = (g.K + BK - 1) / BK;
    const int my_tiles = (total_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int total_iters = my_tiles * KT;
    const int per_z = tiles_m * tiles_n;

    struct TileBase {
        const double* A;
        const double* B;
        double* C;
        int m0, n0;
    };
    auto tile_base = [&](int local) {
        const int t = (int)blockIdx.x + local * (int)gridDim.x;
        const int z = t / per_z, r = t - z * per_z;
        const int nt = r / tiles_m, mt = r - nt * tiles_m;
        const int z1 = z / g.zdiv, z2 = z - z1 * g.zdiv;
        return TileBase{g.A + z1 * g.sA1 + z2 * g.sA2, g.B + z1 * g.sB1 + z2 * g.sB2, g.C + z1 * g.sC1 + z2 * g.sC2,
                        mt * BM, nt * BN};
    };

    constexpr int KV = BK / VEC;
    constexpr int A_CH = BM * KV, A_IT = (A_CH + NT - 1) / NT;
    constexpr int NV = BN / VEC;
    constexpr int B_CH = BKM ? BN * KV : BK * NV, B_IT = (B_CH + NT - 1) / NT;
    const unsigned sA_base = static_cast<unsigned>(__cvta_generic_to_shared(sA));
    const unsigned sB_base = static_cast<unsigned>(__cvta_generic_to_shared(sB));

    auto load_iter = [&](int it) {
        const int local = it / KT, kt = it - local * KT, stage = it % ST;
        const TileBase tb = tile_base(local);
        const int k0 = kt * BK;
#pragma unroll
        for (int i = 0; i < A_IT; ++i) {
            const int c = tid + i * NT;
            if (A_CH % NT != 0 && c >= A_CH) continue;
            const int r = c / KV, kc = (c % KV) * VEC;
            const bool ok = tb.m0 + r < g.M && k0 + kc < g.K;
            cp_async<VEC>(sA_base + 8u * (stage * T::ASZ + r * T::SA + kc),
                          ok ? tb.A + (long long)(tb.m0 + r) * g.lda + k0 + kc : g.A, ok);
        }
#pragma unroll
        for (int i = 0; i < B_IT; ++i) {
            const int c = tid + i * NT;
            if (B_CH % NT != 0 && c >= B_CH) continue;
            if constexpr (BKM) {
                const int r = c / KV, kc = (c % KV) * VEC;
                const bool ok = tb.n0 + r < g.N && k0 + kc < g.K;
                cp_async<VEC>(sB_base + 8u * (stage * T::BSZ + r * T::SB + kc),
                              ok ? tb.B + (long long)(tb.n0 + r) * g.ldb + k0 + kc : g.B, ok);
            } else {
                const int r = c / NV, nc = (c % NV) * VEC;
                const bool ok = k0 + r < g.K && tb.n0 + nc < g.N;
                cp_async<VEC>(sB_base + 8u * (stage * T::BSZ + r * T::SB + nc),
                              ok ? tb.B + (long long)(k0 + r) * g.ldb + tb.n0 + nc : g.B, ok);
            }
        }
    };

    double acc[T::MI][T::NI][2];
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < total_iters) load_iter(s);
        cp_commit();
    }
    const double* tA0 = sA + (wm * WM + gid) * T::SA + tig;
    const double* tB0 = BKM ? sB + (wn * WN + gid) * T::SB + tig : sB + tig * T::SB + wn * WN + gid;
    const bool v2 = (g.ldc % 2 == 0) && (g.sC1 % 2 == 0) && (g.sC2 % 2 == 0) &&
                    ((reinterpret_cast<uintptr_t>(g.C) & 15) == 0);
#pragma unroll 1
    for (int it = 0; it < total_iters; ++it) {
        cp_wait<ST - 2>();
        __syncthreads();
        if (it + ST - 1 < total_iters) load_iter(it + ST - 1);
        cp_commit();
        const int st = it % ST;
        const double* tA = tA0 + st * T::ASZ;
        const double* tB = tB0 + st * T::BSZ;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[T::MI], b[T::NI];
#pragma unroll
            for (int i = 0; i < T::MI; ++i) a[i] = tA[i * 8 * T::SA + kk];
#pragma unroll
            for (int j = 0; j < T::NI; ++j) b[j] = BKM ? tB[j * 8 * T::SB + kk] : tB[kk * T::SB + j * 8];
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
        }
        const int local = it / KT;
        if (it - local * KT == KT - 1) {  // tile done: store while the next tile's slices load
            const TileBase tb = tile_base(local);
            const int mb = tb.m0 + wm * WM + gid, nbase = tb.n0 + wn * WN + 2 * tig;
#pragma unroll
            for (int i = 0; i < T::MI; ++i) {
                const int m = mb + i * 8;
                double* row = tb.C + (long long)m * g.ldc;
#pragma unroll
                for (int j = 0; j < T::NI; ++j) {
                    const int n = nbase + j * 8;
                    const double v0 = g.alpha == 1.0 ? acc[i][j][0] : __dmul_rn(g.alpha, acc[i][j][0]);
                    const double v1 = g.alpha == 1.0 ? acc[i][j][1] : __dmul_rn(g.alpha, acc[i][j][1]);
                    if (m < g.M) {
                        if (v2 && n + 1 < g.N) {
                            *reinterpret_cast<double2*>(row + n) = make_double2(v0, v1);
                        } else {
                            if (n < g.N) row[n] = v0;
                            if (n + 1 < g.N) row[n + 1] = v1;
                        }
                    }
                    acc[i][j][0] = acc[i][j][1] = 0.0;
                }
            }
        }
    }
    cp_wait<0>();
}

// Programmatic dependent launch for the mode products (PQ_PDL=0 disables): the next GEMM's CTAs
// are scheduled while this one drains its last wave.
static bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PQ_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC>
static int launch_persist(const GemmArgs& g, int max_ctas, cudaStream_t s) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    auto kern = k_gemm_persist<BM, BN, BK, WM, WN, ST, BKM, VEC>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
        attr_done = true;
    }
    const long long tm = (g.M + BM - 1) / BM, tn = (g.N + BN - 1) / BN;
    const long long total = tm * tn * g.Z;
    if (total > 2147483647LL) throw std::invalid_argument("mode product: too many tiles");
    const int grid = (int)(total < max_ctas ? total : max_ctas);
    kern<<<grid, T::NT, T::SMEM, s>>>(g, (int)tm, (int)tn, (int)total);
    return 1;
}


template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC, int MINB = 1>
static int launch_cfg(const GemmArgs& g, cudaStream_t s) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    auto kern = k_gemm<BM, BN, BK, WM, WN, ST, BKM, VEC, MINB>;
    static bool attr_done = false;  // per instantiation
    if (!attr_done) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
        attr_done = true;
    }
    const long long gx = (g.M + BM - 1) / BM, gy = (g.N + BN - 1) / BN;
    if (gx > 2147483647LL || gy > 65535) throw std::invalid_argument("mode product: grid too large");
    int launches = 0;
    GemmArgs a = g;
    for (int z0 = 0; z0 < g.Z; z0 += 65535) {
        a.z_off = z0;
        const int zc = g.Z - z0 < 65535 ? g.Z - z0 : 65535;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)gx, (unsigned)gy, (unsigned)zc);
        cfg.blockDim = dim3(T::NT);
        cfg.dynamicSmemBytes = T::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, a);
        ++launches;
    }
    return launches;
}

template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB>
static int launch_chain_cfg(const GemmChain& ch, unsigned* bar, cudaStream_t s) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, false>;
    auto kern = k_gemm_chain<BM, BN, BK, WM, WN, ST, false, 2, MINB>;
    static int per_sm = -1, sms = 0;
    if (per_sm < 0) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T::NT, T::SMEM) != cudaSuccess) per_sm = 0;
    }
    if (per_sm <= 0 || sms <= 0) return 0;
    long long tiles = 0;
    for (int lv = 0; lv < ch.levels; ++lv) {
        const GemmArgs& g = ch.g[lv];
        tiles = std::max(tiles, (long long)((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN) * g.Z);
    }
    const int grid = (int)std::min<long long>((long long)per_sm * sms, tiles);
    if (grid <= 0) return 0;
    cudaMemsetAsync(bar, 0, sizeof(unsigned), s);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(T::NT);
    cfg.dynamicSmemBytes = T::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the level barrier cannot deadlock
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, ch, bar) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return 1;
}

// Tile shapes: 0 = 128x128 (8 warps of 64x32), 1 = 128x64, 2 = 64x128, 3 = 64x64, 4 = 32x32.
#ifndef PQ_BK_BIG
#define PQ_BK_BIG 32
#endif
template <bool BKM>
int launch_gemm_family(const GemmArgs& g, bool vec2, int shape, cudaStream_t s) {
    constexpr int BKB = PQ_BK_BIG;
    constexpr int STB = BKB == 32 ? 3 : 4;
    if (shape == 5) {  // persistent 64x64x16, 3 CTAs per SM
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (sms <= 0) sms = 148;
        }
        const int max_ctas = sms * 3;
        return vec2 ? launch_persist<64, 64, 16, 32, 32, 3, BKM, 2>(g, max_ctas, s)
                    : launch_persist<64, 64, 16, 32, 32, 3, BKM, 1>(g, max_ctas, s);
    }
    switch (shape) {
        case 0: return vec2 ? launch_cfg<128, 128, BKB, 64, 32, STB, BKM, 2>(g, s) : launch_cfg<128, 128, BKB, 64, 32, STB, BKM, 1>(g, s);
        case 1: return vec2 ? launch_cfg<128, 64, BKB, 64, 32, STB, BKM, 2>(g, s) : launch_cfg<128, 64, BKB, 64, 32, STB, BKM, 1>(g, s);
        case 2: return vec2 ? launch_cfg<64, 128, BKB, 32, 64, STB, BKM, 2>(g, s) : launch_cfg<64, 128, BKB, 32, 64, STB, BKM, 1>(g, s);
        case 9:  // exponential = B (k-major), default: 128x32 tiles, four 32x32 warps (4-DMMA gated groups)
            return launch_cfg<128, 32, 16, 32, 32, 2, BKM, 2, 4>(g, s);
        case 6:  // negligible-block skip, exponential = A: 32-row tiles stream only their block's slices
            // (32x128 with four 32x32 warps: +3% over 32x64 on the node-sweep band shapes, +4.5% dense;
            // 16-wide k slices in 2 stages: +2.5-4% over 8-wide in 4 once the load issue path lost its
            // per-slice 64-bit multiplies, tools/gemm_tune.cu, profiles/r01_gemm_tune_bk16.txt)
            return launch_cfg<32, 128, 16, 32, 32, 2, BKM, 2, 4>(g, s);
        case 7:  // PQ_KK_TALL=0: exponential = B (k-major) on 64x32 tiles (BK 16: +3-6% over BK 8)
            return launch_cfg<64, 32, 16, 32, 16, 2, BKM, 2, 6>(g, s);
        case 8:  // exponential = A on small grids (PQ_SMALL_GRID_TILE=1 only, kernels.cu): 64x32 tiles at
                 // 7 CTAs/SM fill the last wave (2048 CTAs in 1.98 waves instead of 1024 in 1.73)
            return launch_cfg<64, 32, 16, 32, 16, 2, BKM, 2, 7>(g, s);
        case 3:
            // 16-byte path: BK = 8, 4 stages and <= 128 registers give 4 CTAs (16 warps) per SM,
            // which keeps the DMMA pipe fed while other warps sit in barriers / epilogues
            // (+3-4% over 64x64x16 at 3 CTAs/SM on every mode shape, r01_gemm_tune_minb.txt)
            if (vec2) return launch_cfg<64, 64, 8, 32, 32, 4, BKM, 2, 4>(g, s);
            // 8-byte path: 4 stages still fit 3 CTAs/SM for row-major B; the k-major B tile is
            // larger and would drop to 2 CTAs/SM, so it keeps 3 stages
            if constexpr (BKM)
                return vec2 ? launch_cfg<64, 64, 16, 32, 32, 3, BKM, 2>(g, s) : launch_cfg<64, 64, 16, 32, 32, 3, BKM, 1>(g, s);
            else
                return vec2 ? launch_cfg<64, 64, 16, 32, 32, 4, BKM, 2>(g, s) : launch_cfg<64, 64, 16, 32, 32, 4, BKM, 1>(g, s);
        default: return vec2 ? launch_cfg<32, 32, 16, 16, 16, 3, BKM, 2>(g, s) : launch_cfg<32, 32, 16, 16, 16, 3, BKM, 1>(g, s);
    }
}

}  // namespace pqb
