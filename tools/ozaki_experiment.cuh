// FP64 mode products on the INT8 tensor cores (tcgen05.mma kind::i8, accumulators in TMEM):
// an error-free digit split of both operands (Ozaki scheme, 7 signed 8-bit digits per value).
//
// For one mode product y[f][i] = sum_j E[i][j] x[f][j] (f runs over the mode-k fibres of x,
// i, j < n = 128) every row of E and every fibre of x is scaled by its own power of two and
// rounded to an integer V with |V| <= 2^54, written as 7 signed base-256 digits:
//     V = sum_{s=1..7} d_s 256^(7-s),  d_s in [-128, 127]      (the bytes of V + OFF, excess 128)
// The digit products d^E_s d^x_t are exact in int8 x int8 -> int32; for each digit order
// c = s + t <= 8 the 128-long dot products accumulate exactly in one int32 TMEM accumulator
// (|acc_c| <= 7 * 128 * 2^14 < 2^24), and the epilogue rebuilds
//     y = 2^(e_i + e_f - 108) sum_{c=2..8} acc_c 256^(14-c)
// in FP64.  The dropped orders c >= 9 and the rounding of the operands to 55 bits bound the error
// by about 2^-50 max|E_i.| max|x_f.| per term -- the order of the FP64 GEMM's own rounding.
//
// Kernel (one persistent CTA per SM, 13 warps, 226 KB shared memory, 512 TMEM columns):
//   warps 0-3  : epilogue.  Warp w reads TMEM lanes 32w.. (= rows of E), fibres in two halves;
//                the second half's pass frees each order accumulator for the next tile's MMAs as
//                soon as it is read; the orders are summed in FP64 and y is stored.
//   warps 4-11 : producers.  Copy E's digit planes into shared memory (A operand, 7 x 16 KB, once
//                per exponential), then per tile load 64 fibres (fp64), find each fibre's exponent
//                (shuffle max over the 8 lanes that share it), split into digits and store them as
//                the B operand (K-major core matrices) in a 2-deep ring.
//   warp 12    : one lane issues the 28 x 4 MMAs (M 128, N 64, K 32; both operands in smem) per
//                tile, order by order, committing each order to its accumulator barrier.
// tools/umma_rate.cu: an M128 kind::i8 MMA costs 48 clocks at N <= 64 and 64 at N = 128 (the
// 4.76 POPS peak), so N = 64 keeps 67% of the tensor rate while 7 accumulators fit in TMEM.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace pqb {
namespace oz {

constexpr int kS = 7;                               // digits per operand
constexpr int kN = 128;                             // factor size (MMA M, and K)
constexpr int kNT = 64;                             // fibres per tile (MMA N)
constexpr int kStages = 2;                          // B ring depth
constexpr int kRing = kStages + 2;                  // fibre-scale ring
constexpr int kPlaneA = kN * kN;                    // 16 KB digit plane of E
constexpr int kPlaneB = kNT * kN;                   // 8 KB digit plane of a tile
constexpr int kABytes = kS * kPlaneA;               // 112 KB
constexpr int kStageBytes = kS * kPlaneB;           // 56 KB
constexpr int kEpiWarps = 4, kProdWarps = 8;  // + 1 MMA warp = 13 warps (<= 128 registers)
constexpr int kThreads = (kEpiWarps + kProdWarps + 1) * 32;
constexpr int kProducers = kProdWarps * 32;
constexpr unsigned long long kOff = 0x80808080808080ull;  // 128 * sum_{b<7} 256^b
struct Bars {
    uint64_t full[kStages], empty[kStages], d_full[kS], d_empty[kS], a_free;
    uint32_t tmem_base;
    double sfx[kRing][kNT];
};
constexpr int kSmemBytes = kABytes + kStages * kStageBytes + static_cast<int>(sizeof(Bars));

struct ModeArgs {
    const int8_t* Ed = nullptr;   // [nE][kS] planes of E's digits, each in the smem core-matrix image
    const int* Ee = nullptr;      // [nE][kN] row exponents
    int e_shared = 0;             // every batch uses digit set 0 (else set z / zdiv)
    const double* x = nullptr;
    double* y = nullptr;
    int Z = 1, zdiv = 1;
    long long sx1 = 0, sx2 = 0, sy1 = 0, sy2 = 0;  // batch z = z1*zdiv + z2 strides
    long long F = 0;              // fibres per batch
    long long fstride = 0, jstride = 0;  // fibre and along-fibre strides (x and y alike)
    int dbg = 0;                  // tools/oz_probe.cu: 1 one MMA per order, 2 no epilogue math, 4 no x loads
    unsigned long long* prof = nullptr;  // tools/oz_probe.cu: per CTA [8] clock64 totals (wait / work per role)
};

// byte offset of element (row r, k) in a K-major core-matrix image with 128-long rows
__host__ __device__ constexpr int cm_off(int r, int k) { return (r >> 3) * 1024 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
                 : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T, int8 x int8 -> int32
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 B contiguous); K-adjacent core
// matrices 128 B apart (LBO), 8-row groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t bdesc(uint32_t addr) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>(128 >> 4) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46);
}
// kind::i8: D s32 (bits 4-5 = 2), A s8 (bits 7-9 = 1), B s8 (bits 10-12 = 1), both K-major,
// N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kNT >> 3) << 17) |
                            (static_cast<uint32_t>(kN >> 4) << 24);
__device__ __forceinline__ void tc_mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc_, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(adesc), "l"(bdesc_), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}

// exponent e with max|v| < 2^e (0 for an all-zero set)
__device__ __forceinline__ int oz_exponent(double amax) {
    if (!(amax > 0.0)) return 0;
    int e;
    frexp(amax, &e);
    return e;
}
// exact int32 -> double without the conversion pipe: 2^52 + 2^31 + a is exact in the mantissa
__device__ __forceinline__ double i2d_exact(int a) {
    return __hiloint2double(0x43300000, static_cast<int>(static_cast<unsigned>(a) ^ 0x80000000u)) - 4503601774854144.0;
}
// excess-128 digit word of v scaled by 2^sh: byte b (b < 7) = d_{7-b} + 128
__device__ __forceinline__ unsigned long long oz_word(double v, double sc) {
    const long long V = __double2ll_rn(v * sc);
    return static_cast<unsigned long long>(V) + kOff;
}

// ---------------------------------------------------------------- E digit planes ----
// One warp per row i of exponential e: plane s of Ed[e] holds digit s of E[e][i][j] at
// cm_off(i, j) (row scaled by 2^(54 - Ee[e][i])), i.e. the exact shared-memory image of the
// MMA's A operand.
__global__ void __launch_bounds__(256) k_oz_split_rows(const double* __restrict__ E, long long sE, int nE,
                                                       int8_t* __restrict__ Ed, int* __restrict__ Ee) {
#if defined(__CUDA_ARCH__)
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= nE * kN) return;
    const int e = warp / kN, i = warp % kN;
    const double* row = E + e * sE + static_cast<long long>(i) * kN;
    double v[4];
    double amax = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        v[q] = row[lane * 4 + q];
        amax = fmax(amax, fabs(v[q]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const int ex = oz_exponent(amax);
    const double sc = ldexp(1.0, 54 - ex);
    unsigned long long w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = oz_word(v[q], sc);
#pragma unroll
    for (int s = 1; s <= kS; ++s) {
        const int b = 7 - s;
        uint32_t packed = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) packed |= static_cast<uint32_t>(((w[q] >> (8 * b)) & 0xFF) ^ 0x80) << (8 * q);
        *reinterpret_cast<uint32_t*>(Ed + (static_cast<long long>(e) * kS + (s - 1)) * kPlaneA + cm_off(i, lane * 4)) = packed;
    }
    if (lane == 0) Ee[e * kN + i] = ex;
#endif
}

// ---------------------------------------------------------------- the mode product ----
__global__ void __launch_bounds__(kThreads, 1) k_oz_mode(ModeArgs a) {
#if defined(__CUDA_ARCH__)
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* ring = smem + kABytes;
    Bars& B = *reinterpret_cast<Bars*>(smem + kABytes + kStages * kStageBytes);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long ntile = (a.F + kNT - 1) / kNT;
    const long long T = static_cast<long long>(a.Z) * ntile;
    const long long t0 = T * blockIdx.x / gridDim.x, t1 = T * (blockIdx.x + 1) / gridDim.x;
    auto e_index = [&](long long t) -> long long { return a.e_shared ? 0 : (t / ntile) / a.zdiv; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&B.full[s], kProducers);
            mbar_init(&B.empty[s], 1);
        }
        for (int c = 0; c < kS; ++c) {
            mbar_init(&B.d_full[c], 1);
            mbar_init(&B.d_empty[c], kEpiWarps * 32);
        }
        mbar_init(&B.a_free, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&B.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tD = B.tmem_base;

    if (warp < kEpiWarps) {
        // ------------------------------------------------------------ epilogue ----
        // two passes of 32 fibres; the second pass frees each order's accumulator as it reads it
        const int i = warp * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
        unsigned long long ew = 0, es = 0;
        const unsigned long long e_start = clock64();
        for (long long t = t0; t < t1; ++t) {
            const long long it = t - t0;
            const long long z = t / ntile;
            const long long z1 = z / a.zdiv, z2 = z % a.zdiv;
            const double si = ldexp(1.0, a.Ee[e_index(t) * kN + i] - 12);
            double* yb = a.y + z1 * a.sy1 + z2 * a.sy2 + static_cast<long long>(i) * a.jstride;
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                const long long f0 = (t % ntile) * kNT + half * 32;
                double part[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) part[q] = 0.0;
                double w = 1.0;
#pragma unroll 1
                for (int c = 0; c < kS; ++c) {
                    if (half == 0) {
                        const unsigned long long w0 = clock64();
                        mbar_wait(&B.d_full[c], static_cast<uint32_t>(it & 1));
                        ew += clock64() - w0;
                        tc_fence_after();
                    }
                    int acc[32];
                    tmem_ld32(tD + lane_off + c * kNT + half * 32, acc);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (half == 1) {
                        tc_fence_before();
                        mbar_arrive(&B.d_empty[c]);
                    }
                    if (!(a.dbg & 2)) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) part[q] = fma(i2d_exact(acc[q]), w, part[q]);
                    }
                    w *= 0.00390625;
                }
                const unsigned long long s0 = clock64();
                const double* sf = B.sfx[it % kRing] + half * 32;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const long long f = f0 + q;
                    if (f < a.F) yb[f * a.fstride] = part[q] * si * sf[q];
                }
                es += clock64() - s0;
            }
        }
        if (a.prof && threadIdx.x == 0) {
            a.prof[blockIdx.x * 8 + 0] = clock64() - e_start;
            a.prof[blockIdx.x * 8 + 1] = ew;
            a.prof[blockIdx.x * 8 + 2] = es;
        }
    } else if (warp < kEpiWarps + kProdWarps) {
        // ------------------------------------------------------------ producers ----
        // thread p: 16-wide k chunk ck of fibres p/8 and p/8 + 32; the next tile's 32 values are
        // loaded right after this tile's digits are stored, so the loads overlap the ring wait
        const int p = threadIdx.x - kEpiWarps * 32;
        const int ck = p & 7, fl0 = p >> 3;
        long long cur_e = -1;
        int reloads = 0;
        unsigned long long pw = 0;
        const unsigned long long p_start = clock64();
        double v[2][16];
        auto load = [&](long long t) {
            const long long z = t / ntile;
            const long long z1 = z / a.zdiv, z2 = z % a.zdiv;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const long long f = (t % ntile) * kNT + fl0 + 32 * u;
                if (f < a.F && !(a.dbg & 4)) {
                    const double* xb =
                        a.x + z1 * a.sx1 + z2 * a.sx2 + f * a.fstride + static_cast<long long>(ck) * 16 * a.jstride;
                    if (a.jstride == 1) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const double2 uu = __ldg(reinterpret_cast<const double2*>(xb) + q);
                            v[u][2 * q] = uu.x;
                            v[u][2 * q + 1] = uu.y;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 16; ++q) v[u][q] = __ldg(xb + q * a.jstride);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[u][q] = (a.dbg & 4) ? 1.0 + q : 0.0;
                }
            }
        };
        if (t0 < t1) load(t0);
        for (long long t = t0; t < t1; ++t) {
            const long long it = t - t0;
            const int st = static_cast<int>(it % kStages);
            const long long e = e_index(t);
            if (e != cur_e) {
                if (reloads > 0) mbar_wait(&B.a_free, static_cast<uint32_t>((reloads - 1) & 1));
                const uint4* src = reinterpret_cast<const uint4*>(a.Ed + e * kABytes);
                uint4* dst = reinterpret_cast<uint4*>(sA);
                for (int q = p; q < kABytes / 16; q += kProducers) dst[q] = src[q];
                cur_e = e;
                ++reloads;
            }
            const unsigned long long w0 = clock64();
            mbar_wait(&B.empty[st], static_cast<uint32_t>(((it / kStages) & 1) ^ 1));
            pw += clock64() - w0;
            uint8_t* stage = ring + st * kStageBytes;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int fl = fl0 + 32 * u;
                double amax = 0.0;
#pragma unroll
                for (int q = 0; q < 16; ++q) amax = fmax(amax, fabs(v[u][q]));
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
                const int ex = oz_exponent(amax);
                const double sc = ldexp(1.0, 54 - ex);
                uint32_t lo[16], hi[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const unsigned long long wd = oz_word(v[u][q], sc) ^ kOff;  // bytes = digits (two's complement)
                    lo[q] = static_cast<uint32_t>(wd);
                    hi[q] = static_cast<uint32_t>(wd >> 32);
                }
                const int off = cm_off(fl, ck * 16);
#pragma unroll
                for (int s = 1; s <= kS; ++s) {
                    const int b = 7 - s;
                    const uint32_t* src = b < 4 ? lo : hi;
                    const uint32_t sel = static_cast<uint32_t>(b & 3);
                    uint32_t out[4];
#pragma unroll
                    for (int w4 = 0; w4 < 4; ++w4) {
                        const uint32_t p01 = __byte_perm(src[4 * w4], src[4 * w4 + 1], sel | ((sel + 4) << 4));
                        const uint32_t p23 = __byte_perm(src[4 * w4 + 2], src[4 * w4 + 3], sel | ((sel + 4) << 4));
                        out[w4] = __byte_perm(p01, p23, 0x5410);
                    }
                    *reinterpret_cast<uint4*>(stage + (s - 1) * kPlaneB + off) = make_uint4(out[0], out[1], out[2], out[3]);
                }
                if (ck == 0) B.sfx[it % kRing][fl] = ldexp(1.0, ex);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&B.full[st]);
            if (t + 1 < t1) load(t + 1);
        }
        if (a.prof && p == 0) {
            a.prof[blockIdx.x * 8 + 3] = clock64() - p_start;
            a.prof[blockIdx.x * 8 + 4] = pw;
        }
    } else if (lane == 0) {
        // ------------------------------------------------------------ MMA issue ----
        const uint32_t a0 = smem_u32(sA);
        unsigned long long mf = 0, me = 0;
        const unsigned long long m_start = clock64();
        for (long long t = t0; t < t1; ++t) {
            const long long it = t - t0;
            const int st = static_cast<int>(it % kStages);
            unsigned long long w0 = clock64();
            mbar_wait(&B.full[st], static_cast<uint32_t>((it / kStages) & 1));
            mf += clock64() - w0;
            tc_fence_after();
            const uint32_t b0 = smem_u32(ring + st * kStageBytes);
#pragma unroll
            for (int c = 2; c <= kS + 1; ++c) {
                w0 = clock64();
                mbar_wait(&B.d_empty[c - 2], static_cast<uint32_t>((it & 1) ^ 1));
                me += clock64() - w0;
                tc_fence_after();
                const uint32_t d = tD + (c - 2) * kNT;
                bool first = true;
#pragma unroll
                for (int s = 1; s < c; ++s) {
                    const int u = c - s;
                    if (s > kS || u > kS) continue;
#pragma unroll
                    for (int ks = 0; ks < kN / 32; ++ks) {
                        if ((a.dbg & 1) && !first) break;
                        tc_mma_ss(d, bdesc(a0 + (s - 1) * kPlaneA + ks * 256), bdesc(b0 + (u - 1) * kPlaneB + ks * 256),
                                  kIdesc, first ? 0u : 1u);
                        first = false;
                    }
                }
                tc_commit(&B.d_full[c - 2]);
            }
            tc_commit(&B.empty[st]);
            if (t + 1 < t1 && e_index(t + 1) != e_index(t)) tc_commit(&B.a_free);
        }
        if (a.prof) {
            a.prof[blockIdx.x * 8 + 5] = clock64() - m_start;
            a.prof[blockIdx.x * 8 + 6] = mf;
            a.prof[blockIdx.x * 8 + 7] = me;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(B.tmem_base));
#endif
}

}  // namespace oz
}  // namespace pqb
