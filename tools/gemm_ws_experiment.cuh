// Warp-specialised variant of the band-tile mode-product GEMM (gemm.cuh k_gemm): one producer warp
// moves the operand rows with cp.async.bulk (the TMA engine's 1-D copies, each row into its padded
// shared-memory row, completion counted on a per-stage mbarrier), and the four consumer warps only
// wait on that barrier, load fragments and issue DMMAs -- no address arithmetic, LDGSTS or block
// barrier in their loop (ncu on k_gemm: ~170 of the ~330 instructions per 16-wide k slice were the
// load issue path).  Requires whole tiles (M % BM, N % BN, K % BK == 0), 16-byte aligned rows and
// no squaring-count carry; launch_gemm_family falls back to k_gemm otherwise.
#pragma once

#include "gemm.cuh"

namespace pqb {

__device__ __forceinline__ uint32_t ws_smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void ws_bar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ws_smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void ws_bar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(ws_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void ws_bar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(ws_smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void ws_bar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t a = ws_smem_u32(b);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void ws_bulk_row(double* dst, const double* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ws_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(ws_smem_u32(bar))
                 : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM>
struct WsCfg {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    static constexpr int NC = T::NT;  // consumer threads
    static constexpr int NT = NC + 32;
    static constexpr int NW = NC / 32;
    static constexpr int SMEM = T::SMEM + 2 * ST * 8;
};

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int MINB>
__global__ void __launch_bounds__(WsCfg<BM, BN, BK, WM, WN, ST, BKM>::NT, MINB) k_gemm_ws(const GemmArgs g) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    using W = WsCfg<BM, BN, BK, WM, WN, ST, BKM>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + ST * T::ASZ;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * (T::ASZ + T::BSZ));
    uint64_t* empty = full + ST;

    const int z = blockIdx.z + g.z_off;
    const int z1 = z / g.zdiv, z2 = z - z1 * g.zdiv;
    const double* __restrict__ A = g.A + z1 * g.sA1 + z2 * g.sA2;
    const double* __restrict__ B = g.B + z1 * g.sB1 + z2 * g.sB2;
    double* C = g.C + z1 * g.sC1 + z2 * g.sC2;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            ws_bar_init(&full[s], 1);
            ws_bar_init(&empty[s], W::NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- the K range this tile streams (negligible-block skip, same rules as k_gemm) ----
    const int wm = (warp < W::NW ? warp : 0) / T::NWN, wn = (warp < W::NW ? warp : 0) % T::NWN;
    int kt_lo = 0, KT = g.K / BK;
    int w_lo = 0, w_hi = KT;
    if (g.band) {
        int e, r0, te, wr, we;
        if (g.band_mode == 3) {
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
        constexpr int SH = BK == 16 ? 1 : (BK == 32 ? 2 : 0);
        kt_lo = hi > lo ? (lo >> SH) : 0;
        KT = min(KT, hi > lo ? ((hi + (1 << SH) - 1) >> SH) : 0);
        if (we <= 32) {
            const int wb = wr >> 5;
            const int2 mine = wb < nb ? br[wb] : make_int2(0, 0);
            w_lo = mine.x >> SH;
            w_hi = (mine.y + (1 << SH) - 1) >> SH;
        } else {
            w_lo = kt_lo;
            w_hi = KT;
        }
    }
    const int NKT = KT > kt_lo ? KT - kt_lo : 0;

    if (warp == W::NW) {
        // ------------------------------------------------------------ producer warp ----
        constexpr uint32_t bytes = (BM * BK + (BKM ? BN * BK : BK * BN)) * 8;
        for (int i = 0; i < NKT; ++i) {
            const int st = i % ST;
            if (i >= ST) ws_bar_wait(&empty[st], static_cast<uint32_t>(((i / ST) - 1) & 1));
            const int k0 = (kt_lo + i) * BK;
            if (lane == 0) ws_bar_expect_tx(&full[st], bytes);
            __syncwarp();
            double* a_dst = sA + st * T::ASZ;
            for (int r = lane; r < BM; r += 32)
                ws_bulk_row(a_dst + r * T::SA, A + (long long)(m0 + r) * g.lda + k0, BK * 8, &full[st]);
            double* b_dst = sB + st * T::BSZ;
            if constexpr (BKM) {
                for (int c = lane; c < BN; c += 32)
                    ws_bulk_row(b_dst + c * T::SB, B + (long long)(n0 + c) * g.ldb + k0, BK * 8, &full[st]);
            } else {
                for (int k = lane; k < BK; k += 32)
                    ws_bulk_row(b_dst + k * T::SB, B + (long long)(k0 + k) * g.ldb + n0, BN * 8, &full[st]);
            }
        }
        asm volatile("griddepcontrol.launch_dependents;");
        return;
    }

    // ------------------------------------------------------------ consumer warps ----
    const int gid = lane >> 2, tig = lane & 3;
    if (g.flop_counter && lane == 0) {
        const long long rows = max(0, min(WM, g.M - (m0 + wm * WM))), cols = max(0, min(WN, g.N - (n0 + wn * WN)));
        const int lo = max(kt_lo, w_lo), hi = min(KT, w_hi);
        const long long kexec = hi > lo ? min(hi * BK, g.K) - lo * BK : 0;
        atomicAdd(g.flop_counter, static_cast<unsigned long long>(2 * rows * cols * kexec));
    }
    double acc[T::MI][T::NI][2];
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* tA0 = sA + (wm * WM + gid) * T::SA + tig;
    const double* tB0 = BKM ? sB + (wn * WN + gid) * T::SB + tig : sB + tig * T::SB + wn * WN + gid;
#pragma unroll 1
    for (int i = 0; i < NKT; ++i) {
        const int st = i % ST;
        ws_bar_wait(&full[st], static_cast<uint32_t>((i / ST) & 1));
        const int kabs = kt_lo + i;
        if (kabs >= w_lo && kabs < w_hi) {
            const double* tA = tA0 + st * T::ASZ;
            const double* tB = tB0 + st * T::BSZ;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[T::MI], b[T::NI];
#pragma unroll
                for (int ii = 0; ii < T::MI; ++ii) a[ii] = tA[ii * 8 * T::SA + kk];
#pragma unroll
                for (int j = 0; j < T::NI; ++j) b[j] = BKM ? tB[j * 8 * T::SB + kk] : tB[kk * T::SB + j * 8];
#pragma unroll
                for (int ii = 0; ii < T::MI; ++ii)
#pragma unroll
                    for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[ii][j], a[ii], b[j]);
            }
        }
        __syncwarp();
        if (lane == 0) ws_bar_arrive(&empty[st]);
    }
    asm volatile("griddepcontrol.launch_dependents;");

    // ---- epilogue (as k_gemm) ----
    const double alpha = g.alpha_z ? g.alpha_z[z1] : g.alpha;
    const int nt = g.nterms ? g.nterms[z1] : 0;
    const int mb = m0 + wm * WM + gid, nbase = n0 + wn * WN + 2 * tig;
    const double* crow = g.coef ? g.coef + (long long)z1 * g.cld : nullptr;
    const double* ext = g.ext ? g.ext + (long long)(z1 / g.ext_group) * g.ext_group * g.ext_s + z2 * g.sC2 : nullptr;
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
            const double* row = src + (long long)m * g.ldc;
#pragma unroll
            for (int j = 0; j < T::NI; ++j) {
                const int n = nbase + j * 8;
                const double2 v = *reinterpret_cast<const double2*>(row + n);
                if (plain) {
                    acc[i][j][0] = __dadd_rn(v.x, acc[i][j][0]);
                    acc[i][j][1] = __dadd_rn(v.y, acc[i][j][1]);
                } else {
                    acc[i][j][0] = __dadd_rn(acc[i][j][0], __dmul_rn(coef, v.x));
                    acc[i][j][1] = __dadd_rn(acc[i][j][1], __dmul_rn(coef, v.y));
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
        double* row = C + (long long)m * g.ldc;
#pragma unroll
        for (int j = 0; j < T::NI; ++j)
            *reinterpret_cast<double2*>(row + nbase + j * 8) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// true when the warp-specialised tile applies: whole tiles, 16-byte aligned rows and bases
template <int BM, int BN, int BK>
static bool ws_ok(const GemmArgs& g) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return !g.sq_count && g.M % BM == 0 && g.N % BN == 0 && g.K % BK == 0 && g.lda % 2 == 0 && g.ldb % 2 == 0 &&
           g.ldc % 2 == 0 && g.sA1 % 2 == 0 && g.sA2 % 2 == 0 && g.sB1 % 2 == 0 && g.sB2 % 2 == 0 && g.sC1 % 2 == 0 &&
           g.sC2 % 2 == 0 && al(g.A) && al(g.B) && al(g.C) && (!g.ext || (g.ext_s % 2 == 0 && al(g.ext)));
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int MINB>
static int launch_ws(const GemmArgs& g, cudaStream_t s) {
    using W = WsCfg<BM, BN, BK, WM, WN, ST, BKM>;
    auto kern = k_gemm_ws<BM, BN, BK, WM, WN, ST, BKM, MINB>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, W::SMEM);
        attr_done = true;
    }
    const long long gx = g.M / BM, gy = g.N / BN;
    if (gx > 2147483647LL || gy > 65535) throw std::invalid_argument("mode product: grid too large");
    int launches = 0;
    GemmArgs a = g;
    for (int z0 = 0; z0 < g.Z; z0 += 65535) {
        a.z_off = z0;
        const int zc = g.Z - z0 < 65535 ? g.Z - z0 : 65535;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)gx, (unsigned)gy, (unsigned)zc);
        cfg.blockDim = dim3(W::NT);
        cfg.dynamicSmemBytes = W::SMEM;
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

}  // namespace pqb
