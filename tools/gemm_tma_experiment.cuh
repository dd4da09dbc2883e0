// A/B experiment (VERDICT r01 "next round" item 5): the exponential-as-A band tile (32x128x16,
// four 32x32 warps, the dominant k_gemm of the node sweep and the squaring) with its operands
// staged by TMA tensor copies (cp.async.bulk.tensor + mbarrier transaction counts, one elected
// thread issues both copies per stage) instead of per-thread 16-byte cp.async.
//
// Shared-memory layouts chosen so the m8n8k4 fragment reads are conflict-free WITHOUT swizzle or
// padding (which TMA boxes cannot express): the operands are viewed as higher-rank tensors whose
// box order interleaves the fragment's fast index:
//   A (exponential rows m, k contiguous): 3D (k_lo = 4, row, k_hi) with strides (8 B, lda*8, 32 B),
//     box {4, 32, BK/4} -> smem [k_hi][row][k_lo]: a warp's A fragment (8 rows x 4 k) is 32
//     consecutive doubles;
//   B (X rows k, n contiguous): 5D (n_lo = 8, k, n_hi, z2, z1) with strides (8 B, ldb*8, 64 B,
//     sB2*8, sB1*8), box {8, BK, BN/8, 1, 1} -> smem [n_hi][k][n_lo]: a B fragment (4 k x 8 n) is 32
//     consecutive doubles.
// Out-of-range box elements (edges, band limits past K) are zero-filled by the TMA unit.
// Plain-store epilogue with alpha (the node sweep / squaring mode products 0 and 1 need no more).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "gemm.cuh"

namespace pqb {

__device__ __forceinline__ void mbar_init(unsigned addr, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(addr), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned addr, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(addr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_3d(unsigned dst, const CUtensorMap* map, unsigned mbar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_5d(unsigned dst, const CUtensorMap* map, unsigned mbar, int c0, int c1, int c2,
                                       int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
        "[%2];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int ST>
struct TmaCfg {
    static constexpr int NWM = BM / WM, NWN = BN / WN, NT = NWM * NWN * 32;
    static constexpr int ASZ = BM * BK, BSZ = BK * BN;  // doubles per stage
    static constexpr int SMEM = ST * (ASZ + BSZ) * 8 + ST * 8 + 128;
    static constexpr int MI = WM / 8, NI = WN / 8;
};

// A rows: band_mode 1 (stacked node exponentials, M = Z*n): row m0; band_mode 2 (exponential z1,
// rows contiguous per z1): row z1*M + m0 -- the A map spans all rows.
template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB>
__global__ void __launch_bounds__(TmaCfg<BM, BN, BK, WM, WN, ST>::NT, MINB)
    k_gemm_tma(const GemmArgs g, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
    using T = TmaCfg<BM, BN, BK, WM, WN, ST>;
    extern __shared__ __align__(128) double smem_tma[];
    double* sA = smem_tma;
    double* sB = smem_tma + ST * T::ASZ;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_tma + ST * (T::ASZ + T::BSZ));
    const int z = blockIdx.z;
    const int z1 = z / g.zdiv, z2 = z - z1 * g.zdiv;
    double* C = g.C + z1 * g.sC1 + z2 * g.sC2;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / T::NWN, wn = warp % T::NWN;
    const int gid = lane >> 2, tig = lane & 3;
    const int arow = (g.band_mode == 2 ? z1 * g.M : 0) + m0;
    const unsigned sA_base = static_cast<unsigned>(__cvta_generic_to_shared(sA));
    const unsigned sB_base = static_cast<unsigned>(__cvta_generic_to_shared(sB));
    const unsigned bar_base = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) mbar_init(bar_base + 8u * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // negligible-block K range (same tables as k_gemm)
    int kt_lo = 0, KT = (g.K + BK - 1) / BK;
    if (g.band) {
        const int e = g.band_mode == 1 ? m0 / g.band_rows : z1;
        const int r0 = g.band_mode == 1 ? m0 % g.band_rows : m0;
        const int2 v = g.band[(long long)e * g.band_stride + (r0 >> 5)];
        constexpr int SH = BK == 16 ? 1 : 0;
        kt_lo = v.y > v.x ? (v.x >> SH) : 0;
        KT = min(KT, v.y > v.x ? ((v.y + (1 << SH) - 1) >> SH) : 0);
    }
    const int NKT = KT > kt_lo ? KT - kt_lo : 0;
    if (g.flop_counter && lane == 0) {
        const long long rows = max(0, min(WM, g.M - (m0 + wm * WM))), cols = max(0, min(WN, g.N - (n0 + wn * WN)));
        const long long kexec = NKT > 0 ? min(KT * BK, g.K) - kt_lo * BK : 0;
        atomicAdd(g.flop_counter, static_cast<unsigned long long>(2 * rows * cols * kexec));
    }
    constexpr unsigned kTx = (T::ASZ + T::BSZ) * 8;
    auto issue = [&](int kt) {  // k-slice kt (relative) into stage kt % ST
        const int s = kt % ST, k0 = (kt_lo + kt) * BK;
        mbar_expect_tx(bar_base + 8u * s, kTx);
        tma_3d(sA_base + 8u * s * T::ASZ, &tmA, bar_base + 8u * s, 0, arow, k0 / 4);
        tma_5d(sB_base + 8u * s * T::BSZ, &tmB, bar_base + 8u * s, 0, k0, n0 / 8, z2, z1);
    };
    if (tid == 0)
        for (int s = 0; s < ST - 1 && s < NKT; ++s) issue(s);

    double acc[T::MI][T::NI][2];
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // fragment bases: A [k_hi][row][k_lo], B [n_hi][k][n_lo]
    const int arow0 = wm * WM + gid;
    const int nb0 = wn * WN / 8;
#pragma unroll 1
    for (int kt = 0; kt < NKT; ++kt) {
        if (tid == 0 && kt + ST - 1 < NKT) issue(kt + ST - 1);
        const int s = kt % ST;
        mbar_wait(bar_base + 8u * s, (kt / ST) & 1);
        const double* tA = sA + s * T::ASZ;
        const double* tB = sB + s * T::BSZ;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[T::MI], b[T::NI];
#pragma unroll
            for (int i = 0; i < T::MI; ++i) a[i] = tA[((kk >> 2) * BM + arow0 + i * 8) * 4 + tig];
#pragma unroll
            for (int j = 0; j < T::NI; ++j) b[j] = tB[((nb0 + j) * BK + kk + tig) * 8 + gid];
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
        }
        __syncthreads();  // every warp is done with stage s before it is refilled (issue at kt + 1)
    }
    asm volatile("griddepcontrol.launch_dependents;");
    const double alpha = g.alpha_z ? g.alpha_z[z1] : g.alpha;
    const int mb = m0 + wm * WM + gid, nbase = n0 + wn * WN + 2 * tig;
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
        const int m = mb + i * 8;
        if (m >= g.M) continue;
        double* row = C + (long long)m * g.ldc;
#pragma unroll
        for (int j = 0; j < T::NI; ++j) {
            const int n = nbase + j * 8;
            const double x0 = alpha * acc[i][j][0], x1 = alpha * acc[i][j][1];
            if (n + 1 < g.N) {
                *reinterpret_cast<double2*>(row + n) = make_double2(x0, x1);
            } else if (n < g.N) {
                row[n] = x0;
            }
        }
    }
}

// host: tensor maps for a band-mode-1/2 mode product (A = exponential rows, B = X row-major)
inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

template <int BM, int BN, int BK>
inline bool tma_maps(const GemmArgs& g, CUtensorMap* A, CUtensorMap* B, char* why = nullptr) {
    auto enc = tma_encoder();
    if (!enc || g.b_kmajor || (g.band_mode != 1 && g.band_mode != 2)) return false;
    const long long rows = g.band_mode == 2 ? (long long)(g.Z / g.zdiv) * g.M : g.M;
    if (g.band_mode == 2 && g.sA1 != (long long)g.M * g.lda) return false;
    cuuint64_t adim[3] = {4, (cuuint64_t)rows, (cuuint64_t)((g.K + 3) / 4)};
    cuuint64_t astr[2] = {(cuuint64_t)g.lda * 8, 32};
    cuuint32_t abox[3] = {4, BM, BK / 4};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(A, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(g.A), adim, astr, abox, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        if (why) snprintf(why, 128, "A map: CUresult %d", (int)r);
        return false;
    }
    const long long Z1 = g.Z / g.zdiv;
    cuuint64_t bdim[5] = {8, (cuuint64_t)g.K, (cuuint64_t)((g.N + 7) / 8), (cuuint64_t)g.zdiv, (cuuint64_t)Z1};
    cuuint64_t bstr[4] = {(cuuint64_t)g.ldb * 8, 64, (cuuint64_t)(g.zdiv > 1 ? g.sB2 * 8 : 16),
                          (cuuint64_t)(Z1 > 1 ? g.sB1 * 8 : 16)};
    cuuint32_t bbox[5] = {8, BK, BN / 8, 1, 1};
    r = enc(B, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(g.B), bdim, bstr, bbox, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        if (why) snprintf(why, 128, "B map: CUresult %d", (int)r);
        return false;
    }
    return true;
}

template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB>
inline int launch_tma(const GemmArgs& g, cudaStream_t s, char* why = nullptr) {
    CUtensorMap A, B;
    if (!tma_maps<BM, BN, BK>(g, &A, &B, why)) return -1;
    using T = TmaCfg<BM, BN, BK, WM, WN, ST>;
    auto kern = k_gemm_tma<BM, BN, BK, WM, WN, ST, MINB>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
        attr = true;
    }
    dim3 grid((g.M + BM - 1) / BM, (g.N + BN - 1) / BN, g.Z);
    kern<<<grid, T::NT, T::SMEM, s>>>(g, A, B);
    return 1;
}

}  // namespace pqb
