// FP64 DMMA mode-product GEMM template (see kernels.cu header comment); instantiated in
// gemm_nk.cu (B row-major, "n contiguous") and gemm_kk.cu (B stored k-contiguous).
#pragma once
#include <stdexcept>

#include "kernels.hpp"

namespace pqb {

// ================================================================ DMMA GEMM =================

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int VEC>
__device__ __forceinline__ void cp_async(double* dst, const double* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int bytes = ok ? 8 * VEC : 0;  // 0 -> zero-fill, nothing read
    if constexpr (VEC == 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
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

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC>
__global__ void __launch_bounds__(TileCfg<BM, BN, BK, WM, WN, ST, BKM>::NT, 1) k_gemm(const GemmArgs g) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + ST * T::ASZ;

    const int z = blockIdx.z + g.z_off;
    const int z1 = z / g.zdiv, z2 = z - z1 * g.zdiv;
    const double* __restrict__ A = g.A + z1 * g.sA1 + z2 * g.sA2;
    const double* __restrict__ B = g.B + z1 * g.sB1 + z2 * g.sB2;
    double* C = g.C + z1 * g.sC1 + z2 * g.sC2;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / T::NWN, wn = warp % T::NWN;
    const int gid = lane >> 2, tig = lane & 3;

    if (g.sq_count && g.sq_round >= g.sq_count[z]) {
        // expm squaring already finished for this matrix: carry it through unchanged.
        for (int e = tid; e < BM * BN; e += T::NT) {
            const int m = m0 + e / BN, n = n0 + e % BN;
            if (m < g.M && n < g.N) C[(long long)m * g.ldc + n] = A[(long long)m * g.lda + n];
        }
        return;
    }

    auto load_stage = [&](int stage, int kt) {
        const int k0 = kt * BK;
        double* dA = sA + stage * T::ASZ;
        double* dB = sB + stage * T::BSZ;
        constexpr int KV = BK / VEC;
#pragma unroll
        for (int c = tid; c < BM * KV; c += T::NT) {
            const int r = c / KV, kc = (c % KV) * VEC;
            const int gm = m0 + r, gk = k0 + kc;
            const bool ok = gm < g.M && gk < g.K;
            cp_async<VEC>(dA + r * T::SA + kc, ok ? A + (long long)gm * g.lda + gk : A, ok);
        }
        if constexpr (BKM) {
#pragma unroll
            for (int c = tid; c < BN * KV; c += T::NT) {
                const int r = c / KV, kc = (c % KV) * VEC;
                const int gn = n0 + r, gk = k0 + kc;
                const bool ok = gn < g.N && gk < g.K;
                cp_async<VEC>(dB + r * T::SB + kc, ok ? B + (long long)gn * g.ldb + gk : B, ok);
            }
        } else {
            constexpr int NV = BN / VEC;
#pragma unroll
            for (int c = tid; c < BK * NV; c += T::NT) {
                const int r = c / NV, nc = (c % NV) * VEC;
                const int gk = k0 + r, gn = n0 + nc;
                const bool ok = gk < g.K && gn < g.N;
                cp_async<VEC>(dB + r * T::SB + nc, ok ? B + (long long)gk * g.ldb + gn : B, ok);
            }
        }
    };

    double acc[T::MI][T::NI][2];
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int KT = (g.K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < KT) load_stage(s, s);
        cp_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
        cp_wait<ST - 2>();
        __syncthreads();
        {
            const int nk = kt + ST - 1;
            if (nk < KT) load_stage(nk % ST, nk);
            cp_commit();
        }
        const int st = kt % ST;
        const double* tA = sA + st * T::ASZ + (wm * WM + gid) * T::SA + tig;
        const double* tB = BKM ? sB + st * T::BSZ + (wn * WN + gid) * T::SB + tig
                               : sB + st * T::BSZ + tig * T::SB + wn * WN + gid;
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
    }
    cp_wait<0>();

    // ---- epilogue (registers -> global), order of the reference's scalar updates ----
    const double alpha = g.alpha_z ? g.alpha_z[z1] : g.alpha;
    const int nt = g.nterms ? g.nterms[z1] : 0;
    const double* crow = g.coef ? g.coef + (long long)z1 * g.cld : nullptr;
    const double* ext = g.ext ? g.ext + (long long)(z1 / g.ext_group) * g.ext_group * g.ext_s + z2 * g.sC2 : nullptr;
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
        const int m = m0 + wm * WM + i * 8 + gid;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < T::NI; ++j) {
            const int nb = n0 + wn * WN + j * 8 + 2 * tig;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int n = nb + e;
                if (n >= g.N) continue;
                const long long off = (long long)m * g.ldc + n;
                double v = __dmul_rn(alpha, acc[i][j][e]);
                if (g.accumulate) v = __dadd_rn(C[off], v);
                for (int t = 0; t < nt; ++t) v = __dadd_rn(v, __dmul_rn(crow[t], ext[t * g.ext_s + off]));
                C[off] = v;
            }
        }
    }
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool BKM, int VEC>
static int launch_cfg(const GemmArgs& g, cudaStream_t s) {
    using T = TileCfg<BM, BN, BK, WM, WN, ST, BKM>;
    auto kern = k_gemm<BM, BN, BK, WM, WN, ST, BKM, VEC>;
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
        kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)zc), T::NT, T::SMEM, s>>>(a);
        ++launches;
    }
    return launches;
}


// Tile shapes: id 0 = 128x128 (8 warps of 64x32), 1 = 128x64, 2 = 64x128, 3 = 64x64.
template <bool BKM>
int launch_gemm_family(const GemmArgs& g, bool vec2, int shape, cudaStream_t s) {
    switch (shape) {
        case 0: return vec2 ? launch_cfg<128, 128, 16, 64, 32, 3, BKM, 2>(g, s) : launch_cfg<128, 128, 16, 64, 32, 3, BKM, 1>(g, s);
        case 1: return vec2 ? launch_cfg<128, 64, 16, 64, 32, 3, BKM, 2>(g, s) : launch_cfg<128, 64, 16, 64, 32, 3, BKM, 1>(g, s);
        case 2: return vec2 ? launch_cfg<64, 128, 16, 32, 64, 3, BKM, 2>(g, s) : launch_cfg<64, 128, 16, 32, 64, 3, BKM, 1>(g, s);
        default: return vec2 ? launch_cfg<64, 64, 16, 32, 32, 3, BKM, 2>(g, s) : launch_cfg<64, 64, 16, 32, 32, 3, BKM, 1>(g, s);
    }
}

}  // namespace pqb
