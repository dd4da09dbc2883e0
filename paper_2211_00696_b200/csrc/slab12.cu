// Fused last-two-mode product of a 3-D Kronecker apply for n1 = n2 = 128 (config 2's and config
// 4's operators): per x-slab X_s = X[i0, :, :] (128 x 128, contiguous),
//     Y_s = (E1 X_s) E2^T          -- mode 1 then mode 2, kron.hpp:65-87 applied twice,
// in ONE kernel.  The mode-1 intermediate never goes to HBM: a CTA owns a 32-row quarter of a
// slab, computes its 32 x 128 block of T = E1 X_s (the 32x128x16 band tile of gemm.cuh, operands
// streamed by cp.async), keeps it in shared memory and multiplies it by E2^T (each warp one
// 32-column block, its E2 fragments read straight from L1/L2 with a one-step register prefetch).
// Per squaring step and column this saves one HBM write + read of the whole vector and one launch
// with its partial last wave.
//
// Bitwise contract: every output element is accumulated over exactly the k4 steps, in the same
// ascending order and DMMA grouping, that the two separate band tiles execute (mode 1: the 16-wide
// k-slices of E1's 32-row block rq, and within them the k4 steps of the element's 8-row group of E1;
// mode 2: likewise for E2's block / group of the output column), so the fused result equals the
// unfused chain bit for bit (tests/test_gpu_slab12.py).
#include <type_traits>

#include "gemm.cuh"

namespace pqb {

namespace {
constexpr int S_N = 128;                       // n1 = n2
constexpr int S_BK = 16, S_ST = 2;             // k-slice width and cp.async stages of the mode-1 phase
constexpr int S_SA = S_BK + 4;                 // padded row strides (conflict-free fragment reads)
constexpr int S_SB = S_N + 4;
constexpr int S_ASZ = 32 * S_SA, S_BSZ = S_BK * S_SB;
constexpr int S_SMEM = S_ST * (S_ASZ + S_BSZ) * 8;  // 44 KB -> 4 CTAs (16 warps) per SM
static_assert(32 * S_N * 8 <= S_SMEM, "the mode-1 block T aliases the pipeline buffers");

// 16-slice range [lo, hi) of a band entry exactly as gemm_tile derives it for a one-block tile
__device__ __forceinline__ void slice_range(const int2* band, long long idx, int& lo, int& hi) {
    lo = 0;
    hi = S_N / S_BK;
    if (!band) return;
    const int2 v = band[idx];
    if (v.y > v.x) {
        lo = v.x >> 1;
        hi = min(hi, (v.y + 1) >> 1);
    } else {
        lo = hi = 0;
    }
}
// DMMAs of the fragment rows (ROWS = true) or columns whose bit is set in MASK; dispatched through a
// switch on the run-time mask so the skipped DMMAs are not issued at all (a plain `if` around them
// is if-converted into predicated DMMAs, which still occupy the tensor pipe)
template <int MASK, bool ROWS>
__device__ __forceinline__ void dmma_masked(double (&acc)[4][4][2], const double (&a)[4], const double (&b)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((MASK >> (ROWS ? i : j)) & 1) dmma_8x8x4(acc[i][j], a[i], b[j]);
}
template <bool ROWS>
__device__ __forceinline__ void dmma_switch(unsigned mask, double (&acc)[4][4][2], const double (&a)[4],
                                            const double (&b)[4]) {
    switch (mask) {
        case 1: dmma_masked<1, ROWS>(acc, a, b); break;
        case 2: dmma_masked<2, ROWS>(acc, a, b); break;
        case 3: dmma_masked<3, ROWS>(acc, a, b); break;
        case 4: dmma_masked<4, ROWS>(acc, a, b); break;
        case 5: dmma_masked<5, ROWS>(acc, a, b); break;
        case 6: dmma_masked<6, ROWS>(acc, a, b); break;
        case 7: dmma_masked<7, ROWS>(acc, a, b); break;
        case 8: dmma_masked<8, ROWS>(acc, a, b); break;
        case 9: dmma_masked<9, ROWS>(acc, a, b); break;
        case 10: dmma_masked<10, ROWS>(acc, a, b); break;
        case 11: dmma_masked<11, ROWS>(acc, a, b); break;
        case 12: dmma_masked<12, ROWS>(acc, a, b); break;
        case 13: dmma_masked<13, ROWS>(acc, a, b); break;
        case 14: dmma_masked<14, ROWS>(acc, a, b); break;
        case 15: dmma_masked<15, ROWS>(acc, a, b); break;
        default: break;
    }
}

// fine gating of 8-row group `grp` (kernels.hpp launch_band_ranges): k4 steps lo | len << 16
__device__ __forceinline__ unsigned fine_range(const int2* band, long long rec, int grp) {
    if (!band) return 0xffffu << 16;
    const int2 v = band[rec + S_N / 32 + grp];
    return v.y > v.x ? static_cast<unsigned>(v.x) | (static_cast<unsigned>(v.y - v.x) << 16) : 0u;
}
}  // namespace

template <bool SKEW, bool PACK>
__global__ void __launch_bounds__(128, 4) k_slab12(const Slab12Args g) {
    extern __shared__ __align__(16) double smem[];
    const int rq = blockIdx.x;
    const long long z = static_cast<long long>(blockIdx.y) + g.z_off;
    const int z1 = static_cast<int>(z / g.n0);
    const long long i0 = z - static_cast<long long>(z1) * g.n0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;

    const double* __restrict__ E1 = g.E1 + z1 * g.sE1;
    const double* __restrict__ E2 = g.E2 + z1 * g.sE2;
    const double* __restrict__ X = g.X + z1 * g.sX + i0 * (S_N * S_N);
    double* Y = g.Y + z1 * g.sY + i0 * (S_N * S_N) + rq * 32 * S_N;

    asm volatile("griddepcontrol.wait;" ::: "memory");

    int lo1, hi1;
    slice_range(g.band1, z1 * g.sband1 + rq, lo1, hi1);
    const int NKT = hi1 > lo1 ? hi1 - lo1 : 0;
    unsigned fine[4];  // phase 1: E1 row groups of this quarter (fragment rows i)
#pragma unroll
    for (int i = 0; i < 4; ++i) fine[i] = fine_range(g.band1, z1 * g.sband1, rq * 4 + i);
    // phase 2's band entries are requested now (lane 0: the warp's coarse entry, lanes 1-4: its four
    // fine entries) and handed out by shuffles after phase 1, instead of a dependent L2 round trip there
    int2 pre2 = make_int2(0, 0);
    if (g.band2 && lane < 5)
        pre2 = g.band2[z1 * g.sband2 + (lane == 0 ? warp : S_N / 32 + warp * 4 + lane - 1)];

    // ---- phase 1: T = E1[rq block] X_s  (32 x 128), cp.async 2-stage pipeline ----
    double* sA = smem;
    double* sB = smem + S_ST * S_ASZ;
    const unsigned sA_base = static_cast<unsigned>(__cvta_generic_to_shared(sA));
    const unsigned sB_base = static_cast<unsigned>(__cvta_generic_to_shared(sB));
    // A: 32 rows x 8 chunks -> 2 per thread (rows r, r + 16); B: 16 rows x 64 chunks -> 8 per thread
    const int ar = tid >> 3, ak = (tid & 7) * 2;
    const double* a_p = E1 + (rq * 32 + ar) * S_N + lo1 * S_BK + ak;
    const unsigned a_dst = sA_base + 8u * (ar * S_SA + ak);
    const int br = tid >> 6, bn = (tid & 63) * 2;
    const double* b_p = X + static_cast<long long>(lo1 * S_BK + br) * S_N + bn;
    const unsigned b_dst = sB_base + 8u * (br * S_SB + bn);
    auto load = [&](int stage) {
#pragma unroll
        for (int it = 0; it < 2; ++it) cp_async<2>(a_dst + 8u * (stage * S_ASZ + it * 16 * S_SA), a_p + it * 16 * S_N, true);
#pragma unroll
        for (int it = 0; it < 8; ++it) cp_async<2>(b_dst + 8u * (stage * S_BSZ + it * 2 * S_SB), b_p + it * 2 * S_N, true);
        a_p += S_BK;
        b_p += S_BK * S_N;
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    if (NKT > 0) load(0);
    cp_commit();
    const double* tA0 = sA + gid * S_SA + tig;
    const double* tB0 = sB + tig * S_SB + warp * 32 + gid;
#pragma unroll 1
    for (int kt = 0; kt < NKT; ++kt) {
        cp_wait<0>();
        __syncthreads();
        if (kt + 1 < NKT) load((kt + 1) & 1);
        cp_commit();
        const double* tA = tA0 + (kt & 1) * S_ASZ;
        const double* tB = tB0 + (kt & 1) * S_BSZ;
        const unsigned q0 = static_cast<unsigned>(((lo1 + kt) * S_BK) >> 2);
        bool full = true;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            full = full && (fine[i] & 0xffffu) <= q0 && q0 + S_BK / 4 <= (fine[i] & 0xffffu) + (fine[i] >> 16);
        if (full) {
#pragma unroll
            for (int kk = 0; kk < S_BK; kk += 4) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = tA[i * 8 * S_SA + kk];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = tB[kk * S_SB + j * 8];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
            }
        } else {
#pragma unroll 1
            for (int kk = 0; kk < S_BK; kk += 4) {
                const unsigned kq = q0 + (kk >> 2);
                unsigned mask = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) mask |= (kq - (fine[i] & 0xffffu) < (fine[i] >> 16) ? 1u : 0u) << i;
                if (mask == 0u) continue;
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = tA[i * 8 * S_SA + kk];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = tB[kk * S_SB + j * 8];
                dmma_switch<true>(mask, acc, a, b);
            }
        }
    }
    unsigned long long f1 = 0;  // executed phase-1 DMMA work of this warp
    if (g.flop_counter)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int flo = static_cast<int>(fine[i] & 0xffffu), fhi = flo + static_cast<int>(fine[i] >> 16);
            f1 += 2ull * 8 * 32 * 4 * max(0, min(hi1 * 4, fhi) - max(lo1 * 4, flo));
        }
    cp_wait<0>();
    __syncthreads();  // every warp is done with the stage buffers: T overwrites them

    // T[r][c] at r*128 + (c ^ ((r & 3) << 2)): the phase-2 A-fragment reads (rows gid, 4
    // consecutive k) then hit 16 distinct bank pairs per half-warp; pairs (c, c+1) stay adjacent.
    double* T = smem;
    const int swz = (gid & 3) << 2;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = i * 8 + gid, c = warp * 32 + j * 8 + 2 * tig;
            *reinterpret_cast<double2*>(T + r * S_N + (c ^ swz)) = make_double2(acc[i][j][0], acc[i][j][1]);
            acc[i][j][0] = acc[i][j][1] = 0.0;
        }
    __syncthreads();

    // ---- phase 2: Y[rq block, warp block] = T E2[warp block]^T, k over E2's block band ----
    int lo2 = 0, hi2 = S_N / S_BK;
    {
        const int cx = __shfl_sync(0xffffffffu, pre2.x, 0), cy = __shfl_sync(0xffffffffu, pre2.y, 0);
        if (g.band2) {  // as slice_range
            if (cy > cx) {
                lo2 = cx >> 1;
                hi2 = min(hi2, (cy + 1) >> 1);
            } else {
                lo2 = hi2 = 0;
            }
        }
    }
    const int kb = lo2 * S_BK, ke = hi2 > lo2 ? hi2 * S_BK : kb;
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // E2 row groups = columns j (as fine_range)
        const int fx = __shfl_sync(0xffffffffu, pre2.x, j + 1), fy = __shfl_sync(0xffffffffu, pre2.y, j + 1);
        fine[j] = !g.band2 ? 0xffffu << 16
                           : fy > fx ? static_cast<unsigned>(fx) | (static_cast<unsigned>(fy - fx) << 16) : 0u;
    }
    // E2 fragment of column group j at k4 step q: row-major E2[(warp*32 + j*8 + gid)][4q + tig] (8 lines
    // per warp load), or the fragment-major copy (PACK: one contiguous 256-byte run per warp load)
    const double* e2 = PACK ? g.E2p + z1 * g.sE2p + static_cast<long long>(warp) * 4 * (S_N / 4) * 32 + lane
                            : E2 + (warp * 32 + gid) * S_N + tig;
    auto ld_e2 = [&](int j, int q) { return PACK ? __ldg(e2 + (j * (S_N / 4) + q) * 32) : __ldg(e2 + j * 8 * S_N + q * 4); };
    const double* tr = T + gid * S_N;
    if constexpr (SKEW) {
        // Skewed k loop: column group j walks its OWN k4 range [qa_j, qa_j + len_j) -- step t
        // multiplies T's columns at k4 = qa_j + t -- so while every group still has steps left all
        // 16 DMMAs of a step issue (T is fully resident, so the groups need not share a k window).
        // Each accumulator still sees its k4 steps in ascending order: bitwise the aligned loop.
        int qa[4], len[4];
        int lmin = 1 << 30;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int lo = max(static_cast<int>(fine[j] & 0xffffu), kb / 4);
            const int hi = min(static_cast<int>(fine[j] & 0xffffu) + static_cast<int>(fine[j] >> 16), ke / 4);
            qa[j] = lo;
            len[j] = max(0, hi - lo);
            lmin = min(lmin, len[j]);
        }
        double bn_[4];
        if (lmin > 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) bn_[j] = ld_e2(j, qa[j]);
        }
#pragma unroll 1
        for (int t = 0; t < lmin; ++t) {
            double b[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = bn_[j];
            if (t + 1 < lmin) {
#pragma unroll
                for (int j = 0; j < 4; ++j) bn_[j] = ld_e2(j, qa[j] + t + 1);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int kc = ((qa[j] + t) * 4 + tig) ^ swz;
                double a[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = tr[i * 8 * S_N + kc];
#pragma unroll
                for (int i = 0; i < 4; ++i) dmma_8x8x4(acc[i][j], a[i], b[j]);
            }
        }
        // the groups' remaining steps (ranges of unequal length at the matrix edges)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            double bnx = lmin < len[j] ? ld_e2(j, qa[j] + lmin) : 0.0;
#pragma unroll 1
            for (int t = lmin; t < len[j]; ++t) {
                const double b = bnx;
                if (t + 1 < len[j]) bnx = ld_e2(j, qa[j] + t + 1);
                const int kc = ((qa[j] + t) * 4 + tig) ^ swz;
                double a[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = tr[i * 8 * S_N + kc];
#pragma unroll
                for (int i = 0; i < 4; ++i) dmma_8x8x4(acc[i][j], a[i], b);
            }
        }
    } else {
        // k4 steps on which the set of active column groups is constant run as one loop of a
        // mask-specialised body (E2 fragments of the active groups prefetched one step ahead)
        auto seg = [&](auto mc, int qa, int qb) {
            constexpr int M = decltype(mc)::value;
            double bn_[4];
    #pragma unroll
            for (int j = 0; j < 4; ++j) bn_[j] = ((M >> j) & 1) ? ld_e2(j, qa) : 0.0;
    #pragma unroll 2
            for (int q = qa; q < qb; ++q) {
                double b[4];
    #pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = bn_[j];
                if (q + 1 < qb) {
    #pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if ((M >> j) & 1) bn_[j] = ld_e2(j, q + 1);
                }
                const int kc = (q * 4 + tig) ^ swz;
                double a[4];
    #pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = tr[i * 8 * S_N + kc];
                dmma_masked<M, false>(acc, a, b);
            }
        };
        for (int q = kb / 4, q1 = ke / 4; q < q1;) {
            unsigned mask = 0;
            int qe = q1;
    #pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int lo = static_cast<int>(fine[j] & 0xffffu), hi = lo + static_cast<int>(fine[j] >> 16);
                if (q >= lo && q < hi) mask |= 1u << j;
                if (lo > q) qe = min(qe, lo);
                if (hi > q) qe = min(qe, hi);
            }
            switch (mask) {
                case 1: seg(std::integral_constant<int, 1>{}, q, qe); break;
                case 2: seg(std::integral_constant<int, 2>{}, q, qe); break;
                case 3: seg(std::integral_constant<int, 3>{}, q, qe); break;
                case 4: seg(std::integral_constant<int, 4>{}, q, qe); break;
                case 5: seg(std::integral_constant<int, 5>{}, q, qe); break;
                case 6: seg(std::integral_constant<int, 6>{}, q, qe); break;
                case 7: seg(std::integral_constant<int, 7>{}, q, qe); break;
                case 8: seg(std::integral_constant<int, 8>{}, q, qe); break;
                case 9: seg(std::integral_constant<int, 9>{}, q, qe); break;
                case 10: seg(std::integral_constant<int, 10>{}, q, qe); break;
                case 11: seg(std::integral_constant<int, 11>{}, q, qe); break;
                case 12: seg(std::integral_constant<int, 12>{}, q, qe); break;
                case 13: seg(std::integral_constant<int, 13>{}, q, qe); break;
                case 14: seg(std::integral_constant<int, 14>{}, q, qe); break;
                case 15: seg(std::integral_constant<int, 15>{}, q, qe); break;
                default: break;
            }
            q = qe;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;");

    if (g.flop_counter) {
        unsigned long long f = f1;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int flo = static_cast<int>(fine[j] & 0xffffu), fhi = flo + static_cast<int>(fine[j] >> 16);
            f += 2ull * 32 * 8 * 4 * max(0, min(ke / 4, fhi) - max(kb / 4, flo));
        }
        if (lane == 0) atomicAdd(g.flop_counter, f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double* row = Y + (i * 8 + gid) * S_N + warp * 32 + 2 * tig;
#pragma unroll
        for (int j = 0; j < 4; ++j) *reinterpret_cast<double2*>(row + j * 8) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

bool slab12_supported(int n1, int n2) { return n1 == S_N && n2 == S_N; }

int launch_slab12(const Slab12Args& g0, cudaStream_t s) {
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(k_slab12<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, S_SMEM);
        cudaFuncSetAttribute(k_slab12<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, S_SMEM);
        cudaFuncSetAttribute(k_slab12<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, S_SMEM);
        cudaFuncSetAttribute(k_slab12<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, S_SMEM);
        attr_done = true;
    }
    static const bool skew = [] {
        const char* v = std::getenv("PQ_SLAB12_SKEW");
        return v ? std::atoi(v) != 0 : true;  // skewed phase-2 loop by default (+2% config 2/4)
    }();
    const long long total = static_cast<long long>(g0.n0) * g0.Z1;
    int launches = 0;
    Slab12Args g = g0;
    for (long long z0 = 0; z0 < total; z0 += 65535) {
        g.z_off = z0;
        const long long zc = total - z0 < 65535 ? total - z0 : 65535;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(S_N / 32, static_cast<unsigned>(zc), 1);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = S_SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (g.E2p)
            skew ? cudaLaunchKernelEx(&cfg, k_slab12<true, true>, g) : cudaLaunchKernelEx(&cfg, k_slab12<false, true>, g);
        else
            skew ? cudaLaunchKernelEx(&cfg, k_slab12<true, false>, g) : cudaLaunchKernelEx(&cfg, k_slab12<false, false>, g);
        ++launches;
    }
    return launches;
}

}  // namespace pqb
