// Tile-configuration sweep for the FP64 DMMA mode-product GEMM (gemm.cuh) on the exact shapes of
// the phi pipeline at n = 128 (config 2) and n = 256 / 512 (configs 3 / 5).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2211_00696_b200/csrc -I tools \
//          -o tools/gemm_tune tools/gemm_tune.cu
#include <cstdio>
#include <algorithm>
#include <vector>
#include <cmath>

#include "gemm.cuh"
#include "gemm_ws_experiment.cuh"
#include "gemm_tma_experiment.cuh"

using namespace pqb;

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__);              \
            return 1;                                                              \
        }                                                                          \
    } while (0)

struct Case {
    const char* name;
    GemmArgs g;
    double flops;
};

template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB = 1>
float run(const Case& c, int reps, cudaEvent_t e0, cudaEvent_t e1) {
    GemmArgs g = c.g;
    auto f = [&] {
        if (g.b_kmajor) launch_cfg<BM, BN, BK, WM, WN, ST, true, 2, MINB>(g, 0);
        else launch_cfg<BM, BN, BK, WM, WN, ST, false, 2, MINB>(g, 0);
    };
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        printf("  launch error %s\n", cudaGetErrorString(err));
        return -1;
    }
    return ms / reps;
}

template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB>
float run_ws(const Case& c, int reps, cudaEvent_t e0, cudaEvent_t e1) {
    GemmArgs g = c.g;
    if (!ws_ok<BM, BN, BK>(g)) return -1;
    auto f = [&] {
        if (g.b_kmajor) launch_ws<BM, BN, BK, WM, WN, ST, true, MINB>(g, 0);
        else launch_ws<BM, BN, BK, WM, WN, ST, false, MINB>(g, 0);
    };
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        printf("  launch error %s\n", cudaGetErrorString(err));
        return -1;
    }
    return ms / reps;
}

// TMA variant of the exponential-as-A band tile; checks its output against the cp.async tile first
template <int BM, int BN, int BK, int WM, int WN, int ST, int MINB>
float run_tma(const Case& c, int reps, cudaEvent_t e0, cudaEvent_t e1, double* Yref, long long count) {
    GemmArgs g = c.g;
    if (g.b_kmajor || (g.band_mode != 1 && g.band_mode != 2)) return -1;
    char why[128] = "";
    launch_cfg<32, 128, 16, 32, 32, 2, false, 2, 4>(g, 0);  // reference result
    cudaMemcpy(Yref, g.C, count * sizeof(double), cudaMemcpyDeviceToDevice);
    cudaMemset(g.C, 0, count * sizeof(double));
    if (launch_tma<BM, BN, BK, WM, WN, ST, MINB>(g, 0, why) < 0) {
        printf("  TMA maps rejected: %s\n", why);
        return -1;
    }
    cudaDeviceSynchronize();
    std::vector<double> a(count), b(count);
    cudaMemcpy(a.data(), Yref, count * sizeof(double), cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), g.C, count * sizeof(double), cudaMemcpyDeviceToHost);
    double diff = 0, mx = 0;
    for (long long i = 0; i < count; ++i) {
        diff = std::max(diff, std::abs(a[i] - b[i]));
        mx = std::max(mx, std::abs(a[i]));
    }
    printf("  TMA check: max|diff| %.3g (max|y| %.3g)%s\n", diff, mx, diff == 0 ? " bitwise equal" : "");
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch_tma<BM, BN, BK, WM, WN, ST, MINB>(g, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        printf("  launch error %s\n", cudaGetErrorString(err));
        return -1;
    }
    return ms / reps;
}

__global__ void fill_rand(double* p, long long n, unsigned seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long x = (i + 1) * 6364136223846793005ull + seed * 1442695040888963407ull;
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdull;
        x ^= x >> 33;
        p[i] = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 128;
    const int Z = argc > 2 ? atoi(argv[2]) : 12;  // nodes (or columns)
    const long long N = (long long)n * n * n;
    double *X, *Y, *E, *EXT;
    CK(cudaMalloc(&X, sizeof(double) * N * Z));
    CK(cudaMalloc(&Y, sizeof(double) * N * Z));
    CK(cudaMalloc(&EXT, sizeof(double) * N * Z));
    CK(cudaMalloc(&E, sizeof(double) * n * n * Z));
    cudaMemset(X, 0, sizeof(double) * N * Z);
    cudaMemset(E, 0, sizeof(double) * n * n * Z);
    if (argc > 5 && atoi(argv[5]) == 1) {  // random operands instead of zeros (data-dependent power)
        fill_rand<<<1024, 256>>>(X, N * Z, 1);
        fill_rand<<<1024, 256>>>(E, (long long)n * n * Z, 2);
        cudaDeviceSynchronize();
        printf("random operands\n");
    }
    cudaMemset(EXT, 0, sizeof(double) * N * Z);
    double* YREF;
    CK(cudaMalloc(&YREF, sizeof(double) * N * Z));
    double *coef, *alpha;
    int* nterms;
    CK(cudaMalloc(&coef, 64 * 64 * 8));
    CK(cudaMalloc(&alpha, 64 * 8));
    CK(cudaMalloc(&nterms, 64 * 4));
    std::vector<int> hn(64);
    for (int i = 0; i < 64; ++i) hn[i] = 1 + i % 4;
    cudaMemcpy(nterms, hn.data(), 64 * 4, cudaMemcpyHostToDevice);
    cudaMemset(coef, 0, 64 * 64 * 8);
    cudaMemset(alpha, 0, 64 * 8);
    const double fl = 2.0 * N * n * Z;
    // optional negligible-block band: each 32-row block rb needs slices [4rb - w, 4rb + 4 + w)
    const int bw = argc > 4 ? atoi(argv[4]) : -1;
    int2* band = nullptr;
    double band_frac = 1.0;
    if (bw >= 0) {
        const int RB = (n + 31) / 32, NS = (n + 7) / 8;
        std::vector<int2> hb(RB * Z);
        long long kept = 0;
        for (int z = 0; z < Z; ++z)
            for (int rb = 0; rb < RB; ++rb) {
                const int lo = std::max(0, 4 * rb - bw), hi = std::min(NS, 4 * rb + 4 + bw);
                hb[z * RB + rb] = make_int2(lo, hi);
                kept += hi - lo;
            }
        band_frac = (double)kept / (RB * NS * Z);
        CK(cudaMalloc(&band, sizeof(int2) * hb.size()));
        cudaMemcpy(band, hb.data(), sizeof(int2) * hb.size(), cudaMemcpyHostToDevice);
        printf("band half-width %d slices: %.2f of the K work kept\n", bw, band_frac);
    }
    std::vector<Case> cases;
    {  // mode 0, stacked nodes: (Z n x n) . (n x n^2)
        GemmArgs g;
        g.A = E; g.lda = n; g.B = X; g.ldb = (long long)n * n; g.C = Y; g.ldc = (long long)n * n;
        g.M = Z * n; g.N = n * n; g.K = n; g.Z = 1;
        if (band) { g.band = band; g.band_mode = 1; g.band_rows = n; g.band_stride = (n + 31) / 32; }
        cases.push_back({"mode0", g, fl * band_frac});
    }
    {  // mode 1: batch (Z * n) of (n x n) . (n x n)
        GemmArgs g;
        g.A = E; g.lda = n; g.B = X; g.ldb = n; g.C = Y; g.ldc = n;
        g.M = n; g.N = n; g.K = n; g.Z = Z * n; g.zdiv = n;
        g.sA1 = (long long)n * n; g.sB1 = N; g.sB2 = (long long)n * n; g.sC1 = N; g.sC2 = (long long)n * n;
        if (band) { g.band = band; g.band_mode = 2; g.band_rows = n; g.band_stride = (n + 31) / 32; }
        cases.push_back({"mode1", g, fl * band_frac});
    }
    {  // mode 2 (last): X (n^2 x n) . E^T, batch Z
        GemmArgs g;
        g.A = X; g.lda = n; g.B = E; g.b_kmajor = 1; g.ldb = n; g.C = Y; g.ldc = n;
        g.M = n * n; g.N = n; g.K = n; g.Z = Z;
        g.sA1 = N; g.sB1 = (long long)n * n; g.sC1 = N;
        if (band) { g.band = band; g.band_mode = 3; g.band_rows = n; g.band_stride = (n + 31) / 32; }
        cases.push_back({"mode2", g, fl * band_frac});
    }
    {  // mode 2 + squaring epilogue (p = 4 groups: 1..4 extra addends)
        GemmArgs g = cases.back().g;
        g.sB1 = 0;
        g.band = nullptr;
        g.alpha_z = alpha; g.ext = EXT; g.ext_s = N; g.ext_group = 4; g.coef = coef; g.cld = 4; g.nterms = nterms;
        cases.push_back({"mode2+sq", g, fl});
    }
    {  // batched square products of the expm (Z matrices of n x n), as in expm_core
        const int cnt = argc > 3 ? atoi(argv[3]) : 81;
        GemmArgs g;
        g.A = E; g.B = X; g.C = Y; g.M = g.N = g.K = n; g.lda = g.ldb = g.ldc = n; g.Z = cnt;
        g.sA1 = 0; g.sB1 = g.sC1 = (long long)n * n;
        cases.push_back({"expm-sq", g, 2.0 * n * n * n * (double)cnt});
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (const Case& c : cases) {
        printf("%-9s n=%d Z=%d  GFLOP=%.2f\n", c.name, n, Z, c.flops / 1e9);
#define T(BM, BN, BK, WM, WN, ST, MINB)                                                                \
    {                                                                                                  \
        float ms = run<BM, BN, BK, WM, WN, ST, MINB>(c, 5, e0, e1);                                    \
        if (ms > 0)                                                                                    \
            printf("  %3dx%3dx%2d w%2dx%2d st%d minb%d : %8.1f us  %6.2f TF/s\n", BM, BN, BK, WM, WN, ST, MINB, \
                   ms * 1e3, c.flops / (ms * 1e-3) / 1e12);                                            \
    }
#define TW(BM, BN, BK, WM, WN, ST, MINB)                                                               \
    {                                                                                                  \
        float ms = run_ws<BM, BN, BK, WM, WN, ST, MINB>(c, 5, e0, e1);                                 \
        if (ms > 0)                                                                                    \
            printf("  WS %3dx%3dx%2d w%2dx%2d st%d minb%d : %8.1f us  %6.2f TF/s\n", BM, BN, BK, WM, WN, ST, MINB, \
                   ms * 1e3, c.flops / (ms * 1e-3) / 1e12);                                            \
    }
        T(32, 128, 16, 32, 32, 2, 4)
        T(32, 96, 16, 32, 32, 2, 5)
        T(32, 96, 16, 32, 32, 2, 6)
        T(32, 160, 16, 32, 32, 2, 3)
        T(32, 160, 16, 32, 32, 2, 4)
        T(32, 128, 16, 32, 32, 2, 5)
        T(32, 128, 8, 32, 32, 2, 6)
        T(32, 128, 8, 32, 32, 2, 7)
        T(32, 128, 8, 32, 32, 3, 6)
        T(32, 128, 16, 32, 32, 3, 3)
        T(32, 128, 16, 32, 32, 3, 4)
        T(32, 256, 16, 32, 32, 2, 2)
        T(32, 256, 16, 32, 64, 2, 2)
        T(32, 128, 16, 32, 64, 2, 4)
        T(32, 128, 16, 32, 16, 2, 3)
        T(32, 128, 16, 32, 16, 2, 2)
        T(32, 128, 16, 32, 16, 3, 2)
        T(32, 128, 8, 32, 16, 3, 3)
        T(32, 128, 16, 16, 32, 2, 3)
#define TT(BM, BN, BK, WM, WN, ST, MINB)                                                               \
    {                                                                                                  \
        float ms = run_tma<BM, BN, BK, WM, WN, ST, MINB>(c, 5, e0, e1, YREF, N * Z);                   \
        if (ms > 0)                                                                                    \
            printf("  TMA %3dx%3dx%2d w%2dx%2d st%d minb%d : %8.1f us  %6.2f TF/s\n", BM, BN, BK, WM, WN, ST, MINB, \
                   ms * 1e3, c.flops / (ms * 1e-3) / 1e12);                                            \
    }
        TT(32, 128, 16, 32, 32, 2, 4)
        TT(32, 128, 16, 32, 32, 3, 3)
        TT(32, 128, 16, 32, 32, 3, 4)
        TT(32, 128, 16, 32, 32, 4, 3)
        TT(32, 128, 16, 32, 32, 2, 5)
        TT(32, 128, 8, 32, 32, 3, 7)
        TT(32, 128, 8, 32, 32, 4, 5)
        TT(32, 128, 8, 32, 32, 2, 8)
        TT(32, 128, 8, 32, 32, 3, 6)
        TW(32, 128, 16, 32, 32, 2, 3)
        TW(32, 128, 16, 32, 32, 3, 3)
        TW(32, 128, 16, 32, 32, 2, 4)
        TW(32, 128, 8, 32, 32, 4, 3)
        T(64, 32, 16, 32, 16, 2, 6)
        T(64, 32, 16, 32, 16, 2, 7)
        T(64, 32, 16, 32, 16, 2, 8)
        T(64, 32, 16, 32, 16, 3, 5)
        T(64, 32, 16, 32, 16, 3, 6)
        T(64, 32, 16, 16, 16, 2, 4)
        T(64, 32, 16, 16, 16, 2, 3)
        T(64, 32, 16, 32, 8, 2, 4)
        TW(64, 32, 16, 32, 16, 2, 4)
        TW(64, 32, 16, 32, 16, 3, 4)
        TW(64, 32, 16, 32, 16, 4, 4)
        TW(64, 32, 8, 32, 16, 4, 5)
    }
    return 0;
}
