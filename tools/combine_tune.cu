// Sweep of the streaming node-combination kernel (kernels.cu k_node_combine) on the config-2
// shapes: N = 128^3, p = 4, 13-node (level 1, MODE 1) and 25-node (level 2, MODE 2) passes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2211_00696_b200/csrc \
//          -o tools/combine_tune tools/combine_tune.cu
#include "kernels.cu"

// kernels.cu's GEMM dispatcher references the instantiation units; the sweep never calls it
namespace pqb {
int launch_gemm_nk(const GemmArgs&, bool, int, cudaStream_t) { return 0; }
int launch_gemm_kk(const GemmArgs&, bool, int, cudaStream_t) { return 0; }
}  // namespace pqb

#include <vector>

using namespace pqb;

template <int W, int MODE, int U, int MINB>
float run(long long N, int q, const double* V, const int* sl, const double* cf, const double* cc, const double* prev,
          double* acc, double* stats, int reps, unsigned grid_cap, long long vstride = 0) {
    if (!vstride) vstride = N;
    const long long NW = N / W;
    long long b = (NW + 255) / 256;
    if (b > grid_cap) b = grid_cap;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto f = [&] {
        k_node_combine<4, W, MODE, U, MINB><<<(unsigned)b, 256>>>(NW, q, V, vstride / W, sl, cf, cc, prev, acc, N / W, 1, stats);
    };
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

int main() {
    const long long N = 128LL * 128 * 128;
    const int Q = 25;
    double *V, *acc, *prev, *cf, *cc, *stats;
    int* sl;
    cudaMalloc(&V, sizeof(double) * (N + 8192) * Q);
    cudaMalloc(&acc, sizeof(double) * N * 4);
    cudaMalloc(&prev, sizeof(double) * N * 4);
    cudaMalloc(&cf, sizeof(double) * Q * 4);
    cudaMalloc(&cc, sizeof(double) * Q * 4);
    cudaMalloc(&stats, sizeof(double) * 8);
    cudaMalloc(&sl, sizeof(int) * Q);
    std::vector<int> h(Q);
    for (int i = 0; i < Q; ++i) h[i] = i;
    cudaMemcpy(sl, h.data(), sizeof(int) * Q, cudaMemcpyHostToDevice);
    cudaMemset(V, 0, sizeof(double) * (N + 8192) * Q);
    cudaMemset(prev, 0, sizeof(double) * N * 4);
    cudaMemset(cf, 0, sizeof(double) * Q * 4);
    cudaMemset(cc, 0, sizeof(double) * Q * 4);
    const double mb1 = (13 + 4) * N * 8.0, mb2 = (25 + 8) * N * 8.0;
#define S(W, U, MINB, PAD)                                                                                         \
    {                                                                                                              \
        float a = run<W, 1, U, MINB>(N, 13, V, sl, cf, cc, nullptr, acc, stats, 20, 4736, N + PAD);                \
        float b = run<W, 2, U, MINB>(N, 25, V, sl, cf, nullptr, prev, acc, stats, 20, 4736, N + PAD);              \
        printf("W%d U%d minb%d pad%5d : L1 %7.1f us %5.2f TB/s   L2 %7.1f us %5.2f TB/s\n", W, U, MINB, PAD, a * 1e3, \
               mb1 / (a * 1e-3) / 1e12, b * 1e3, mb2 / (b * 1e-3) / 1e12);                                          \
    }
    {  // the production dispatcher (node_combine): cp.async ring for 16-byte-aligned inputs
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto timeit = [&](auto&& f) {
            f();
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            for (int r = 0; r < 20; ++r) f();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            return ms / 20;
        };
        float a = timeit([&] { node_combine(N, 4, 13, V, N, sl, cf, cc, nullptr, acc, N, 1, stats, 1, 0); });
        float b = timeit([&] { node_combine(N, 4, 25, V, N, sl, cf, nullptr, prev, acc, N, 1, stats, 2, 0); });
        float c = timeit([&] { node_combine(N, 4, 25, V, N, sl, cf, nullptr, nullptr, acc, N, 1, nullptr, 0, 0); });
        printf("dispatcher ring      : L1 %7.1f us %5.2f TB/s   L2 %7.1f us %5.2f TB/s   M0 %7.1f us %5.2f TB/s (%s)\n",
               a * 1e3, mb1 / (a * 1e-3) / 1e12, b * 1e3, mb2 / (b * 1e-3) / 1e12, c * 1e3,
               (29 * N * 8.0) / (c * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    S(2, 4, 3, 0)
    S(2, 4, 3, 32)
    S(2, 4, 3, 256)
    S(2, 4, 3, 512)
    S(2, 4, 3, 1024)
    S(2, 4, 3, 4096)
    S(2, 8, 2, 512)
    S(2, 4, 4, 512)
#define T(W, U, MINB, CAP)                                                                                        \
    {                                                                                                             \
        float a = run<W, 1, U, MINB>(N, 13, V, sl, cf, cc, nullptr, acc, stats, 20, CAP);                         \
        float b = run<W, 2, U, MINB>(N, 25, V, sl, cf, nullptr, prev, acc, stats, 20, CAP);                       \
        float c0 = run<W, 0, U, MINB>(N, 25, V, sl, cf, nullptr, nullptr, acc, stats, 20, CAP);                    \
        printf("W%d U%d minb%d cap%6d : L1 %7.1f us %5.2f TB/s   L2 %7.1f us %5.2f TB/s   M0 %7.1f us %5.2f TB/s (%s)\n", \
               W, U, MINB, CAP, a * 1e3, mb1 / (a * 1e-3) / 1e12, b * 1e3, mb2 / (b * 1e-3) / 1e12, c0 * 1e3,          \
               (29 * N * 8.0) / (c0 * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));                           \
    }
    T(2, 4, 1, 4736)
    T(2, 4, 3, 4736)
    T(2, 4, 4, 4736)
    T(2, 8, 1, 4736)
    T(2, 8, 3, 4736)
    T(2, 2, 4, 4736)
    T(1, 4, 4, 4736)
    T(1, 8, 4, 4736)
    T(1, 8, 6, 4736)
    T(2, 4, 3, 1184)
    T(2, 4, 3, 592)
    T(2, 8, 2, 592)
    T(2, 1, 4, 4736)
    return 0;
}
