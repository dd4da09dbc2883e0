#include <cstdio>
#include <cuda_runtime.h>
// sum of q streams -> 1 output; R = consecutive warp-chunks (512 B each) per stream visit
template <int R>
__global__ void __launch_bounds__(256) k_sum(long long NW, int q, const double2* __restrict__ V, long long vs, double2* out) {
    const long long warp_base = ((blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32) * 32 * R;
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * blockDim.x * R;
    for (long long b = warp_base; b < NW; b += stride) {
        double2 acc[R];
        for (int r = 0; r < R; ++r) acc[r] = make_double2(0, 0);
        int i = 0;
        for (; i + 4 <= q; i += 4) {
            double2 v[4][R];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int r = 0; r < R; ++r) v[u][r] = __ldg(V + (i + u) * vs + b + r * 32 + lane);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int r = 0; r < R; ++r) { acc[r].x += v[u][r].x; acc[r].y += v[u][r].y; }
        }
        for (; i < q; ++i)
#pragma unroll
            for (int r = 0; r < R; ++r) { double2 v = __ldg(V + i * vs + b + r * 32 + lane); acc[r].x += v.x; acc[r].y += v.y; }
#pragma unroll
        for (int r = 0; r < R; ++r) out[b + r * 32 + lane] = acc[r];
    }
}
int main() {
    const long long N = 128LL * 128 * 128, NW = N / 2;
    double2 *V, *out;
    cudaMalloc(&V, sizeof(double) * N * 26);
    cudaMalloc(&out, sizeof(double) * N);
    cudaMemset(V, 0, sizeof(double) * N * 26);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int q : {4, 8, 13, 25}) {
        for (int cap : {592, 1184, 2368, 4736, 8192}) {
            auto go = [&](auto R_) {
                constexpr int R = decltype(R_)::value;
                long long blocks = (NW / R + 255) / 256; if (blocks > cap) blocks = cap;
                k_sum<R><<<blocks, 256>>>(NW, q, V, NW, out);
                cudaEventRecord(e0);
                for (int it = 0; it < 20; ++it) k_sum<R><<<blocks, 256>>>(NW, q, V, NW, out);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
                printf("q=%2d cap=%5d R=%d: %7.1f us  %5.2f TB/s\n", q, cap, R, ms * 1e3, (q + 1) * N * 8.0 / (ms * 1e-3) / 1e12);
            };
            go(std::integral_constant<int, 1>());
            go(std::integral_constant<int, 4>());
        }
    }
}
