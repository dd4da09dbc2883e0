// FP64 CUDA-core throughput probe (DFMA and separate DMUL+DADD), 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <bool FMA>
__global__ void k(double* out, double a, double b, int iters) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = FMA ? fma(x[i], a, b) : __dadd_rn(__dmul_rn(x[i], a), b);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.0) out[0] = s;
}
int main() {
    double* o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int fma = 0; fma < 2; ++fma) {
        for (int bps : {4, 8}) {
            const int blocks = 148 * bps, thr = 256;
            auto go = [&] { fma ? k<true><<<blocks, thr>>>(o, 0.999, 1e-3, iters) : k<false><<<blocks, thr>>>(o, 0.999, 1e-3, iters); };
            go();
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            go();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)blocks * thr * iters * 8 * (fma ? 1 : 2);  // instructions (lane ops)
            printf("%s blocks/SM=%d: %.3f ms  %.2f T lane-instr/s  (%.1f TFLOP/s)\n", fma ? "DFMA     " : "DMUL+DADD", bps, ms,
                   ops / (ms * 1e-3) / 1e12, (double)blocks * thr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
        }
    }
}
