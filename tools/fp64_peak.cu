// FP64 roofline denominators for this pool's B200s (MEASURED_PEAKS.json has none):
//   (1) DMMA peak: mma.sync m8n8k4 f64 in a register-only loop, 8 independent chains/warp
//   (2) DFMA peak: plain fma.rn.f64 loop
//   (3) fp64 streaming copy (read+write bytes) for the HBM roofline
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void copy_f64(const double2* __restrict__ x, double2* __restrict__ y, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n2; i += st) y[i] = x[i];
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps, thr = 32 * wpb;
      dmma_loop<<<grid, thr>>>(out, 100); CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0); dmma_loop<<<grid, thr>>>(out, iters); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = 2.0 * 256 * 8 * (double)iters * grid * wpb;  // 8x8x4 = 256 FMA per warp-mma
      printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_block\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", wpb, bps, flops / best / 1e9);
    }
  }
  for (int wpb : {8, 16, 32}) {
    int grid = sms * 2, thr = 32 * wpb;
    dfma_loop<<<grid, thr>>>(out, 100); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0); dfma_loop<<<grid, thr>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * (double)iters * grid * thr;
    printf("{\"probe\":\"dfma\",\"threads\":%d,\"tflops\":%.3f}\n", thr, flops / best / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 2 GiB of doubles per buffer
  double *x, *y; CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8));
  cudaMemset(x, 0, n * 8);
  float best = 1e30f;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(e0); copy_f64<<<sms * 8, 512>>>((const double2*)x, (double2*)y, n / 2); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("{\"probe\":\"copy_f64\",\"gbs\":%.1f}\n", 2.0 * n * 8 / best / 1e6);
  return 0;
}
