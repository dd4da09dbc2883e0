// Probe for tools/ozaki_experiment.cuh: the INT8-tensor-core (tcgen05 kind::i8) FP64 mode product against a
// plain FP64 kernel, on config-2 shapes (n = 128, d = 3, N = 2^21) for each mode, plus timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I tools \
//        tools/oz_probe.cu -o tools/oz_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>

#include "ozaki_experiment.cuh"

using namespace pqb::oz;

#define CK(x)                                                                                         \
    do {                                                                                              \
        cudaError_t e_ = (x);                                                                         \
        if (e_ != cudaSuccess) {                                                                      \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);          \
            exit(1);                                                                                  \
        }                                                                                             \
    } while (0)

// y[z][l][i][r] = sum_j E[z1][i][j] x[z][l][j][r], z1 = z / zdiv  (O x n x I layout per batch)
__global__ void k_ref(const double* E, long long sE, const double* x, double* y, int Z, int zdiv, long long sx1,
                      long long sx2, long long O, long long I) {
    const long long tot = static_cast<long long>(Z) * O * 128 * I;
    for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < tot; id += (long long)gridDim.x * blockDim.x) {
        const long long r = id % I, i = (id / I) % 128, o = (id / (I * 128)) % O, z = id / (I * 128 * O);
        const long long z1 = z / zdiv, z2 = z % zdiv;
        const double* Er = E + z1 * sE + i * 128;
        const double* xb = x + z1 * sx1 + z2 * sx2 + o * 128 * I + r;
        double s = 0.0;
        for (int j = 0; j < 128; ++j) s = fma(Er[j], xb[j * I], s);
        y[z * O * 128 * I + o * 128 * I + i * I + r] = s;
    }
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    const int n = 128;
    const long long N = 1LL << 21;
    const int ncol = 4;  // columns (batches) per product
    int dev;
    CK(cudaGetDevice(&dev));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // E: an advection-diffusion exponential-like banded matrix (entries decay off the diagonal)
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double> hE(static_cast<size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) hE[i * n + j] = std::exp(-0.15 * std::abs(i - j) * std::abs(i - j)) * (1.0 + 0.3 * nd(rng));
    std::vector<double> hx(static_cast<size_t>(ncol) * N);
    for (auto& v : hx) v = nd(rng);
    double *E, *x, *y, *yr;
    CK(cudaMalloc(&E, hE.size() * 8));
    CK(cudaMalloc(&x, hx.size() * 8));
    CK(cudaMalloc(&y, hx.size() * 8));
    CK(cudaMalloc(&yr, hx.size() * 8));
    CK(cudaMemcpy(E, hE.data(), hE.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
    int8_t* Ed;
    int* Ee;
    CK(cudaMalloc(&Ed, kABytes));
    CK(cudaMalloc(&Ee, n * 4));
    k_oz_split_rows<<<(n * 32 + 255) / 256, 256>>>(E, 0, 1, Ed, Ee);
    CK(cudaGetLastError());
    CK(cudaFuncSetAttribute(k_oz_mode, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int mode = 0; mode < 3; ++mode) {
        const long long O = mode == 0 ? 1 : (mode == 1 ? 128 : 128 * 128);
        const long long I = N / (O * 128);
        ModeArgs m;
        m.Ed = Ed;
        m.Ee = Ee;
        m.e_shared = 1;
        m.x = x;
        m.y = y;
        if (I > 1) {
            m.Z = ncol * static_cast<int>(O);
            m.zdiv = static_cast<int>(O);
            m.sx1 = N;
            m.sx2 = 128 * I;
            m.sy1 = N;
            m.sy2 = 128 * I;
            m.F = I;
            m.fstride = 1;
            m.jstride = I;
        } else {
            m.Z = ncol;
            m.zdiv = 1;
            m.sx1 = N;
            m.sy1 = N;
            m.F = O;
            m.fstride = 128;
            m.jstride = 1;
        }
        CK(cudaMemset(y, 0, hx.size() * 8));
        k_oz_mode<<<sms, kThreads, kSmemBytes>>>(m);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        k_ref<<<4 * sms, 256>>>(E, 0, x, yr, ncol, 1, N, 0, O, I);
        CK(cudaDeviceSynchronize());
        std::vector<double> hy(hx.size()), hr(hx.size());
        CK(cudaMemcpy(hy.data(), y, hy.size() * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hr.data(), yr, hr.size() * 8, cudaMemcpyDeviceToHost));
        double num = 0, den = 0, mx = 0;
        long long bad = 0;
        for (size_t q = 0; q < hy.size(); ++q) {
            const double d = hy[q] - hr[q];
            num += d * d;
            den += hr[q] * hr[q];
            mx = std::fmax(mx, std::fabs(d) / (std::fabs(hr[q]) + 1e-300));
            if (!(std::fabs(d) <= 1e-10 * (std::fabs(hr[q]) + 1.0))) ++bad;
        }
        float ms = 0;
        CK(cudaEventRecord(a));
        for (int r = 0; r < reps; ++r) k_oz_mode<<<sms, kThreads, kSmemBytes>>>(m);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        const double us = 1e3 * ms / reps;
        const double bytes = 2.0 * 8 * ncol * N, flops = 2.0 * 128 * ncol * N;
        double dus[8];
        for (int dbg = 1; dbg < 8; ++dbg) {
            ModeArgs md = m;
            md.dbg = dbg;
            CK(cudaEventRecord(a));
            for (int r = 0; r < reps; ++r) k_oz_mode<<<sms, kThreads, kSmemBytes>>>(md);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            dus[dbg] = 1e3 * ms / reps;
        }
        printf("dbg us (1 one-mma-per-order, 2 no-epi-math, 3, 4 no-x-loads, 5, 6, 7): %.1f %.1f %.1f %.1f %.1f %.1f %.1f\n", dus[1], dus[2], dus[3],
               dus[4], dus[5], dus[6], dus[7]);
        {
            unsigned long long* dp;
            CK(cudaMalloc(&dp, sms * 8 * 8));
            ModeArgs mp = m;
            mp.prof = dp;
            k_oz_mode<<<sms, kThreads, kSmemBytes>>>(mp);
            CK(cudaDeviceSynchronize());
            std::vector<unsigned long long> hp(sms * 8);
            CK(cudaMemcpy(hp.data(), dp, sms * 64, cudaMemcpyDeviceToHost));
            double avg[8] = {0};
            for (int q = 0; q < sms; ++q)
                for (int k = 0; k < 8; ++k) avg[k] += hp[q * 8 + k] / (double)sms;
            printf("clk per CTA: epi total %.0f wait_full %.0f store %.0f | prod total %.0f wait_empty %.0f | mma total %.0f wait_full %.0f wait_dempty %.0f\n",
                   avg[0], avg[1], avg[2], avg[3], avg[4], avg[5], avg[6], avg[7]);
            CK(cudaFree(dp));
        }
        printf("{\"mode\": %d, \"O\": %lld, \"I\": %lld, \"rel2\": %.3e, \"max_elem_rel\": %.3e, \"bad\": %lld, \"us\": %.2f, "
               "\"GBps\": %.0f, \"fp64_equiv_TFs\": %.2f, \"sample\": [%.17g, %.17g]}\n",
               mode, O, I, std::sqrt(num / den), mx, bad, us, bytes / us * 1e-3, flops / us * 1e-6, hy[12345], hr[12345]);
    }
    return 0;
}
