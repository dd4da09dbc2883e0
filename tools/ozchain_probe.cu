// Probe for tools/ozchain.cuh: y = (E0 (x) E1 (x) E2) x, n = 128, d = 3, 4 columns, on the int8
// tensor cores with the operand carried in digit form, against a plain FP64 chain; timings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I tools tools/ozchain_probe.cu -o tools/ozchain_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "ozchain.cuh"

using namespace ozc;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

// plain FP64 mode product on [ncol][O][128][I]
__global__ void k_ref(const double* E, const double* x, double* y, int ncol, long long O, long long I) {
    const long long tot = static_cast<long long>(ncol) * O * 128 * I;
    for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < tot; id += (long long)gridDim.x * blockDim.x) {
        const long long r = id % I, i = (id / I) % 128, o = id / (I * 128);
        const double* Er = E + i * 128;
        const double* xb = x + o * 128 * I + r;
        double s = 0.0;
        for (int j = 0; j < 128; ++j) s = fma(Er[j], xb[j * I], s);
        y[id] = s;
    }
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    const int ncol = 4;
    const long long N = 128LL * 128 * 128;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::mt19937_64 rng(11);
    std::normal_distribution<double> nd;
    std::vector<double> hE(3 * 128 * 128);
    const double wid[3] = {0.05, 0.2, 0.6};
    for (int m = 0; m < 3; ++m)
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j)
                hE[(m * 128 + i) * 128 + j] = std::exp(-wid[m] * (i - j) * (i - j)) * (1.0 + 0.2 * nd(rng)) + (i == j ? 0.1 : 0.0);
    std::vector<double> hx(ncol * N);
    for (auto& v : hx) v = nd(rng);
    double *E, *x, *y, *ya, *yb;
    CK(cudaMalloc(&E, hE.size() * 8));
    CK(cudaMalloc(&x, hx.size() * 8));
    CK(cudaMalloc(&y, hx.size() * 8));
    CK(cudaMalloc(&ya, hx.size() * 8));
    CK(cudaMalloc(&yb, hx.size() * 8));
    CK(cudaMemcpy(E, hE.data(), hE.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
    int8_t *Ed, *T0, *T1, *T2;
    int *Ee, *gE, *ex;
    CK(cudaMalloc(&Ed, 3 * kABytes));
    CK(cudaMalloc(&Ee, 3 * 128 * 4));
    CK(cudaMalloc(&gE, 3 * 4));
    CK(cudaMalloc(&ex, 3 * ncol * 4));
    const size_t tiles = static_cast<size_t>(ncol) * 256 * kTileBytes;
    CK(cudaMalloc(&T0, tiles));
    CK(cudaMalloc(&T1, tiles));
    CK(cudaMalloc(&T2, tiles));
    std::vector<int> init(3 * ncol, -1022);
    CK(cudaMemcpy(gE, init.data(), 12, cudaMemcpyHostToDevice));
    for (int m = 0; m < 3; ++m) k_split_E<<<16, 256>>>(E + m * 128 * 128, Ed + m * kABytes, Ee + m * 128, gE + m);
    CK(cudaFuncSetAttribute(k_chain_mode, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    CK(cudaDeviceSynchronize());
    auto chain = [&](bool timed_parts, float* part_ms) {
        cudaEvent_t ev[6];
        if (timed_parts)
            for (auto& e : ev) CK(cudaEventCreate(&e));
        if (timed_parts) CK(cudaEventRecord(ev[0]));
        CK(cudaMemcpyAsync(ex, init.data(), ncol * 4, cudaMemcpyHostToDevice));
        k_colmax<<<dim3(2 * sms, ncol), 256>>>(x, N, ex);
        k_split_x<<<ncol * 256, 256>>>(x, ex, T0);
        if (timed_parts) CK(cudaEventRecord(ev[1]));
        for (int m = 0; m < 3; ++m) {
            ChainArgs a;
            a.mode = m;
            a.ncol = ncol;
            a.Ed = Ed + m * kABytes;
            a.Ee = Ee + m * 128;
            a.gE = gE + m;
            a.Bin = m == 0 ? T0 : (m == 1 ? T1 : T2);
            a.ein = ex + m * ncol;
            a.Bout = m == 0 ? T1 : (m == 1 ? T2 : nullptr);
            a.eout = m < 2 ? ex + (m + 1) * ncol : nullptr;
            a.y = y;
            k_chain_mode<<<sms, kThreads, kSmemBytes>>>(a);
            if (timed_parts) CK(cudaEventRecord(ev[2 + m]));
        }
        if (timed_parts) {
            CK(cudaEventSynchronize(ev[4]));
            for (int k = 0; k < 4; ++k) CK(cudaEventElapsedTime(&part_ms[k], ev[k], ev[k + 1]));
        }
    };
    float pm[4];
    chain(true, pm);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    // reference chain
    k_ref<<<4 * sms, 256>>>(E, x, ya, ncol, 1, 16384);
    k_ref<<<4 * sms, 256>>>(E + 16384, ya, yb, ncol, 128, 128);
    k_ref<<<4 * sms, 256>>>(E + 2 * 16384, yb, ya, ncol, 16384, 1);
    CK(cudaDeviceSynchronize());
    std::vector<double> hy(hx.size()), hr(hx.size());
    CK(cudaMemcpy(hy.data(), y, hy.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), ya, hr.size() * 8, cudaMemcpyDeviceToHost));
    for (int c = 0; c < ncol; ++c) {
        double num = 0, den = 0;
        for (long long q = 0; q < N; ++q) {
            const double d = hy[c * N + q] - hr[c * N + q];
            num += d * d;
            den += hr[c * N + q] * hr[c * N + q];
        }
        printf("col %d rel2 %.3e  sample %.17g %.17g\n", c, std::sqrt(num / den), hy[c * N + 4321], hr[c * N + 4321]);
    }
    float best[4] = {1e9f, 1e9f, 1e9f, 1e9f};
    for (int r = 0; r < reps; ++r) {
        chain(true, pm);
        for (int k = 0; k < 4; ++k) best[k] = std::fmin(best[k], pm[k]);
    }
    printf("{\"split_us\": %.1f, \"mode0_us\": %.1f, \"mode1_us\": %.1f, \"mode2_us\": %.1f, \"chain_us\": %.1f, \"ncol\": %d}\n",
           1e3 * best[0], 1e3 * best[1], 1e3 * best[2], 1e3 * best[3], 1e3 * (best[0] + best[1] + best[2] + best[3]), ncol);
    // per-role clocks and the no-epilogue floor, per mode
    {
        unsigned long long* dp;
        CK(cudaMalloc(&dp, sms * 6 * 8));
        for (int m = 0; m < 3; ++m) {
            for (int dbg = 0; dbg < 2; ++dbg) {
                ChainArgs a;
                a.mode = m;
                a.ncol = ncol;
                a.Ed = Ed + m * kABytes;
                a.Ee = Ee + m * 128;
                a.gE = gE + m;
                a.Bin = m == 0 ? T0 : (m == 1 ? T1 : T2);
                a.ein = ex + m * ncol;
                a.Bout = m == 0 ? T1 : (m == 1 ? T2 : nullptr);
                a.eout = m < 2 ? ex + (m + 1) * ncol : nullptr;
                a.y = y;
                a.dbg = dbg;
                a.prof = dp;
                cudaEvent_t e0, e1;
                CK(cudaEventCreate(&e0));
                CK(cudaEventCreate(&e1));
                CK(cudaEventRecord(e0));
                k_chain_mode<<<sms, kThreads, kSmemBytes>>>(a);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                std::vector<unsigned long long> hp(sms * 6);
                CK(cudaMemcpy(hp.data(), dp, sms * 48, cudaMemcpyDeviceToHost));
                double avg[6] = {0};
                for (int q = 0; q < sms; ++q)
                    for (int k = 0; k < 6; ++k) avg[k] += hp[q * 6 + k] / (double)sms;
                printf("mode %d dbg %d: %.1f us | epi %.0f (wait %.0f) | mma %.0f (wait full %.0f, wait acc %.0f) | tma wait %.0f clk\n",
                       m, dbg, 1e3 * ms, avg[0], avg[1], avg[2], avg[3], avg[4], avg[5]);
            }
        }
    }
    // fp64 reference chain time for scale
    cudaEvent_t a0, a1;
    CK(cudaEventCreate(&a0));
    CK(cudaEventCreate(&a1));
    CK(cudaEventRecord(a0));
    k_ref<<<4 * sms, 256>>>(E, x, ya, ncol, 1, 16384);
    CK(cudaEventRecord(a1));
    CK(cudaEventSynchronize(a1));
    float ms;
    CK(cudaEventElapsedTime(&ms, a0, a1));
    printf("naive fp64 mode-0 product: %.1f us\n", 1e3 * ms);
    return 0;
}
