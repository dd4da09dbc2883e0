// tcgen05.mma kind::i8 issue rate on one SM: clocks per MMA for M = 128, K = 32 and several N,
// A from TMEM (ts) or shared memory (ss), B from shared memory.  Operands are zeros.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I tools tools/umma_rate.cu -o tools/umma_rate
#include <cstdio>
#include "ozaki_experiment.cuh"

using namespace pqb::oz;

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int N, bool TS>
__global__ void k_rate(unsigned long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    for (int q = threadIdx.x; q < 64 * 1024 / 4; q += blockDim.x) reinterpret_cast<uint32_t*>(sm)[q] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                                   (static_cast<uint32_t>(128 >> 4) << 24);
        const uint32_t s0 = smem_u32(sm);
        const uint32_t d = tb + 256;
        unsigned long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            if (TS) tc_mma_ts(d, tb + (r & 7) * 8, bdesc(s0 + (r & 3) * 256), idesc, r > 0);
            else mma_ss(d, bdesc(s0 + 32768 + (r & 3) * 256), bdesc(s0 + (r & 3) * 256), idesc, r > 0);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

// the chain kernel's pattern: A = 7 K-major planes of 16 KB, B = 7 MN-major planes of 8 KB (N = 64),
// 28 digit products x 4 k-steps per tile, random operand bytes
template <int NN>
__global__ void k_rate_chain(unsigned long long* out, int tiles, int bmn) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    uint32_t seed = 12345u + threadIdx.x * 7919u + blockIdx.x;
    for (int q = threadIdx.x; q < (112 + 64) * 1024 / 4; q += blockDim.x) {
        seed = seed * 1664525u + 1013904223u;
        reinterpret_cast<uint32_t*>(sm)[q] = seed;
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(bmn) << 16) |
                               (static_cast<uint32_t>(NN >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
        const uint32_t a0 = smem_u32(sm), b0 = a0 + 112 * 1024;
        constexpr int dstep = NN <= 64 ? NN : 0;  // accumulators overlap above N = 64 (timing only)
        unsigned long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            for (int c = 2; c <= 8; ++c) {
                bool first = true;
                for (int s = 1; s < c; ++s) {
                    const int u = c - s;
                    if (s > 7 || u > 7) continue;
                    for (int ks = 0; ks < 4; ++ks) {
                        auto dsc = [](uint32_t addr, uint32_t lbo, uint32_t sbo) {
                            return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>(lbo >> 4) << 16) |
                                   (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);
                        };
                        const uint64_t ad = dsc(a0 + (s - 1) * 16384 + ks * 256, 128, 1024);
                        const uint32_t bp = NN <= 64 ? (u - 1) * 8192 : ((u - 1) & 1) * NN * 128;  // B planes
                        const uint64_t bd = bmn ? dsc(b0 + bp + ks * 512, 128, 2048)
                                                : dsc(b0 + bp + ks * 256, 128, 1024);
                        mma_ss(tb + (c - 2) * dstep, ad, bd, idesc, first ? 0u : 1u);
                        first = false;
                    }
                }
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int N, bool TS>
void run(unsigned long long* d, int sms) {
    const int reps = 4096;
    cudaFuncSetAttribute(k_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    k_rate<N, TS><<<sms, 128, 65536>>>(d, reps);
    k_rate<N, TS><<<sms, 128, 65536>>>(d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[256];
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double clk = 0;
    for (int i = 0; i < sms; ++i) clk += h[i];
    clk /= sms * (double)reps;
    const double ops = 2.0 * 128 * N * 32;
    printf("{\"N\": %d, \"A\": \"%s\", \"clk_per_mma\": %.2f, \"int8_ops_per_clk_per_sm\": %.0f, \"POPS_at_1.965GHz_148SM\": %.2f, \"err\": \"%s\"}\n",
           N, TS ? "tmem" : "smem", clk, ops / clk, ops / clk * 148 * 1.965e9 / 1e15, cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 256 * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<16, true>(d, sms);
    run<32, true>(d, sms);
    run<64, true>(d, sms);
    run<128, true>(d, sms);
    run<256, true>(d, sms);
    run<32, false>(d, sms);
    run<64, false>(d, sms);
    run<128, false>(d, sms);
    run<256, false>(d, sms);
    auto chain_run = [&](auto kern, int nn) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024);
    for (int bmn = 0; bmn < 2; ++bmn) {
        const int tiles = 20;
        kern<<<sms, 128, 176 * 1024>>>(d, tiles, bmn);
        kern<<<sms, 128, 176 * 1024>>>(d, tiles, bmn);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[256];
        cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
        double clk = 0;
        for (int i = 0; i < sms; ++i) clk += h[i];
        clk /= sms * (double)tiles * 112;
        const double ops = 2.0 * 128 * nn * 32;
        printf("{\"chain_pattern\": true, \"N\": %d, \"B\": \"%s\", \"clk_per_mma\": %.2f, \"chip_POPS_at_1.965GHz\": %.2f, \"err\": \"%s\"}\n",
               nn, bmn ? "MN-major" : "K-major", clk, ops / clk * 148 * 1.965e9 / 1e15, cudaGetErrorString(e));
    }
    };
    chain_run(k_rate_chain<64>, 64);
    chain_run(k_rate_chain<128>, 128);
    chain_run(k_rate_chain<256>, 256);
    return 0;
}
