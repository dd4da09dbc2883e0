// Instantiations of the DMMA GEMM with B row-major (modes 0..d-2, expm products).
#include "gemm.cuh"

namespace pqb {
int launch_gemm_nk(const GemmArgs& g, bool vec2, int shape, cudaStream_t s) {
    return launch_gemm_family<false>(g, vec2, shape, s);
}

// Chained small products (row-major B, 16-byte aligned operands): 32x32x16 tiles, 4 warps.
int launch_gemm_chain(const GemmArgs* levels, int count, unsigned* bar, cudaStream_t s) {
    if (count <= 0 || count > kMaxChain) return 0;
    GemmChain ch;
    ch.levels = count;
    for (int i = 0; i < count; ++i) {
        const GemmArgs& g = levels[i];
        const bool vec2 = !g.b_kmajor && g.K % 2 == 0 && g.N % 2 == 0 && g.lda % 2 == 0 && g.ldb % 2 == 0 &&
                          g.sA1 % 2 == 0 && g.sA2 % 2 == 0 && g.sB1 % 2 == 0 && g.sB2 % 2 == 0 &&
                          (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(g.B) & 15) == 0;
        if (!vec2 || g.band || g.nterms || g.accumulate || g.Z > 65535) return 0;
        ch.g[i] = g;
    }
    return launch_chain_cfg<32, 32, 16, 16, 16, 3, 1>(ch, bar, s);
}
}  // namespace pqb
