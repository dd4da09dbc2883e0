// Instantiations of the DMMA GEMM with B row-major (modes 0..d-2, expm products).
#include "gemm.cuh"

namespace pqb {
int launch_gemm_nk(const GemmArgs& g, bool vec2, int shape, cudaStream_t s) {
    return launch_gemm_family<false>(g, vec2, shape, s);
}
}  // namespace pqb
