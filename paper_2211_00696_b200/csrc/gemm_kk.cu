// Instantiations of the DMMA GEMM with B k-contiguous (last mode: X E^T).
#include "gemm.cuh"

namespace pqb {
int launch_gemm_kk(const GemmArgs& g, bool vec2, int shape, cudaStream_t s) {
    return launch_gemm_family<true>(g, vec2, shape, s);
}
}  // namespace pqb
