// linear_kernel instantiations, token tiles 16..64 (see gemm_kernel.cuh)
#include "gemm_gated.cuh"
namespace ms {
MS_LINEAR_INSTANTIATE(16) MS_LINEAR_INSTANTIATE(32) MS_LINEAR_INSTANTIATE(48) MS_LINEAR_INSTANTIATE(64)
MS_GATED_INSTANTIATE(16) MS_GATED_INSTANTIATE(32) MS_GATED_INSTANTIATE(48) MS_GATED_INSTANTIATE(64)
}  // namespace ms
