// linear_kernel instantiations, token tiles 16..64 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"
namespace ms {
MS_LINEAR_INSTANTIATE(16) MS_LINEAR_INSTANTIATE(32) MS_LINEAR_INSTANTIATE(48) MS_LINEAR_INSTANTIATE(64)
}  // namespace ms
