// linear_kernel instantiations, token tiles 208..256 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"
namespace ms {
MS_LINEAR_INSTANTIATE(208) MS_LINEAR_INSTANTIATE(224) MS_LINEAR_INSTANTIATE(240) MS_LINEAR_INSTANTIATE(256)
}  // namespace ms
