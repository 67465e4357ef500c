// linear_kernel instantiations, token tiles 144..192 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"
namespace ms {
MS_LINEAR_INSTANTIATE(144) MS_LINEAR_INSTANTIATE(160) MS_LINEAR_INSTANTIATE(176) MS_LINEAR_INSTANTIATE(192)
}  // namespace ms
