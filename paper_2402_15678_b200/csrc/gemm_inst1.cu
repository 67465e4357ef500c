// linear_kernel instantiations, token tiles 80..128 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"
namespace ms {
MS_LINEAR_INSTANTIATE(80) MS_LINEAR_INSTANTIATE(96) MS_LINEAR_INSTANTIATE(112) MS_LINEAR_INSTANTIATE(128)
}  // namespace ms
