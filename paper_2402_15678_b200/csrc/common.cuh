// Shared helpers for the speculate-vote-verify kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <utility>

#include "../../include/minions.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_2402_15678_b200 kernels target sm_100a only"
#endif

namespace ms {

// Count of kernel launches issued through the C-ABI (read by bench.py as
// `gpu_launches`).  Defined in capi.cu.
void count_launch(int n = 1);

// Programmatic dependent launch (PDL): every kernel of this library is
// launched with programmatic stream serialization, waits on its predecessor
// with griddepcontrol.wait before touching data the predecessor may have
// written, and releases its dependents early with launch_dependents — so
// the next kernel's prologue (TMEM alloc, barrier init, descriptor fetch,
// weight-tile prefetch) overlaps this kernel's tail, in streams and in CUDA
// graphs alike.  MS_PDL=0 in the environment disables the attribute.
bool pdl_enabled();

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline int launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                  int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  ++n;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  if (cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...) != cudaSuccess) return -5;
  count_launch();
  return 0;
}

// Force-load a kernel (lazy module loading would otherwise load it at first
// launch, which can block behind a spin-waiting kernel of another stream —
// the tensor-parallel peer protocol relies on concurrent kernels).
template <typename F>
inline int preload_fn(F f) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f)) == cudaSuccess ? 0 : 1;
}

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MS_OK : MS_ERR_CUDA;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

// 16-byte vector of 8 bf16
struct alignas(16) bf16x8 {
  __nv_bfloat162 h[4];
};

__device__ __forceinline__ void unpack8(const bf16x8& v, float* f) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(v.h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ bf16x8 pack8(const float* f) {
  bf16x8 v;
#pragma unroll
  for (int i = 0; i < 4; ++i) v.h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

// Rotary position embedding, rotate-half pairing (dim i <-> i + D/2, the
// Llama convention): for i < D/2, with (c, s) = rope[pos][i],
//   y[i] = x[i] c - x[i + D/2] s,   y[i + D/2] = x[i + D/2] c + x[i] s.
// Rotates the 8 dims [dim0, dim0 + 8) of one head in place; `pf` holds the
// partner dims (dim0 +- D/2), `cs` the table row of the position (fp32).
__device__ __forceinline__ void rope8(float* f, const float* pf, const float2* __restrict__ cs, int dim0,
                                      int half) {
  const bool lo = dim0 < half;
  const int i0 = lo ? dim0 : dim0 - half;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 t = cs[i0 + j];
    f[j] = lo ? f[j] * t.x - pf[j] * t.y : f[j] * t.x + pf[j] * t.y;
  }
}

// silu(g) * u with the fast exponential and division (ex2.approx, rcp.approx:
// a few ulp of fp32, far below the bf16 rounding of the output); the gated
// GEMM epilogues run it once per output element — 70B verify forward 29.1 ->
// 28.8 ms at Q = 7 against expf / IEEE division (same-box A/B, round 2)
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

// KV-cache addressing.  Contiguous: caches [slots, Hkv, T, D].  Paged (table
// != null): a block pool [n_blocks, Hkv, bs, D] and a block table [slots,
// max_blocks] of pool indices, position t of a slot living in block
// table[slot][t / bs], row t % bs.  Returns the ROW index (times D = element).
struct KVPage {
  const int32_t* table;
  int max_blocks;
  int bs;
};

__device__ __forceinline__ int64_t kv_row(const KVPage& pg, int slot, int Hkv, int h, int T, int t) {
  if (!pg.table) return ((int64_t)slot * Hkv + h) * T + t;
  const int blk = pg.table[(int64_t)slot * pg.max_blocks + t / pg.bs];
  return ((int64_t)blk * Hkv + h) * pg.bs + (t % pg.bs);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value, index) argmax with first-index tie-break; NaN never wins.
__device__ __forceinline__ void argmax_merge(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__device__ __forceinline__ void warp_argmax(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmax_merge(v, i, v2, i2);
  }
}

}  // namespace ms
