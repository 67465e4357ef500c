// Probe (not product code): how fast can a grid of CTAs stream a weight
// matrix with the TMA structure ms_linear uses — one producer thread, a ring
// of S stages of [box_rows x 64] bf16 tiles (128B swizzle, mbarrier
// complete_tx), a consumer thread that releases each stage as soon as it
// lands (no MMA)?  Variants: stages, box rows, CTAs per SM (via smem),
// row-major [N, K] walk (tile = 128 rows at one k-block).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_probe tools/tma_stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t@!p bra W_%=;\n\t}" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(pol)
      : "memory");
}

struct P {
  int n_tiles, kb, S, box_rows, cta_per_tile_split;
};

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, P p, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int S = p.S, BYTES = p.box_rows * 128;
  uint64_t* full = (uint64_t*)(sm + S * BYTES);
  uint64_t* empty = full + 16;
  const int split = blockIdx.x % p.cta_per_tile_split, tile = blockIdx.x / p.cta_per_tile_split;
  const int kb0 = split * p.kb / p.cta_per_tile_split, kb1 = (split + 1) * p.kb / p.cta_per_tile_split;
  const int nk = kb1 - kb0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x == 0) {
    for (int i = 0; i < nk; ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      mbar_expect(&full[s], BYTES);
      // the tile's box_rows weight rows at k-block kb0 + i
      tma2d(sm + s * BYTES, &tm, &full[s], (kb0 + i) * 64, tile * p.box_rows, pol);
    }
  } else if (threadIdx.x == 32) {
    int acc = 0;
    for (int i = 0; i < nk; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      acc += sm[s * BYTES + (i & 127)];
      mbar_arrive(&empty[s]);
    }
    if (acc == 123456789) sink[0] = acc;
  }
}

int main() {
  cudaFree(0);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const long N = 57344, K = 8192;  // the 70B gate/up weight
  void* w;
  cudaMalloc(&w, N * K * 2);
  cudaMemset(w, 1, N * K * 2);
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct V {
    int box_rows, S, ctas_per_sm_target, splits;
  };
  std::vector<V> vs;
  for (int box : {128, 64, 256})
    for (int S : {2, 4, 6, 8, 12})
      for (int occ : {1, 2, 3})
        for (int sp : {1, 2}) vs.push_back({box, S, occ, sp});
  for (auto v : vs) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)v.box_rows};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("{\"error\": \"tmap\"}\n");
      continue;
    }
    P p;
    p.box_rows = v.box_rows;
    p.n_tiles = (int)(N / v.box_rows);
    p.kb = (int)(K / 64);
    p.S = v.S;
    p.cta_per_tile_split = v.splits;
    // occupancy target via shared memory: the ring, padded up to 228KB / occ
    int ring = v.S * v.box_rows * 128 + 1024 + 512;
    int smem = ring;
    int target = (227 * 1024) / v.ctas_per_sm_target - 2048;
    if (smem < target) smem = target;
    if (ring > 227 * 1024) continue;
    if (smem > 227 * 1024) smem = 227 * 1024;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = p.n_tiles * v.splits;
    for (int rep = 0; rep < 2; ++rep) stream_kernel<<<grid, 64, smem>>>(tm, p, sink);
    cudaEventRecord(e0);
    const int R = 5;
    for (int rep = 0; rep < R; ++rep) stream_kernel<<<grid, 64, smem>>>(tm, p, sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stream_kernel, 64, smem);
    printf("{\"box_rows\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"splits\": %d, \"grid\": %d, \"us\": %.1f, \"TBs\": %.3f, \"err\": \"%s\"}\n",
           v.box_rows, v.S, occ, v.splits, grid, ms * 1e3 / R, (double)N * K * 2 / (ms * 1e-3 / R) / 1e12,
           cudaGetErrorString(err));
  }
  return 0;
}
