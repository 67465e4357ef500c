// Tensor-parallel collectives of the LLM verify forward over peer memory
// (NVLink / NVSwitch): the Megatron split of the verifier —
// column-parallel QKV / gate-up, row-parallel O / down projections followed by
// a sum over ranks, vocab-parallel LM head followed by a cross-rank argmax.
//
// Instead of an NCCL allreduce (whose algorithm — and so summation order —
// NCCL picks by message size), the sum is two fixed-order kernels over
// symmetric buffers that every rank maps (CUDA IPC):
//
//   GEMM          rank r writes its fp32 partial P_r [R, d] (rank 0 adds the
//                 residual in the GEMM epilogue)                (ms_linear)
//   signal        publish epoch e to every rank's flag slot r     (ms_tp_signal)
//   reduce-gather rank r waits for all flags >= e, sums column slice r of
//                 P_0 .. P_{t-1} in rank order (fp32, one bf16 rounding) and
//                 stores it into EVERY rank's residual stream x (two-shot:
//                 reads (t-1)/t of R*d*4 B, writes (t-1)/t of R*d*2 B per rank)
//                                                             (ms_tp_reduce_gather)
//   signal        second flag set
//   RMSNorm       waits for the second flags, then normalises x   (ms_rmsnorm_wait)
//
// PDL: a wait kernel releases its dependents (the next GEMM, which prefetches
// its weights before griddepcontrol.wait) at its start only when `early` is
// set — ranks on distinct GPUs, where this overlaps the weight stream with the
// collective.  Ranks sharing one GPU (the single-GPU protocol test) release
// after the wait: an early-launched GEMM would hold the shared GPU's shared
// memory while this rank spins on a peer that needs it (deadlock).
//
// The result is bitwise identical on every rank and does not depend on R
// (a row's sum never depends on other rows), so the TP forward keeps the
// batch invariance the lossless speculative engine relies on.  Buffer reuse
// is safe with one buffer per flag set: a rank overwrites P_r only after its
// RMSNorm waited for every rank's second flag, i.e. after every rank finished
// reading P_r.  Epochs are device counters (CUDA-graph replays keep counting).
// Waits are bounded: after 20 s of wall time a kernel sets *err and gives up (no hang).
#include "common.cuh"

namespace ms {

constexpr unsigned long long kWaitLimitNs = 20ull * 1000 * 1000 * 1000;  // 20 s

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// wait until flags[0..t) >= the local epoch counter (one polling thread per
// CTA, exponential __nanosleep backoff so pollers do not starve the kernels
// they wait for), then CTA barrier.  Bounded by wall time: *err = 1, proceed.
__device__ __forceinline__ void wait_flags(const int* flags, const int* epoch, int t, int* err) {
  if (threadIdx.x == 0) {
    const int e = *reinterpret_cast<const volatile int*>(epoch);
    unsigned long long t0 = 0;
    for (int j = 0; j < t; ++j) {
      unsigned ns = 32;
      while (ld_acquire_sys(flags + j) < e) {
        __nanosleep(ns);
        if (ns < 2048) ns <<= 1;
        const unsigned long long now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        if (now - t0 > kWaitLimitNs) {
          atomicExch(err, 1);
          break;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void tp_signal_kernel(int* const* __restrict__ peer_flags, int rank, int t, int* epoch) {
  pdl_wait();
  pdl_trigger();
  // the previous kernels' global writes (this rank's partials / x slices) are
  // complete at this kernel's start; make them visible system-wide first
  __threadfence_system();
  const int e = *epoch + 1;
  *epoch = e;
  for (int j = 0; j < t; ++j) st_release_sys(peer_flags[j] + rank, e);
}

// grid (row blocks, column slice chunks); rank `rank` owns columns
// [rank * d / t, (rank + 1) * d / t)
__global__ void __launch_bounds__(256)
tp_reduce_gather_kernel(const float* const* __restrict__ parts, int64_t ldp,
                        __nv_bfloat16* const* __restrict__ xs, int64_t ldx, const int* flags,
                        const int* epoch, int rank, int t, int R, int d, int* err, int early) {
  pdl_wait();
  if (early) pdl_trigger();
  wait_flags(flags, epoch, t, err);
  if (!early) pdl_trigger();
  const int cols = d / t;
  const int c0 = rank * cols;
  const int n4 = cols / 4;  // float4 column groups of the slice
  const int rows_per = (R + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows_per, r1 = min(R, r0 + rows_per);
  for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < (r1 - r0) * n4; e += blockDim.x * gridDim.y) {
    const int r = r0 + e / n4;
    const int c = c0 + (e % n4) * 4;
    float4 acc = __ldcv(reinterpret_cast<const float4*>(parts[0] + (int64_t)r * ldp + c));
    for (int j = 1; j < t; ++j) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(parts[j] + (int64_t)r * ldp + c));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    for (int j = 0; j < t; ++j) *reinterpret_cast<uint2*>(xs[j] + (int64_t)r * ldx + c) = pk;
  }
}

// Fused variant: the row-parallel GEMM's epilogue already pushed every
// rank's fp32 partial of THIS rank's column slice into local receive slots
// recv[j][row][0..slice) (ms_linear_tp_scatter, peer stores overlapped with
// the GEMM's other tiles); after the flags, the sum is local reads only, and
// the bf16 slice is stored into every rank's residual stream (all-gather).
__global__ void __launch_bounds__(256)
tp_reduce_recv_kernel(const float* __restrict__ recv, int rows_cap, int slice,
                      __nv_bfloat16* const* __restrict__ xs, int64_t ldx, const int* flags, const int* epoch,
                      int rank, int t, int R, int* err, int early) {
  pdl_wait();
  if (early) pdl_trigger();
  wait_flags(flags, epoch, t, err);
  if (!early) pdl_trigger();
  const int n4 = slice / 4;
  const int rows_per = (R + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows_per, r1 = min(R, r0 + rows_per);
  const int64_t src_stride = (int64_t)rows_cap * slice;
  for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < (r1 - r0) * n4; e += blockDim.x * gridDim.y) {
    const int r = r0 + e / n4;
    const int c = (e % n4) * 4;
    float4 acc = __ldcg(reinterpret_cast<const float4*>(recv + (int64_t)r * slice + c));
    for (int j = 1; j < t; ++j) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(recv + j * src_stride + (int64_t)r * slice + c));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    const int col = rank * slice + c;
    for (int j = 0; j < t; ++j) *reinterpret_cast<uint2*>(xs[j] + (int64_t)r * ldx + col) = pk;
  }
}

// RMSNorm with a leading wait on the second flag set (rows of x complete on
// every rank), one CTA of 128 threads per row, fp32 statistics.
__global__ void __launch_bounds__(128)
rmsnorm_wait_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, const __nv_bfloat16* __restrict__ g,
                    float eps, int d, __nv_bfloat16* __restrict__ out, int64_t ldo, const int* flags,
                    const int* epoch, int t, int* err, int early) {
  pdl_wait();
  if (early) pdl_trigger();
  wait_flags(flags, epoch, t, err);
  if (!early) pdl_trigger();
  const int r = blockIdx.x;
  const __nv_bfloat16* xr = x + (int64_t)r * ldx;
  float q = 0.f;
  for (int i = threadIdx.x * 8; i < d; i += 128 * 8) {
    float f[8];
    unpack8(*reinterpret_cast<const bf16x8*>(xr + i), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) q += f[j] * f[j];
  }
  __shared__ float red[4];
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  const float rstd = rsqrtf((red[0] + red[1] + red[2] + red[3]) / (float)d + eps);
  for (int i = threadIdx.x * 8; i < d; i += 128 * 8) {
    float f[8], gg[8];
    unpack8(*reinterpret_cast<const bf16x8*>(xr + i), f);
    unpack8(*reinterpret_cast<const bf16x8*>(g + i), gg);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * rstd * gg[j];
    *reinterpret_cast<bf16x8*>(out + (int64_t)r * ldo + i) = pack8(f);
  }
}

// local (value, global index) argmax of each logits row of this rank's vocab
// slice, packed into one u64 whose unsigned max is the first-index argmax:
// high word = order-preserving float key, low word = ~index.
__device__ __forceinline__ uint32_t f2key(float v) {
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(256)
tp_argmax_local_kernel(const float* __restrict__ logits, int64_t ld, int Vr, int v0,
                       unsigned long long* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const float* row = logits + (int64_t)r * ld;
  unsigned long long best = 0ull;
  for (int i = threadIdx.x; i < Vr; i += blockDim.x) {
    const float v = row[i];
    if (v != v) continue;  // NaN never wins
    const unsigned long long k = ((unsigned long long)f2key(v) << 32) | (uint32_t)(~(uint32_t)(v0 + i));
    best = k > best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k = __shfl_xor_sync(0xffffffffu, best, o);
    best = k > best ? k : best;
  }
  __shared__ unsigned long long red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = red[w] > best ? red[w] : best;
    best = red[0] > best ? red[0] : best;
    out[r] = best;
  }
}

__global__ void tp_argmax_combine_kernel(const unsigned long long* const* __restrict__ peer, int t, int R,
                                         const int* flags, const int* epoch, int32_t* __restrict__ out,
                                         int* err, int early) {
  pdl_wait();
  if (early) pdl_trigger();
  wait_flags(flags, epoch, t, err);
  if (!early) pdl_trigger();
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    unsigned long long best = 0ull;
    for (int j = 0; j < t; ++j) {
      const unsigned long long k = __ldcv(peer[j] + r);
      best = k > best ? k : best;
    }
    out[r] = (int32_t)(~(uint32_t)(best & 0xffffffffull));
  }
}

int preload_tp() {
  return preload_fn(tp_signal_kernel) + preload_fn(tp_reduce_gather_kernel) + preload_fn(tp_reduce_recv_kernel) +
         preload_fn(rmsnorm_wait_kernel) +
         preload_fn(tp_argmax_local_kernel) + preload_fn(tp_argmax_combine_kernel);
}

}  // namespace ms

extern "C" int ms_ipc_alloc(int64_t bytes, void** ptr, void* handle) {
  if (bytes <= 0 || !ptr || !handle) return MS_ERR_VALUE;
  void* p = nullptr;
  if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) return MS_ERR_CUDA;
  if (cudaMemset(p, 0, (size_t)bytes) != cudaSuccess) return MS_ERR_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
    cudaFree(p);
    return MS_ERR_CUDA;
  }
  memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return MS_OK;
}

extern "C" int ms_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

extern "C" int ms_ipc_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return MS_ERR_VALUE;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return MS_ERR_CUDA;
  return MS_OK;
}

extern "C" int ms_ipc_close(void* ptr) {
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? MS_OK : MS_ERR_CUDA;
}

extern "C" int ms_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? MS_OK : MS_ERR_CUDA; }

extern "C" int ms_tp_signal(int* const* peer_flags, int rank, int t, int* epoch, void* stream) {
  if (!peer_flags || !epoch || t < 1 || rank < 0 || rank >= t) return MS_ERR_VALUE;
  return ms::launch(ms::tp_signal_kernel, dim3(1), dim3(1), 0, (cudaStream_t)stream, 1, peer_flags, rank, t,
                    epoch);
}

extern "C" int ms_tp_reduce_gather(const float* const* parts, int64_t ldp, void* const* xs_v,
                                   int64_t ldx, const int* flags, const int* epoch, int rank, int t, int R,
                                   int d, int* err, int early, void* stream) {
  auto* const* xs = reinterpret_cast<__nv_bfloat16* const*>(xs_v);
  if (!parts || !xs || !flags || !epoch || !err || t < 1 || rank < 0 || rank >= t || R < 0) return MS_ERR_VALUE;
  if (d % (4 * t) || ldp % 4 || ldx % 4) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  const int cols4 = d / t / 4;
  const int gy = (cols4 + 255) / 256;
  const int gx = R < 32 ? R : 32;
  return ms::launch(ms::tp_reduce_gather_kernel, dim3(gx, gy), dim3(256), 0, (cudaStream_t)stream, 1, parts,
                    ldp, xs, ldx, flags, epoch, rank, t, R, d, err, early);
}

extern "C" int ms_rmsnorm_wait(const void* x, int64_t ldx, const void* gamma, float eps, int R, int d, void* out,
                               int64_t ldo, const int* flags, const int* epoch, int t, int* err, int early,
                               void* stream) {
  if (!x || !gamma || !out || !flags || !epoch || !err || R < 0 || t < 1) return MS_ERR_VALUE;
  if (d % 8 || ldx % 8 || ldo % 8) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  return ms::launch(ms::rmsnorm_wait_kernel, dim3(R), dim3(128), 0, (cudaStream_t)stream, 1,
                    (const __nv_bfloat16*)x, ldx, (const __nv_bfloat16*)gamma, eps, d, (__nv_bfloat16*)out, ldo,
                    flags, epoch, t, err, early);
}

extern "C" int ms_tp_argmax_local(const float* logits, int64_t ld, int R, int Vr, int v0, uint64_t* out,
                                  void* stream) {
  if (!logits || !out || R < 0 || Vr < 1 || ld < Vr) return MS_ERR_VALUE;
  if (R == 0) return MS_OK;
  return ms::launch(ms::tp_argmax_local_kernel, dim3(R), dim3(256), 0, (cudaStream_t)stream, 1, logits, ld, Vr, v0,
                    (unsigned long long*)out);
}

extern "C" int ms_tp_argmax_combine(const uint64_t* const* peer, int t, int R, const int* flags, const int* epoch,
                                    int32_t* out, int* err, int early, void* stream) {
  if (!peer || !flags || !epoch || !out || !err || t < 1 || R < 0) return MS_ERR_VALUE;
  if (R == 0) return MS_OK;
  return ms::launch(ms::tp_argmax_combine_kernel, dim3(1), dim3(256), 0, (cudaStream_t)stream, 1,
                    (const unsigned long long* const*)peer, t, R, flags, epoch, out, err, early);
}

extern "C" int ms_tp_reduce_recv_gather(const float* recv, int rows_cap, int slice, void* const* xs_v, int64_t ldx,
                                        const int* flags, const int* epoch, int rank, int t, int R, int* err,
                                        int early, void* stream) {
  auto* const* xs = reinterpret_cast<__nv_bfloat16* const*>(xs_v);
  if (!recv || !xs || !flags || !epoch || !err || t < 1 || rank < 0 || rank >= t || R < 0 || rows_cap < R)
    return MS_ERR_VALUE;
  if (slice % 4 || ldx % 4) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  const int gy = (slice / 4 + 255) / 256;
  const int gx = R < 32 ? R : 32;
  return ms::launch(ms::tp_reduce_recv_kernel, dim3(gx, gy), dim3(256), 0, (cudaStream_t)stream, 1, recv, rows_cap,
                    slice, xs, ldx, flags, epoch, rank, t, R, err, early);
}
