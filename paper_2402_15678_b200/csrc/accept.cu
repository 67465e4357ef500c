// K8 (row argmax) + K9 (greedy accept + commit).
//
// Greedy verify is verify() (aggspec/verification.py:29-77) on point-mass draft
// and target distributions: position i is accepted iff the draft token equals
// the target argmax (q = 1 <= o = 1); the first mismatch is rejected with
// certainty (u >= 1 - 0/1 never holds) and the residual max(o - q, 0) is the
// target's point mass, so the emitted correction is the target argmax; full
// acceptance emits the bonus target argmax at position s.  The commit then
// truncates to the remaining budget and cuts after the first stop token
// (aggspec/engine.py:300-313).
#include "common.cuh"

namespace ms {

// ---------------------------------------------------------------------------
// Row argmax: max value, then the smallest index (np.argmax's first index).
// ---------------------------------------------------------------------------

constexpr int kArgmaxThreads = 256;

// ---------------------------------------------------------------------------
// Greedy accept: one warp per request, lanes sweep the s positions 32 at a time.
// ---------------------------------------------------------------------------
constexpr int kAcceptWarps = 4;

__global__ void __launch_bounds__(kAcceptWarps * 32)
accept_greedy_kernel(const int32_t* __restrict__ draft, const int32_t* __restrict__ tgt,
                     const int32_t* __restrict__ remaining, int stop_token, int B, int S,
                     int32_t* __restrict__ n_acc_out, int32_t* __restrict__ emitted,
                     int32_t* __restrict__ n_emit_out, int32_t* __restrict__ finished_out,
                     int32_t* __restrict__ kv_len) {
  pdl_wait();
  pdl_trigger();
  const int lane = lane_id();
  const int b = blockIdx.x * kAcceptWarps + (threadIdx.x >> 5);
  if (b >= B) return;
  const int32_t* d = draft + (int64_t)b * S;
  const int32_t* t = tgt + (int64_t)b * (S + 1);
  // accepted count = first mismatch (or S)
  int n_acc = S;
  for (int base = 0; base < S; base += 32) {
    const int i = base + lane;
    const bool mis = i < S && __ldg(d + i) != __ldg(t + i);
    const unsigned m = __ballot_sync(0xffffffffu, mis);
    if (m) {
      n_acc = base + __ffs(m) - 1;
      break;
    }
  }
  // emitted = target argmax[0..n_acc] (draft[:n_acc] equals it there)
  const int rem = remaining[b];
  int n_emit = min(n_acc + 1, max(rem, 0));
  bool stopped = false;
  if (stop_token >= 0) {
    for (int base = 0; base < n_emit; base += 32) {
      const int i = base + lane;
      const bool hit = i < n_emit && __ldg(t + i) == stop_token;
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (m) {
        n_emit = base + __ffs(m);  // inclusive of the stop token
        stopped = true;
        break;
      }
    }
  }
  int32_t* e = emitted + (int64_t)b * (S + 1);
  for (int i = lane; i <= S; i += 32) e[i] = i < n_emit ? __ldg(t + i) : -1;
  if (lane == 0) {
    const bool fin = stopped || (rem - n_emit) <= 0;
    n_acc_out[b] = n_acc;
    n_emit_out[b] = n_emit;
    finished_out[b] = fin ? 1 : 0;
    if (kv_len && !fin) kv_len[b] += n_acc + 1;
  }
}

// One CTA per row: the whole row is reduced in one block (vectorised loads,
// fixed first-index tie-break) — one launch, no scratch, no atomics.  (The
// earlier chunked atomicMax variant needed init + rows + finalize launches; in
// a drafter step those three tiny launches sat on the critical path.)
template <bool kBf16>
__global__ void __launch_bounds__(kArgmaxThreads)
argmax_row_kernel(const void* __restrict__ logits, int V, int64_t ld, int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x;
  float best = -INFINITY;
  int bidx = 0x7fffffff;
  if constexpr (kBf16) {
    const __nv_bfloat16* p = (const __nv_bfloat16*)logits + row * ld;
    int v0 = 0;
    if ((((uintptr_t)p) & 15) == 0) {
      const int nv = V / 8;
      for (int c = threadIdx.x; c < nv; c += kArgmaxThreads) {
        float f[8];
        unpack8(*reinterpret_cast<const bf16x8*>(p + c * 8), f);
#pragma unroll
        for (int j = 0; j < 8; ++j) argmax_merge(best, bidx, f[j], c * 8 + j);
      }
      v0 = nv * 8;
    }
    for (int t = v0 + threadIdx.x; t < V; t += kArgmaxThreads) argmax_merge(best, bidx, bf2f(p[t]), t);
  } else {
    const float* p = (const float*)logits + row * ld;
    int v0 = 0;
    if ((((uintptr_t)p) & 15) == 0) {
      const int nv = V / 4;
      for (int c = threadIdx.x; c < nv; c += kArgmaxThreads) {
        const float4 v = *reinterpret_cast<const float4*>(p + c * 4);
        argmax_merge(best, bidx, v.x, c * 4);
        argmax_merge(best, bidx, v.y, c * 4 + 1);
        argmax_merge(best, bidx, v.z, c * 4 + 2);
        argmax_merge(best, bidx, v.w, c * 4 + 3);
      }
      v0 = nv * 4;
    }
    for (int t = v0 + threadIdx.x; t < V; t += kArgmaxThreads) argmax_merge(best, bidx, p[t], t);
  }
  warp_argmax(best, bidx);
  __shared__ float sv[kArgmaxThreads / 32];
  __shared__ int si[kArgmaxThreads / 32];
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) {
    sv[w] = best;
    si[w] = bidx;
  }
  __syncthreads();
  if (w == 0) {
    best = lane_id() < kArgmaxThreads / 32 ? sv[lane_id()] : -INFINITY;
    bidx = lane_id() < kArgmaxThreads / 32 ? si[lane_id()] : 0x7fffffff;
    warp_argmax(best, bidx);
    if (lane_id() == 0) out[row] = bidx == 0x7fffffff ? 0 : bidx;  // all-NaN row -> 0
  }
}

static int launch_argmax(const void* logits, int is_bf16, int R, int V, int64_t ld,
                         unsigned long long* /*ws: unused*/, int32_t* out, cudaStream_t st) {
  return is_bf16 ? launch(argmax_row_kernel<true>, dim3(R), dim3(kArgmaxThreads), 0, st, 1, logits, V, ld, out)
                 : launch(argmax_row_kernel<false>, dim3(R), dim3(kArgmaxThreads), 0, st, 1, logits, V, ld, out);
}

int preload_accept() {
  return preload_fn(argmax_row_kernel<true>) + preload_fn(argmax_row_kernel<false>) +
         preload_fn(accept_greedy_kernel);
}

}  // namespace ms

extern "C" int ms_argmax_rows(const void* logits, int is_bf16, int R, int V, int64_t ld,
                              int32_t* out, void* ws, void* stream) {
  if (R < 0 || V < 1 || ld < V) return MS_ERR_VALUE;
  if (R == 0) return MS_OK;
  if (!logits || !out || !ws) return MS_ERR_VALUE;
  if (R > 65535) return MS_ERR_UNSUPPORTED;
  return ms::launch_argmax(logits, is_bf16, R, V, ld, (unsigned long long*)ws, out,
                           (cudaStream_t)stream);
}

extern "C" int ms_accept_greedy(const int32_t* draft, const int32_t* tgt_argmax,
                                const int32_t* remaining, int stop_token, int B, int S,
                                int32_t* n_acc, int32_t* emitted, int32_t* n_emit,
                                int32_t* finished, int32_t* kv_len, void* stream) {
  if (B < 0) return MS_ERR_VALUE;
  if (S < 1) return MS_ERR_VALUE;  // "draft must contain at least one token"
  if (S > 4096) return MS_ERR_UNSUPPORTED;
  if (B == 0) return MS_OK;
  if (!draft || !tgt_argmax || !remaining || !n_acc || !emitted || !n_emit || !finished)
    return MS_ERR_VALUE;
  const int blocks = (B + ms::kAcceptWarps - 1) / ms::kAcceptWarps;
  return ms::launch(ms::accept_greedy_kernel, dim3(blocks), dim3(ms::kAcceptWarps * 32), 0,
                    (cudaStream_t)stream, 1, draft, tgt_argmax, remaining, stop_token, B, S, n_acc,
                    emitted, n_emit, finished, kv_len);
}

extern "C" int ms_accept_greedy_logits(const int32_t* draft, const void* logits, int is_bf16,
                                       int V, const int32_t* remaining, int stop_token, int B,
                                       int S, int32_t* tgt_argmax_ws, void* argmax_ws,
                                       int32_t* n_acc, int32_t* emitted, int32_t* n_emit,
                                       int32_t* finished, int32_t* kv_len, void* stream) {
  if (B < 0 || V < 1) return MS_ERR_VALUE;
  if (S < 1) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  int st = ms_argmax_rows(logits, is_bf16, B * (S + 1), V, V, tgt_argmax_ws, argmax_ws, stream);
  if (st != MS_OK) return st;
  return ms_accept_greedy(draft, tgt_argmax_ws, remaining, stop_token, B, S, n_acc, emitted,
                          n_emit, finished, kv_len, stream);
}
