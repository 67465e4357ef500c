// Glue kernels of one speculation round that keep the whole round on the
// device (and therefore capturable in one CUDA graph):
//
//  * draft_commit — after an SSM decode step's argmax: record the drafted token
//    into drafts[b, k, j] (the tokens list draft_sequence builds,
//    aggspec/oracles.py:146-152) and feed it to the SSM's next step.  Optional
//    fidelity injection (bench mode): with probability
//    f_k — decided by a counter-based hash of (seed, request key, k, absolute
//    position) — the drafted token is replaced by the target's greedy
//    continuation at that position, the device analogue of the reference's
//    PerturbedOracle fidelity knob (aggspec/oracles.py:108-132).  The SSM's
//    forward pass is always computed in full.
//  * pack_verify — the verifier's input rows [last context token | voted path],
//    i.e. the contexts ctx + tokens[:i] of aggspec/engine.py:294-296.
#include "common.cuh"

namespace ms {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void draft_commit_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ ctx_len,
                                    int B, int j, int k, int K, int S,
                                    const int32_t* __restrict__ teacher, int64_t ld_teacher,
                                    const int32_t* __restrict__ req_key, float f, uint64_t seed,
                                    int32_t* __restrict__ drafts, int32_t* __restrict__ next_tok) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int t = tok[b];
  if (teacher) {
    const int64_t p = (int64_t)ctx_len[b] + j;  // absolute position of this draft token
    const uint64_t key = (uint64_t)(uint32_t)req_key[b];
    const uint64_t h = splitmix64(seed ^ splitmix64((key << 40) ^ ((uint64_t)k << 32) ^ (uint64_t)p));
    const float u = (float)(h >> 40) * (1.0f / 16777216.0f);
    if (u < f && p < ld_teacher) {
      const int32_t tt = teacher[(int64_t)b * ld_teacher + p];
      if (tt >= 0) t = tt;
    }
  }
  drafts[((int64_t)b * K + k) * S + j] = t;
  if (next_tok) next_tok[b] = t;
}

// Grouped form (the K drafters batched as row groups, tok [G*B], group k =
// drafter k): drafts[b, k, j] = tok[k*B + b] (with drafter k's fidelity).
struct Fidelity8 {
  float f[8];
};

__global__ void draft_commit_grouped_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ ctx_len,
                                            int B, int j, int G, int S, const int32_t* __restrict__ teacher,
                                            int64_t ld_teacher, const int32_t* __restrict__ req_key,
                                            Fidelity8 fid, uint64_t seed, int32_t* __restrict__ drafts,
                                            int32_t* __restrict__ next_tok) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G * B) return;
  const int k = e / B, b = e - k * B;
  int t = tok[e];
  if (teacher) {
    const int64_t p = (int64_t)ctx_len[b] + j;
    const uint64_t key = (uint64_t)(uint32_t)req_key[b];
    const uint64_t h = splitmix64(seed ^ splitmix64((key << 40) ^ ((uint64_t)k << 32) ^ (uint64_t)p));
    const float u = (float)(h >> 40) * (1.0f / 16777216.0f);
    if (u < fid.f[k] && p < ld_teacher) {
      const int32_t tt = teacher[(int64_t)b * ld_teacher + p];
      if (tt >= 0) t = tt;
    }
  }
  drafts[((int64_t)b * G + k) * S + j] = t;
  if (next_tok) next_tok[e] = t;
}

__global__ void pack_verify_kernel(const int32_t* __restrict__ last, const int32_t* __restrict__ path,
                                   int B, int S, int32_t* __restrict__ vin) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B * (S + 1)) return;
  const int b = e / (S + 1), i = e - b * (S + 1);
  vin[e] = i == 0 ? last[b] : path[(int64_t)b * S + i - 1];
}

int preload_spec() {
  return preload_fn(draft_commit_kernel) + preload_fn(draft_commit_grouped_kernel) + preload_fn(pack_verify_kernel);
}

}  // namespace ms

extern "C" int ms_draft_commit(const int32_t* tok, const int32_t* ctx_len, int B, int j, int k,
                               int K, int S, const int32_t* teacher, int64_t ld_teacher,
                               const int32_t* req_key, float fidelity, uint64_t seed,
                               int32_t* drafts, int32_t* next_tok, void* stream) {
  if (B < 0 || j < 0 || j >= S || k < 0 || k >= K) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!tok || !drafts || (teacher && (!ctx_len || !req_key))) return MS_ERR_VALUE;
  return ms::launch(ms::draft_commit_kernel, dim3((B + 127) / 128), dim3(128), 0, (cudaStream_t)stream, 1,
                    tok, ctx_len, B, j, k, K, S, teacher, ld_teacher, req_key, fidelity, seed, drafts,
                    next_tok);
}

extern "C" int ms_pack_verify(const int32_t* last, const int32_t* path, int B, int S,
                              int32_t* vin, void* stream) {
  if (B < 0 || S < 1) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!last || !path || !vin) return MS_ERR_VALUE;
  const int n = B * (S + 1);
  return ms::launch(ms::pack_verify_kernel, dim3((n + 127) / 128), dim3(128), 0, (cudaStream_t)stream, 1,
                    last, path, B, S, vin);
}

extern "C" int ms_draft_commit_grouped(const int32_t* tok, const int32_t* ctx_len, int B, int j, int G, int S,
                                       const int32_t* teacher, int64_t ld_teacher, const int32_t* req_key,
                                       const float* fidelity, uint64_t seed, int32_t* drafts, int32_t* next_tok,
                                       void* stream) {
  if (B < 0 || G < 1 || G > 8 || S < 1 || j < 0 || j >= S) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!tok || !ctx_len || !drafts || (teacher && (!req_key || !fidelity))) return MS_ERR_VALUE;
  ms::Fidelity8 f;
  for (int k = 0; k < 8; ++k) f.f[k] = (fidelity && k < G) ? fidelity[k] : 0.f;
  const int n = G * B;
  return ms::launch(ms::draft_commit_grouped_kernel, dim3((n + 127) / 128), dim3(128), 0, (cudaStream_t)stream, 1,
                    tok, ctx_len, B, j, G, S, teacher, ld_teacher, req_key, f, seed, drafts, next_tok);
}
