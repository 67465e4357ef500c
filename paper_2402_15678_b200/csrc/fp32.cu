// fp32 verification mode — the model forward with fp32 activations, fp32 KV
// cache and fp32 accumulation everywhere (weights are the same bf16 tensors,
// exactly representable in fp32).
//
// north_star asks for "accepted token sequences and vote results bit-exact in
// the fp32 verification mode": the reference engine (aggspec/engine.py:
// 252-330) driven by fp32 CPU model oracles (ModelOracle.next_dist,
// aggspec/oracles.py:19-26; oracle/opt_ref.py / llama_ref.py with exact=True)
// must produce the same token streams, drafts, votes, accept counts, weights
// and speculation lengths as SpecEngine(precision="fp32").  The bf16 path
// rounds activations to bf16 between kernels (its own contract); here nothing
// is rounded below fp32, so the device and the CPU oracle differ only by fp32
// summation order (~1e-6 relative), far below the argmax margins.
//
// These kernels are plain SIMT fp32 (FFMA): this mode exists for parity, not
// speed — tensor-core fp32 emulation would buy nothing the tests need.  Every
// output depends only on its own row (fixed k order, fixed key order), so the
// mode keeps the bf16 path's batch invariance (speculative == greedy).
#include "common.cuh"

namespace ms {

// ---------------------------------------------------------------------------
// embed: x[r] = tok_emb[tok[r]] (+ pos_emb[start[r / Q] + r % Q + pos_offset])
// ---------------------------------------------------------------------------
__global__ void embed_f32_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ start, int Q,
                                 const __nv_bfloat16* __restrict__ te, const __nv_bfloat16* __restrict__ pe,
                                 int pos_offset, int d, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int pos = start[r / Q] + r % Q;
  const __nv_bfloat16* a = te + (int64_t)tok[r] * d;
  const __nv_bfloat16* b = pe ? pe + (int64_t)(pos + pos_offset) * d : nullptr;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float v = bf2f(a[i]);
    if (b) v = __fadd_rn(v, bf2f(b[i]));
    out[(int64_t)r * d + i] = v;
  }
}

// ---------------------------------------------------------------------------
// LayerNorm (two-pass: mean, then mean of squared deviations — the oracle's
// formula) or RMSNorm, fp32 in / out.  One CTA of 128 threads per row.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float block_sum128(float v, float* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  return (red[0] + red[1]) + (red[2] + red[3]);
}

template <bool RMS>
__global__ void __launch_bounds__(128)
norm_f32_kernel(const float* __restrict__ x, int64_t ldx, const int32_t* __restrict__ rows,
                const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, float eps, int d,
                float* __restrict__ out, int64_t ldo) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[4];
  const int r = blockIdx.x;
  const float* xr = x + (int64_t)(rows ? rows[r] : r) * ldx;
  float* orow = out + (int64_t)r * ldo;
  float mean = 0.f;
  if (!RMS) {
    float s = 0.f;
    for (int i = threadIdx.x; i < d; i += 128) s += xr[i];
    mean = block_sum128(s, red) / (float)d;
  }
  float s2 = 0.f;
  for (int i = threadIdx.x; i < d; i += 128) {
    const float t = xr[i] - mean;
    s2 = fmaf(t, t, s2);
  }
  const float rstd = __frcp_rn(__fsqrt_rn(block_sum128(s2, red) / (float)d + eps));
  for (int i = threadIdx.x; i < d; i += 128) {
    const float y = __fmul_rn(__fmul_rn(xr[i] - mean, rstd), bf2f(g[i]));
    orow[i] = RMS ? y : __fadd_rn(y, bf2f(b[i]));
  }
}

// ---------------------------------------------------------------------------
// linear: out[m, n] = act(sum_k x[m, k] w[n, k] + bias[n]) (+ residual[m, n])
// x fp32 [M, ldx], w bf16 [N, K] (nn.Linear layout), out fp32.  64 x 64
// output tile per 256-thread CTA, 4 x 4 per thread, k tiles of 32 staged in
// shared memory; each output sums k in ascending order (fp32 FMA).
// GATED: w is the Llama 64-row interleaved gate/up weight; output column j
// uses gate row (j/64)*128 + j%64 and up row +64; out = silu(g) * u.
// ---------------------------------------------------------------------------
constexpr int F32_BM = 64, F32_BN = 64, F32_BK = 32;

template <bool GATED>
__global__ void __launch_bounds__(256)
linear_f32_kernel(const float* __restrict__ x, int64_t ldx, const __nv_bfloat16* __restrict__ w,
                  const __nv_bfloat16* __restrict__ bias, const float* residual, int64_t ldr, float* out,
                  int64_t ldo, int M, int N, int K, int act) {
  pdl_wait();
  pdl_trigger();
  constexpr int NW = GATED ? 2 : 1;
  __shared__ float xs[F32_BK][F32_BM + 4];
  __shared__ float ws[NW][F32_BK][F32_BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * F32_BM, n0 = blockIdx.x * F32_BN;  // n0: output column
  float acc[NW][4][4];
#pragma unroll
  for (int q = 0; q < NW; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[q][i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += F32_BK) {
    // stage x tile [64 rows x 32 k] transposed and w tile(s) [64 cols x 32 k]
    for (int e = tid; e < F32_BM * F32_BK; e += 256) {
      const int r = e / F32_BK, kk = e % F32_BK;
      const int m = m0 + r, k = k0 + kk;
      xs[kk][r] = (m < M && k < K) ? x[(int64_t)m * ldx + k] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      for (int e = tid; e < F32_BN * F32_BK; e += 256) {
        const int c = e / F32_BK, kk = e % F32_BK;
        const int n = n0 + c, k = k0 + kk;
        int64_t row = n;
        if (GATED) row = (int64_t)(n / 64) * 128 + n % 64 + 64 * q;
        ws[q][kk][c] = (n < N && k < K) ? bf2f(w[row * K + k]) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < F32_BK; ++kk) {
      float a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = xs[kk][ty + 16 * i];
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        float bb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bb[j] = ws[q][kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[q][i][j] = fmaf(a[i], bb[j], acc[q][i][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v;
      if (GATED) {
        const float gt = acc[0][i][j], up = acc[1][i][j];
        v = __fmul_rn(__fdiv_rn(gt, __fadd_rn(1.0f, expf(-gt))), up);
      } else {
        v = acc[0][i][j];
        if (bias) v = __fadd_rn(v, bf2f(bias[n]));
        if (act == 1) v = fmaxf(v, 0.f);
      }
      if (residual) v = __fadd_rn(v, residual[(int64_t)m * ldr + n]);
      out[(int64_t)m * ldo + n] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// KV append (fp32 cache [slots, Hkv, T, D]): rows r = b*Q + i of qkv
// [B*Q, ldq] ([q: H*D | k: Hkv*D | v: Hkv*D]) at position start[b] + i of
// slot[b]; K rotated (rotate-half RoPE, fp32 table [pos, D/2, (cos, sin)])
// when rope != NULL.  One CTA per (row, KV head), D threads.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float rope_elem(const float* v, int dd, int D, const float2* cs) {
  const int half = D / 2;
  if (dd < half) {
    const float2 t = cs[dd];
    return __fsub_rn(__fmul_rn(v[dd], t.x), __fmul_rn(v[dd + half], t.y));
  }
  const float2 t = cs[dd - half];
  return __fadd_rn(__fmul_rn(v[dd], t.x), __fmul_rn(v[dd - half], t.y));
}

__global__ void kv_append_f32_kernel(const float* __restrict__ qkv, int64_t ldq, int Q, int H, int Hkv, int D,
                                     const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                                     float* __restrict__ kc, float* __restrict__ vc,
                                     const float2* __restrict__ rope) {
  pdl_wait();
  const int r = blockIdx.x, hk = blockIdx.y, dd = threadIdx.x;
  const int b = r / Q, pos = start[b] + r % Q;
  if (pos < 0 || pos >= T) return;
  const float* kr = qkv + (int64_t)r * ldq + (int64_t)(H + hk) * D;
  const float* vr = qkv + (int64_t)r * ldq + (int64_t)(H + Hkv + hk) * D;
  const int64_t o = (((int64_t)slot[b] * Hkv + hk) * T + pos) * D + dd;
  kc[o] = rope ? rope_elem(kr, dd, D, rope + (int64_t)pos * (D / 2)) : kr[dd];
  vc[o] = vr[dd];
}

// ---------------------------------------------------------------------------
// Causal attention over the cache: one warp per (request, query head, query
// row); query row i of request b sits at position p = start[b] + i and sees
// keys 0..p.  Keys are walked in chunks of 32 (lane j scores key c+j), with an
// online softmax across chunks; lane l owns output dims l, l+32, ... (D <= 128).
// OPT_SCALE_Q: the query is scaled before the dot product (opt_ref: q *
// scale, then q k^T); otherwise the score is scaled (llama_ref).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
attention_f32_kernel(const float* __restrict__ qkv, int64_t ldq, int Q, int H, int Hkv, int D,
                     const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                     const float* __restrict__ kc, const float* __restrict__ vc, const float2* __restrict__ rope,
                     float scale, int scale_q, float* __restrict__ out, int64_t ldo, int n_items) {
  pdl_wait();
  pdl_trigger();
  __shared__ float qs[4][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * 4 + warp;  // (b, h, i) flattened, i fastest
  if (item >= n_items) return;
  const int i = item % Q, h = (item / Q) % H, b = item / (Q * H);
  const int r = b * Q + i;
  const int pos = start[b] + i;
  const int hk = h / (H / Hkv);
  const float* qr = qkv + (int64_t)r * ldq + (int64_t)h * D;
  for (int dd = lane; dd < D; dd += 32) {
    float v = rope ? rope_elem(qr, dd, D, rope + (int64_t)pos * (D / 2)) : qr[dd];
    qs[warp][dd] = scale_q ? __fmul_rn(v, scale) : v;
  }
  __syncwarp();
  const float* kb = kc + ((int64_t)slot[b] * Hkv + hk) * T * D;
  const float* vb = vc + ((int64_t)slot[b] * Hkv + hk) * T * D;
  float m = -INFINITY, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int nk = min(pos + 1, T);
  for (int c = 0; c < nk; c += 32) {
    const int j = c + lane;
    float sc = -INFINITY;
    if (j < nk) {
      const float* kr = kb + (int64_t)j * D;
      float s = 0.f;
      for (int dd = 0; dd < D; ++dd) s = fmaf(qs[warp][dd], kr[dd], s);
      sc = scale_q ? s : __fmul_rn(s, scale);
    }
    const float cm = warp_max(sc);
    const float mn = fmaxf(m, cm);
    const float alpha = expf(m - mn);  // m = -inf on the first chunk -> 0
    const float p = (j < nk) ? expf(sc - mn) : 0.f;
    l = l * alpha + warp_sum(p);
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[t] *= alpha;
    const int cn = min(32, nk - c);
    for (int jj = 0; jj < cn; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj);
      const float* vr = vb + (int64_t)(c + jj) * D;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int dd = lane + 32 * t;
        if (dd < D) acc[t] = fmaf(pj, vr[dd], acc[t]);
      }
    }
    m = mn;
  }
  float* orow = out + (int64_t)r * ldo + (int64_t)h * D;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int dd = lane + 32 * t;
    if (dd < D) orow[dd] = __fdiv_rn(acc[t], l);
  }
}

int preload_fp32() {
  return preload_fn(embed_f32_kernel) + preload_fn(norm_f32_kernel<true>) + preload_fn(norm_f32_kernel<false>) +
         preload_fn(linear_f32_kernel<true>) + preload_fn(linear_f32_kernel<false>) +
         preload_fn(kv_append_f32_kernel) + preload_fn(attention_f32_kernel);
}

}  // namespace ms

using namespace ms;

extern "C" int ms_embed_f32(const int32_t* tok, const int32_t* start, int Q, const void* tok_emb,
                            const void* pos_emb, int pos_offset, int R, int d, float* out, void* stream) {
  if (R < 0 || Q < 1 || d < 1) return MS_ERR_VALUE;
  if (R == 0) return MS_OK;
  if (!tok || !start || !tok_emb || !out) return MS_ERR_VALUE;
  return launch(embed_f32_kernel, dim3(R), dim3(128), 0, (cudaStream_t)stream, 1, tok, start, Q,
                (const __nv_bfloat16*)tok_emb, (const __nv_bfloat16*)pos_emb, pos_offset, d, out);
}

extern "C" int ms_norm_f32(const float* x, int64_t ldx, const int32_t* rows, const void* gamma, const void* beta,
                           float eps, int rms, int R, int d, float* out, int64_t ldo, void* stream) {
  if (R < 0 || d < 1 || ldx < d || ldo < d) return MS_ERR_VALUE;
  if (R == 0) return MS_OK;
  if (!x || !gamma || (!rms && !beta) || !out) return MS_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  auto* g = (const __nv_bfloat16*)gamma;
  auto* b = (const __nv_bfloat16*)beta;
  if (rms) return launch(norm_f32_kernel<true>, dim3(R), dim3(128), 0, st, 1, x, ldx, rows, g, b, eps, d, out, ldo);
  return launch(norm_f32_kernel<false>, dim3(R), dim3(128), 0, st, 1, x, ldx, rows, g, b, eps, d, out, ldo);
}

extern "C" int ms_linear_f32(const float* x, int64_t ldx, const void* w, const void* bias, const float* residual,
                             int64_t ldr, float* out, int64_t ldo, int M, int N, int K, int act, void* stream) {
  if (M < 0 || N < 1 || K < 1 || act < 0 || act > 2 || ldx < K) return MS_ERR_VALUE;
  const int No = act == 2 ? N / 2 : N;
  if (act == 2 && (N % 128 || bias)) return MS_ERR_UNSUPPORTED;
  if (ldo < No || (residual && ldr < No)) return MS_ERR_VALUE;
  if (M == 0) return MS_OK;
  if (!x || !w || !out) return MS_ERR_VALUE;
  dim3 grid((No + F32_BN - 1) / F32_BN, (M + F32_BM - 1) / F32_BM);
  if (grid.y > 65535) return MS_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  auto* wb = (const __nv_bfloat16*)w;
  auto* bb = (const __nv_bfloat16*)bias;
  if (act == 2)
    return launch(linear_f32_kernel<true>, grid, dim3(256), 0, st, 1, x, ldx, wb, bb, residual, ldr, out, ldo, M,
                  No, K, act);
  return launch(linear_f32_kernel<false>, grid, dim3(256), 0, st, 1, x, ldx, wb, bb, residual, ldr, out, ldo, M,
                No, K, act);
}

extern "C" int ms_attention_f32(const float* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                                const int32_t* slot, const int32_t* start, int T, float* k_cache, float* v_cache,
                                const float* rope, float scale, int scale_q, float* out, int64_t ldo,
                                void* stream) {
  if (B < 0 || Q < 1 || H < 1 || Hkv < 1 || H % Hkv || D < 1 || T < 1) return MS_ERR_VALUE;
  if (D > 128 || (rope && D % 2)) return MS_ERR_UNSUPPORTED;
  if (ldq < (int64_t)(H + 2 * Hkv) * D || ldo < (int64_t)H * D) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache || !out) return MS_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch(kv_append_f32_kernel, dim3(B * Q, Hkv), dim3(D), 0, st, 1, qkv, ldq, Q, H, Hkv, D, slot, start,
                  T, k_cache, v_cache, (const float2*)rope);
  if (rc) return rc;
  const int n_items = B * H * Q;
  return launch(attention_f32_kernel, dim3((n_items + 3) / 4), dim3(128), 0, st, 1, qkv, ldq, Q, H, Hkv, D, slot,
                start, T, (const float*)k_cache, (const float*)v_cache, (const float2*)rope, scale, scale_q, out,
                ldo, n_items);
}
