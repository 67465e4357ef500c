// K2/K6/K7 — the non-GEMM pieces of an OPT-style decoder forward:
//   embed (token + learned position), LayerNorm and the KV-cache append of
//   long (prefill) chunks.  The attention itself is attention.cu.
//
// These replace the model forward that the reference abstracts away behind
// ModelOracle.next_dist (aggspec/oracles.py:19-26), called per position by
// draft_sequence (aggspec/oracles.py:148) and by _do_verify_batch
// (aggspec/engine.py:294-296).  All are HBM-bound: activations and the KV
// cache are read once with 16-byte vector loads.
//
// Numerics contract (shared with the fp32 oracle in oracle/opt_ref.py):
// activations/weights/KV are bf16; every reduction is fp32; each kernel rounds
// its result to bf16 exactly once.  Every row's result depends only on that
// row's inputs (no dependence on the number of rows or the batch), which makes
// the forward batch-invariant.
#include "common.cuh"

namespace ms {

// ---------------------------------------------------------------------------
// embed: x[r] = tok_emb[tok[r]] + pos_emb[start[r / Q] + r % Q + pos_offset]
// ---------------------------------------------------------------------------
__global__ void embed_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ start, int Q,
                             const __nv_bfloat16* __restrict__ te, const __nv_bfloat16* __restrict__ pe,
                             int pos_offset, int d, __nv_bfloat16* __restrict__ out, int rpg, int64_t tstride) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int pos = start[r / Q] + r % Q;
  if (rpg > 0) te += (int64_t)(r / rpg) * tstride;  // row group = its own table (grouped drafters)
  const bf16x8* a = reinterpret_cast<const bf16x8*>(te + (int64_t)tok[r] * d);
  const bf16x8* b = pe ? reinterpret_cast<const bf16x8*>(pe + (int64_t)(pos + pos_offset) * d) : nullptr;
  bf16x8* o = reinterpret_cast<bf16x8*>(out + (int64_t)r * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    float fa[8], fb[8];
    unpack8(a[i], fa);
    if (b) {
      unpack8(b[i], fb);
#pragma unroll
      for (int j = 0; j < 8; ++j) fa[j] += fb[j];
    }
    o[i] = pack8(fa);
  }
}

// ---------------------------------------------------------------------------
// LayerNorm over d (fp32 statistics, two-pass on registers), bf16 out; with
// RMS = true the Llama RMSNorm y = x * rsqrt(mean(x^2) + eps) * g (no mean,
// no bias).  One CTA of 128 threads per row; each thread holds d/1024 16-byte
// vectors.
// ---------------------------------------------------------------------------
template <int VPT, bool RMS = false>  // bf16x8 vectors per thread
__global__ void __launch_bounds__(128)
layernorm_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, const int32_t* __restrict__ rows,
                 const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, float eps,
                 int d, __nv_bfloat16* __restrict__ out, int64_t ldo, int rpg, int64_t gstride) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (rpg > 0) g += (int64_t)(r / rpg) * gstride;  // output-row group = its own gain (grouped drafters)
  const int nv = d / 8;
  const bf16x8* xr = reinterpret_cast<const bf16x8*>(x + (int64_t)(rows ? rows[r] : r) * ldx);
  float v[VPT][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * 128;
    if (i < nv) {
      unpack8(xr[i], v[k]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[k][j];
    }
  }
  __shared__ float red[4];
  __shared__ float stat;
  if (RMS) s = 0.f;  // no centring
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) stat = (red[0] + red[1] + red[2] + red[3]) / (float)d;
  __syncthreads();
  const float mean = stat;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * 128;
    if (i < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float c = RMS ? v[k][j] : v[k][j] - mean;
        q += c * c;
      }
    }
  }
  q = warp_sum(q);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) stat = rsqrtf((red[0] + red[1] + red[2] + red[3]) / (float)d + eps);
  __syncthreads();
  const float rstd = stat;
  const bf16x8* gv = reinterpret_cast<const bf16x8*>(g);
  const bf16x8* bv = reinterpret_cast<const bf16x8*>(b);
  bf16x8* o = reinterpret_cast<bf16x8*>(out + (int64_t)r * ldo);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * 128;
    if (i < nv) {
      float fg[8], fb[8], y[8];
      unpack8(gv[i], fg);
      if (RMS) {
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = v[k][j] * rstd * fg[j];
      } else {
        unpack8(bv[i], fb);
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = (v[k][j] - mean) * rstd * fg[j] + fb[j];
      }
      o[i] = pack8(y);
    }
  }
}

// ---------------------------------------------------------------------------
// KV append: rows r = b*Q + i of qkv [R, (H + 2*Hkv)*D] (Q | K | V column
// blocks) -> cache[slot[b], hk, start[b]+i, :], cache layout [slots, Hkv, T, D]
// bf16 (K and V separate).  With a RoPE table the K rows are rotated at their
// absolute position first (fp32, one bf16 rounding).
// ---------------------------------------------------------------------------
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Q, int H, int Hkv,
                                 int D, const int32_t* __restrict__ slot, const int32_t* __restrict__ start,
                                 int T, __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                                 const float2* __restrict__ rope, KVPage pg) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int b = r / Q, i = r - b * Q;
  const int p = start[b] + i;
  if (p < 0 || p >= T) return;
  const int hd8 = Hkv * D / 8;
  const bf16x8* src = reinterpret_cast<const bf16x8*>(qkv + (int64_t)r * ldq + (int64_t)H * D);  // skip Q
  const int sl = slot[b];
  const int v8 = D / 8;
  for (int e = threadIdx.x; e < 2 * hd8; e += blockDim.x) {
    const int kv = e >= hd8;
    const int f = (e - kv * hd8) * 8;  // feature within K (or V)
    const int h = f / D, dd = f - h * D;
    bf16x8 val = src[e];
    if (!kv && rope) {
      const int c = dd / 8;
      const int pc = c < v8 / 2 ? c + v8 / 2 : c - v8 / 2;
      float fv[8], pf[8];
      unpack8(val, fv);
      unpack8(src[h * v8 + pc], pf);
      rope8(fv, pf, rope + (int64_t)p * (D / 2), dd, D / 2);
      val = pack8(fv);
    }
    __nv_bfloat16* dst = (kv ? vc : kc) + kv_row(pg, sl, Hkv, h, T, p) * D + dd;
    *reinterpret_cast<bf16x8*>(dst) = val;
  }
}

// Gated SiLU of a prefill gate/up GEMM's fp32 output (cuBLAS, 64-row
// interleaved weight: output tile t = columns 128t..128t+63 gate, 128t+64..
// 128t+127 up): out[m][64t + j] = bf16(silu(g) * u) — the same fp32 formula
// and single rounding as ms_linear's gated epilogue.  One thread per 4 outputs
// (16-byte gate / up loads, 8-byte store).
__global__ void gated_silu_kernel(const float* __restrict__ gu, int64_t ldg, int M, int N2,
                                  __nv_bfloat16* __restrict__ out, int64_t ldo) {
  pdl_wait();
  pdl_trigger();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // quad index
  const int qpr = N2 / 4;                                               // quads per row
  if (q >= (int64_t)M * qpr) return;
  const int m = (int)(q / qpr), o = (int)(q - (int64_t)m * qpr) * 4;  // output feature
  const int t = o / 64, j = o - t * 64;
  const float* row = gu + (int64_t)m * ldg + t * 128 + j;
  const float4 g = *reinterpret_cast<const float4*>(row);
  const float4 u = *reinterpret_cast<const float4*>(row + 64);
  __nv_bfloat162 lo = __floats2bfloat162_rn(silu_mul(g.x, u.x), silu_mul(g.y, u.y));
  __nv_bfloat162 hi = __floats2bfloat162_rn(silu_mul(g.z, u.z), silu_mul(g.w, u.w));
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(out + (int64_t)m * ldo + o) = pk;
}

int preload_model() {
  int n = preload_fn(embed_kernel) + preload_fn(kv_append_kernel) + preload_fn(gated_silu_kernel);
  n += preload_fn(layernorm_kernel<1, false>) + preload_fn(layernorm_kernel<2, false>) +
       preload_fn(layernorm_kernel<3, false>) + preload_fn(layernorm_kernel<4, false>) +
       preload_fn(layernorm_kernel<5, false>) + preload_fn(layernorm_kernel<6, false>) +
       preload_fn(layernorm_kernel<7, false>) + preload_fn(layernorm_kernel<8, false>);
  n += preload_fn(layernorm_kernel<1, true>) + preload_fn(layernorm_kernel<2, true>) +
       preload_fn(layernorm_kernel<3, true>) + preload_fn(layernorm_kernel<4, true>) +
       preload_fn(layernorm_kernel<5, true>) + preload_fn(layernorm_kernel<6, true>) +
       preload_fn(layernorm_kernel<7, true>) + preload_fn(layernorm_kernel<8, true>);
  return n;
}

}  // namespace ms

extern "C" int ms_embed_grouped(const int32_t* tok, const int32_t* start, int Q, const void* tok_emb,
                                int64_t tstride, int rpg, const void* pos_emb, int pos_offset, int R, int d,
                                void* out, void* stream) {
  if (R < 0 || d < 8 || Q < 1 || rpg < 0) return MS_ERR_VALUE;
  if (d % 8) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  if (!tok || !start || !tok_emb || !out) return MS_ERR_VALUE;
  return ms::launch(ms::embed_kernel, dim3(R), dim3(128), 0, (cudaStream_t)stream, 1, tok, start, Q,
                    (const __nv_bfloat16*)tok_emb, (const __nv_bfloat16*)pos_emb, pos_offset, d,
                    (__nv_bfloat16*)out, rpg, tstride);
}

extern "C" int ms_embed(const int32_t* tok, const int32_t* start, int Q, const void* tok_emb,
                        const void* pos_emb, int pos_offset, int R, int d, void* out, void* stream) {
  return ms_embed_grouped(tok, start, Q, tok_emb, 0, 0, pos_emb, pos_offset, R, d, out, stream);
}

template <bool RMS>
static int norm_launch(const void* x, int64_t ldx, const int32_t* rows, const void* gamma, const void* beta,
                       float eps, int R, int d, void* out, int64_t ldo, void* stream, int rpg = 0,
                       int64_t gstride = 0) {
  if (R < 0 || d < 8) return MS_ERR_VALUE;
  if (d % 8 || d > 8 * 128 * 8 || ldx % 8 || ldo % 8) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  if (!x || !gamma || (!RMS && !beta) || !out) return MS_ERR_VALUE;
  const int vpt = (d / 8 + 127) / 128;
  cudaStream_t st = (cudaStream_t)stream;
  auto* xi = (const __nv_bfloat16*)x;
  auto* g = (const __nv_bfloat16*)gamma;
  auto* b = (const __nv_bfloat16*)beta;
  auto* o = (__nv_bfloat16*)out;
  switch (vpt) {
    case 1: return ms::launch(ms::layernorm_kernel<1, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
    case 2: return ms::launch(ms::layernorm_kernel<2, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
    case 3: return ms::launch(ms::layernorm_kernel<3, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
    case 4: return ms::launch(ms::layernorm_kernel<4, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
    case 5: return ms::launch(ms::layernorm_kernel<5, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
    case 6: return ms::launch(ms::layernorm_kernel<6, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
    case 7: return ms::launch(ms::layernorm_kernel<7, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
    default: return ms::launch(ms::layernorm_kernel<8, RMS>, dim3(R), dim3(128), 0, st, 1, xi, ldx, rows, g, b, eps, d, o, ldo, rpg, gstride);
  }
}

extern "C" int ms_layernorm(const void* x, int64_t ldx, const int32_t* rows, const void* gamma,
                            const void* beta, float eps, int R, int d, void* out, int64_t ldo,
                            void* stream) {
  return norm_launch<false>(x, ldx, rows, gamma, beta, eps, R, d, out, ldo, stream);
}

extern "C" int ms_rmsnorm(const void* x, int64_t ldx, const int32_t* rows, const void* gamma, float eps,
                          int R, int d, void* out, int64_t ldo, void* stream) {
  return norm_launch<true>(x, ldx, rows, gamma, nullptr, eps, R, d, out, ldo, stream);
}

extern "C" int ms_gated_silu(const float* gu, int64_t ldg, int M, int N, void* out, int64_t ldo, void* stream) {
  if (M < 0 || N < 0 || N % 128 || ldg < N || ldo < N / 2) return MS_ERR_VALUE;
  if (M == 0 || N == 0) return MS_OK;
  if (!gu || !out) return MS_ERR_VALUE;
  if (ldg % 4 || ldo % 4 || (reinterpret_cast<uintptr_t>(gu) & 15) || (reinterpret_cast<uintptr_t>(out) & 7))
    return MS_ERR_UNSUPPORTED;
  const int64_t quads = (int64_t)M * (N / 8);
  const int64_t blocks = (quads + 255) / 256;
  if (blocks > 0x7fffffff) return MS_ERR_UNSUPPORTED;
  return ms::launch(ms::gated_silu_kernel, dim3((unsigned)blocks), dim3(256), 0, (cudaStream_t)stream, 1, gu, ldg, M,
                    N / 2, (__nv_bfloat16*)out, ldo);
}

extern "C" int ms_rmsnorm_grouped(const void* x, int64_t ldx, const int32_t* rows, const void* gamma,
                                  int64_t gstride, int rpg, float eps, int R, int d, void* out, int64_t ldo,
                                  void* stream) {
  if (rpg < 1) return MS_ERR_VALUE;
  return norm_launch<true>(x, ldx, rows, gamma, nullptr, eps, R, d, out, ldo, stream, rpg, gstride);
}

extern "C" int ms_kv_append_paged(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                                  const int32_t* slot, const int32_t* start, int T, void* k_cache,
                                  void* v_cache, const void* rope, const int32_t* block_table, int max_blocks,
                                  int block_size, void* stream) {
  if (B < 0 || Q < 1 || H < 1 || Hkv < 1 || D < 8 || T < 1) return MS_ERR_VALUE;
  if (H % Hkv) return MS_ERR_VALUE;
  if (block_table && (block_size < 1 || max_blocks < 1 || T > max_blocks * block_size)) return MS_ERR_VALUE;
  if (D % 8 || ldq % 8 || (rope && D % 16)) return MS_ERR_UNSUPPORTED;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache) return MS_ERR_VALUE;
  const ms::KVPage pg{block_table, max_blocks, block_size};
  return ms::launch(ms::kv_append_kernel, dim3(B * Q), dim3(128), 0, (cudaStream_t)stream, 1,
                    (const __nv_bfloat16*)qkv, ldq, Q, H, Hkv, D, slot, start, T, (__nv_bfloat16*)k_cache,
                    (__nv_bfloat16*)v_cache, (const float2*)rope, pg);
}

extern "C" int ms_kv_append_gqa(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                                const int32_t* slot, const int32_t* start, int T, void* k_cache,
                                void* v_cache, const void* rope, void* stream) {
  return ms_kv_append_paged(qkv, ldq, B, Q, H, Hkv, D, slot, start, T, k_cache, v_cache, rope, nullptr, 0, 0,
                            stream);
}

extern "C" int ms_kv_append(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                            const int32_t* slot, const int32_t* start, int T, void* k_cache,
                            void* v_cache, void* stream) {
  return ms_kv_append_gqa(qkv, ldq, B, Q, H, H, D, slot, start, T, k_cache, v_cache, nullptr, stream);
}
