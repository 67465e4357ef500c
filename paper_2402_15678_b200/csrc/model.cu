// K2/K6/K7 — the non-GEMM pieces of an OPT-style decoder forward:
//   embed (token + learned position), LayerNorm, KV-cache append, and the
//   KV-cache attention of Q consecutive query rows per request (Q = s+1 for
//   the LLM verify forward, 1 for an SSM decode step, the catch-up length for
//   an SSM's first step of a round).
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
                             int pos_offset, int d, __nv_bfloat16* __restrict__ out) {
  const int r = blockIdx.x;
  const int pos = start[r / Q] + r % Q;
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
// LayerNorm over d (fp32 statistics, two-pass on registers), bf16 out.
// One CTA of 128 threads per row; each thread holds d/1024 16-byte vectors.
// ---------------------------------------------------------------------------
template <int VPT>  // bf16x8 vectors per thread
__global__ void __launch_bounds__(128)
layernorm_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, const int32_t* __restrict__ rows,
                 const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, float eps,
                 int d, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  const int r = blockIdx.x;
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
        const float c = v[k][j] - mean;
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
      unpack8(bv[i], fb);
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = (v[k][j] - mean) * rstd * fg[j] + fb[j];
      o[i] = pack8(y);
    }
  }
}

// ---------------------------------------------------------------------------
// KV append: rows r = b*Q + i of qkv [R, 3*H*D] -> cache[slot[b], h, start[b]+i, :]
// cache layout [slots, H, T, D] bf16 (K and V separate).
// ---------------------------------------------------------------------------
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Q, int H, int D,
                                 const int32_t* __restrict__ slot, const int32_t* __restrict__ start,
                                 int T, __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc) {
  const int r = blockIdx.x;
  const int b = r / Q, i = r - b * Q;
  const int p = start[b] + i;
  if (p < 0 || p >= T) return;
  const int hd8 = H * D / 8;
  const bf16x8* src = reinterpret_cast<const bf16x8*>(qkv + (int64_t)r * ldq);
  const int64_t sb = (int64_t)slot[b] * H;
  for (int e = threadIdx.x; e < 2 * hd8; e += blockDim.x) {
    const int kv = e >= hd8;
    const int f = (e - kv * hd8) * 8;  // feature within K (or V)
    const int h = f / D, dd = f - h * D;
    bf16x8 val = src[hd8 + e];  // skip Q
    __nv_bfloat16* dst = (kv ? vc : kc) + ((sb + h) * T + p) * D + dd;
    *reinterpret_cast<bf16x8*>(dst) = val;
  }
}

// ---------------------------------------------------------------------------
// Attention of Q causal query rows per (request, head) over the KV cache.
// Query i of request b sits at position start[b]+i and attends to cache
// positions 0..start[b]+i.  One CTA (4 warps) per (b, h); warp w owns the
// 32-key blocks kb with kb % 4 == w (a fixed partition, independent of Q), so
// each query's result is the same whatever the other queries are.
//   scores: lane = key, q from smem (fp32), D-length dot per query
//   P·V:    lane = D/32 output dims, V rows read coalesced
// ---------------------------------------------------------------------------
constexpr int kAttnWarps = 4;

template <int D, int QMAX>
__global__ void __launch_bounds__(kAttnWarps * 32)
attention_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Qtot, int H,
                 const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                 const __nv_bfloat16* __restrict__ kc, const __nv_bfloat16* __restrict__ vc,
                 float scale, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  constexpr int DL = D / 32;  // output dims per lane
  const int b = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float sq[QMAX][D];
  __shared__ float sp[kAttnWarps][QMAX][33];
  __shared__ float sm[kAttnWarps][QMAX], sl[kAttnWarps][QMAX];
  __shared__ float sacc[QMAX][D];

  // this CTA's query chunk: rows q0 .. q0+Q-1 of the request's Qtot rows
  const int q0 = blockIdx.z * QMAX;
  const int Q = min(QMAX, Qtot - q0);
  const int p0 = start[b] + q0;
  const int64_t cbase = ((int64_t)slot[b] * H + h) * T * D;
  const __nv_bfloat16* K = kc + cbase;
  const __nv_bfloat16* V = vc + cbase;
  // stage q (pre-scaled) in fp32
  for (int e = threadIdx.x; e < Q * D; e += blockDim.x) {
    const int i = e / D, dd = e - i * D;
    sq[i][dd] = bf2f(qkv[(int64_t)(b * Qtot + q0 + i) * ldq + h * D + dd]) * scale;
  }
  __syncthreads();

  float m[QMAX], l[QMAX], acc[QMAX][DL];
#pragma unroll
  for (int i = 0; i < QMAX; ++i) {
    m[i] = -INFINITY;
    l[i] = 0.f;
#pragma unroll
    for (int j = 0; j < DL; ++j) acc[i][j] = 0.f;
  }
  const int n_keys = min(p0 + Q, T);  // keys 0 .. p0+Q-1
  const int n_blocks = (n_keys + 31) / 32;
  for (int kb = warp; kb < n_blocks; kb += kAttnWarps) {
    const int t = kb * 32 + lane;
    float sc[QMAX];
    if (t < n_keys) {
      const bf16x8* kr = reinterpret_cast<const bf16x8*>(K + (int64_t)t * D);
#pragma unroll
      for (int i = 0; i < QMAX; ++i) sc[i] = 0.f;
#pragma unroll 4
      for (int c = 0; c < D / 8; ++c) {
        float kf[8];
        unpack8(kr[c], kf);
#pragma unroll
        for (int i = 0; i < QMAX; ++i) {
          if (i < Q) {
#pragma unroll
            for (int j = 0; j < 8; ++j) sc[i] = fmaf(sq[i][c * 8 + j], kf[j], sc[i]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < QMAX; ++i)
        if (t > p0 + i) sc[i] = -INFINITY;  // causal
    } else {
#pragma unroll
      for (int i = 0; i < QMAX; ++i) sc[i] = -INFINITY;
    }
    // online softmax update per query (warp-wide over the 32 keys)
#pragma unroll
    for (int i = 0; i < QMAX; ++i) {
      if (i < Q) {
        const float bm = warp_max(sc[i]);
        const float mn = fmaxf(m[i], bm);
        float p = 0.f, corr = 1.f;
        if (mn != -INFINITY) {
          p = __expf(sc[i] - mn);
          corr = __expf(m[i] - mn);
        }
        l[i] = l[i] * corr + warp_sum(p);
        m[i] = mn;
#pragma unroll
        for (int j = 0; j < DL; ++j) acc[i][j] *= corr;
        sp[warp][i][lane] = p;
      }
    }
    __syncwarp();
    const int kmax = min(32, n_keys - kb * 32);
    for (int jj = 0; jj < kmax; ++jj) {
      const __nv_bfloat16* vr = V + (int64_t)(kb * 32 + jj) * D + lane * DL;
      float vf[DL];
      if constexpr (DL == 4) {
        const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(vr);
        float2 a = __bfloat1622float2(v2[0]), c = __bfloat1622float2(v2[1]);
        vf[0] = a.x; vf[1] = a.y; vf[2] = c.x; vf[3] = c.y;
      } else {
        float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        vf[0] = a.x; vf[1] = a.y;
      }
#pragma unroll
      for (int i = 0; i < QMAX; ++i) {
        if (i < Q) {
          const float pw = sp[warp][i][jj];
#pragma unroll
          for (int j = 0; j < DL; ++j) acc[i][j] = fmaf(pw, vf[j], acc[i][j]);
        }
      }
    }
    __syncwarp();
  }
  // combine the 4 warps in warp order (fixed order => deterministic)
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < QMAX; ++i) {
      sm[warp][i] = m[i];
      sl[warp][i] = l[i];
    }
  }
  __syncthreads();
  float f[QMAX];
#pragma unroll
  for (int i = 0; i < QMAX; ++i) {
    float mx = sm[0][i];
#pragma unroll
    for (int w = 1; w < kAttnWarps; ++w) mx = fmaxf(mx, sm[w][i]);
    f[i] = m[i] == -INFINITY ? 0.f : __expf(m[i] - mx);
  }
  for (int w = 0; w < kAttnWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < QMAX; ++i) {
        if (i < Q) {
#pragma unroll
          for (int j = 0; j < DL; ++j) {
            const float c = acc[i][j] * f[i];
            sacc[i][lane * DL + j] = w == 0 ? c : sacc[i][lane * DL + j] + c;
          }
        }
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < Q * D; e += blockDim.x) {
    const int i = e / D, dd = e - i * D;
    float mx = sm[0][i];
#pragma unroll
    for (int w = 1; w < kAttnWarps; ++w) mx = fmaxf(mx, sm[w][i]);
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w)
      L += sm[w][i] == -INFINITY ? 0.f : sl[w][i] * __expf(sm[w][i] - mx);
    out[(int64_t)(b * Qtot + q0 + i) * ldo + h * D + dd] = f2bf(sacc[i][dd] / L);
  }
}

template <int D>
static int launch_attention(const void* qkv, int64_t ldq, int B, int Q, int H, const int32_t* slot,
                            const int32_t* start, int T, const void* kc, const void* vc, float scale,
                            void* out, int64_t ldo, cudaStream_t st) {
  const int qm = Q <= 1 ? 1 : Q <= 4 ? 4 : Q <= 8 ? 8 : Q <= 13 ? 13 : Q <= 17 ? 17 : 16;
  dim3 grid(B, H, (Q + qm - 1) / qm);
  const auto* q = (const __nv_bfloat16*)qkv;
  const auto* k = (const __nv_bfloat16*)kc;
  const auto* v = (const __nv_bfloat16*)vc;
  auto* o = (__nv_bfloat16*)out;
#define MS_ATTN(QM)                                                                              \
  attention_kernel<D, QM><<<grid, kAttnWarps * 32, 0, st>>>(q, ldq, Q, H, slot, start, T, k, v, \
                                                            scale, o, ldo)
  if (Q <= 1) MS_ATTN(1);
  else if (Q <= 4) MS_ATTN(4);
  else if (Q <= 8) MS_ATTN(8);
  else if (Q <= 13) MS_ATTN(13);
  else if (Q <= 17) MS_ATTN(17);
  else MS_ATTN(16);  // long prefill: chunks of 16 queries per CTA
#undef MS_ATTN
  count_launch();
  return launch_status();
}

}  // namespace ms

extern "C" int ms_embed(const int32_t* tok, const int32_t* start, int Q, const void* tok_emb,
                        const void* pos_emb, int pos_offset, int R, int d, void* out, void* stream) {
  if (R < 0 || d < 8 || Q < 1) return MS_ERR_VALUE;
  if (d % 8) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  if (!tok || !start || !tok_emb || !out) return MS_ERR_VALUE;
  ms::embed_kernel<<<R, 128, 0, (cudaStream_t)stream>>>(
      tok, start, Q, (const __nv_bfloat16*)tok_emb, (const __nv_bfloat16*)pos_emb, pos_offset, d,
      (__nv_bfloat16*)out);
  ms::count_launch();
  return ms::launch_status();
}

extern "C" int ms_layernorm(const void* x, int64_t ldx, const int32_t* rows, const void* gamma,
                            const void* beta, float eps, int R, int d, void* out, int64_t ldo,
                            void* stream) {
  if (R < 0 || d < 8) return MS_ERR_VALUE;
  if (d % 8 || d > 8 * 128 * 8 || ldx % 8 || ldo % 8) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  if (!x || !gamma || !beta || !out) return MS_ERR_VALUE;
  const int vpt = (d / 8 + 127) / 128;
  cudaStream_t st = (cudaStream_t)stream;
  auto* xi = (const __nv_bfloat16*)x;
  auto* g = (const __nv_bfloat16*)gamma;
  auto* b = (const __nv_bfloat16*)beta;
  auto* o = (__nv_bfloat16*)out;
  switch (vpt) {
    case 1: ms::layernorm_kernel<1><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
    case 2: ms::layernorm_kernel<2><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
    case 3: ms::layernorm_kernel<3><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
    case 4: ms::layernorm_kernel<4><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
    case 5: ms::layernorm_kernel<5><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
    case 6: ms::layernorm_kernel<6><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
    case 7: ms::layernorm_kernel<7><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
    default: ms::layernorm_kernel<8><<<R, 128, 0, st>>>(xi, ldx, rows, g, b, eps, d, o, ldo); break;
  }
  ms::count_launch();
  return ms::launch_status();
}

extern "C" int ms_kv_append(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                            const int32_t* slot, const int32_t* start, int T, void* k_cache,
                            void* v_cache, void* stream) {
  if (B < 0 || Q < 1 || H < 1 || D < 8 || T < 1) return MS_ERR_VALUE;
  if (D % 8 || ldq % 8) return MS_ERR_UNSUPPORTED;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache) return MS_ERR_VALUE;
  ms::kv_append_kernel<<<B * Q, 128, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)qkv, ldq, Q, H, D, slot, start, T, (__nv_bfloat16*)k_cache,
      (__nv_bfloat16*)v_cache);
  ms::count_launch();
  return ms::launch_status();
}

extern "C" int ms_attention(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                            const int32_t* slot, const int32_t* start, int T, const void* k_cache,
                            const void* v_cache, float scale, void* out, int64_t ldo, void* stream) {
  if (B < 0 || Q < 1 || H < 1 || T < 1) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache || !out) return MS_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  if (D == 64)
    return ms::launch_attention<64>(qkv, ldq, B, Q, H, slot, start, T, k_cache, v_cache, scale, out, ldo, st);
  if (D == 128)
    return ms::launch_attention<128>(qkv, ldq, B, Q, H, slot, start, T, k_cache, v_cache, scale, out, ldo, st);
  return MS_ERR_UNSUPPORTED;
}
