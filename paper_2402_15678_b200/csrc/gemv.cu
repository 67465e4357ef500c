// K1 (drafter decode) — low-latency projection for a handful of token rows.
//
//   out[m, n] = act(sum_k x[m, k] * w[n, k] + bias[n]) + residual[m, n],  M <= 64
//
// A drafter's decode step multiplies 16 token rows by 1-5 MB weights, ~90
// dependent launches per step: its cost is the latency of each GEMM, not
// bytes.  The tcgen05 path pays for 128-row weight tiles, TMEM, mbarriers and
// a cross-CTA split-K reduction on every launch; here one CTA owns 16 output
// features for all rows, its 4 warps split K and reduce in shared memory, and
// the products run on warp-level MMAs (m16n8k16, token rows on M) fed straight
// from global memory with 16-byte loads — no TMEM, no clusters, no scratch.
//
// The 16-byte loads use a permuted K order inside each 32-element chunk (the
// same permutation for x and w, so the dot products are unchanged): lane
// (g, t) reads elements 8t..8t+7 of its rows and feeds them to two m16n8k16
// steps.  The reduction order is fixed, so results are deterministic and a
// row's result does not depend on M.  Weight loads for the first chunks are
// issued before griddepcontrol.wait (PDL), like the tcgen05 path.
//
// act 2 (gated SiLU over the 64-row interleaved gate/up weight of ms_linear):
// a CTA computes 8 gate rows and their 8 up partners (+64) and writes the 8
// outputs silu(g) * u.
#include "common.cuh"

namespace ms {

int coresident();  // attention.cu (ms_set_coresident)
constexpr int kGvN = 16;  // output features per CTA (two n8 tiles)

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// NW warps split K (4, or 8 for long K such as a drafter's down projection,
// K = 3072: 96 KB of weights per CTA, so twice the warps keep twice the loads
// in flight); PRE chunks per warp are requested before the dependency wait.
// NW = 2 is the co-resident shape (ms_set_coresident: drafter steps beside
// the verifier): 64 threads x <= 128 registers, ~2 KB of shared memory — it
// fits next to two verify-GEMM CTAs on an SM.
template <int MT, int kGvWarps>  // 16-row token tiles, K-splitting warps
__global__ void __launch_bounds__(kGvWarps * 32, kGvWarps == 2 ? 8 : 1)
gemv_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, const __nv_bfloat16* __restrict__ w,
            const __nv_bfloat16* __restrict__ bias, const __nv_bfloat16* __restrict__ residual,
            int64_t ldr, void* __restrict__ out, int64_t ldc, int out_f32, int M, int N, int K, int act,
            int64_t w_gstride, float rms_eps) {
  __shared__ float red[kGvWarps][MT * 16][kGvN + 1];
  __shared__ float rsq[kGvWarps][MT * 16];  // folded RMSNorm: per-warp sums of squares of x rows
  const bool rms = rms_eps >= 0.f;
  // row group blockIdx.y (grouped drafters): its M rows, its own weight
  {
    const int grp = blockIdx.y;
    x += (int64_t)grp * M * ldx;
    w += grp * w_gstride;
    if (bias) bias += (int64_t)grp * N;
    if (residual) residual += (int64_t)grp * M * ldr;
    out = reinterpret_cast<char*>(out) + (int64_t)grp * M * ldc * (out_f32 ? 4 : 2);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool gated = act == 2;
  // gated: outputs o0..o0+7, gate rows (o0 / 64) * 128 + o0 % 64 + [0, 8), up rows +64
  const int o0 = blockIdx.x * (kGvN / 2);
  const int n0 = gated ? (o0 / 64) * 128 + o0 % 64 : blockIdx.x * kGvN;
  // this warp's K range, in 32-element chunks
  const int nch = K / 32;
  const int c0 = warp * nch / kGvWarps, c1 = (warp + 1) * nch / kGvWarps;
  // weight rows of the two n8 tiles (clamped: rows >= N are computed, not stored)
  const int wr0 = min(n0 + g, N - 1), wr1 = min(n0 + (gated ? 64 : 8) + g, N - 1);
  const uint4* w0 = reinterpret_cast<const uint4*>(w + (int64_t)wr0 * K) + t;
  const uint4* w1 = reinterpret_cast<const uint4*>(w + (int64_t)wr1 * K) + t;

  constexpr int PRE = kGvWarps == 4 ? 4 : 8;  // chunks of weights loaded before the dependency wait
  uint4 wpre0[PRE], wpre1[PRE];
#pragma unroll
  for (int i = 0; i < PRE; ++i) {
    if (c0 + i < c1) {
      wpre0[i] = __ldg(w0 + (int64_t)(c0 + i) * 4);
      wpre1[i] = __ldg(w1 + (int64_t)(c0 + i) * 4);
    }
  }
  pdl_wait();
  pdl_trigger();

  float acc[MT][2][4];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) acc[m][n][0] = acc[m][n][1] = acc[m][n][2] = acc[m][n][3] = 0.f;
  // token rows of the m tiles (clamped; rows >= M are computed, not stored)
  const uint4* xr[MT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    xr[m][0] = reinterpret_cast<const uint4*>(x + (int64_t)min(m * 16 + g, M - 1) * ldx) + t;
    xr[m][1] = reinterpret_cast<const uint4*>(x + (int64_t)min(m * 16 + 8 + g, M - 1) * ldx) + t;
  }

  float ss[MT][2];  // folded RMSNorm: this lane's sums of squares of rows g, g+8 (its 8-element slices)
#pragma unroll
  for (int m = 0; m < MT; ++m) ss[m][0] = ss[m][1] = 0.f;
  auto sq8 = [](const uint4& v) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      a = fmaf(f.x, f.x, a);
      a = fmaf(f.y, f.y, a);
    }
    return a;
  };
  auto step = [&](const uint4& wa, const uint4& wb, int c) {
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const uint4 xa = xr[m][0][(int64_t)c * 4];  // row g:   elements 8t..8t+7 of chunk c
      const uint4 xb = xr[m][1][(int64_t)c * 4];  // row g+8
      if (rms) {
        ss[m][0] += sq8(xa);
        ss[m][1] += sq8(xb);
      }
      // k-step A uses elements (0,1)|(2,3), k-step B uses (4,5)|(6,7)
      mma_bf16_16816(acc[m][0], xa.x, xb.x, xa.y, xb.y, wa.x, wa.y);
      mma_bf16_16816(acc[m][0], xa.z, xb.z, xa.w, xb.w, wa.z, wa.w);
      mma_bf16_16816(acc[m][1], xa.x, xb.x, xa.y, xb.y, wb.x, wb.y);
      mma_bf16_16816(acc[m][1], xa.z, xb.z, xa.w, xb.w, wb.z, wb.w);
    }
  };
#pragma unroll
  for (int i = 0; i < PRE; ++i)
    if (c0 + i < c1) step(wpre0[i], wpre1[i], c0 + i);
  for (int c = c0 + PRE; c < c1; c += 4) {
    uint4 wa[4], wb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c + u < c1) {
        wa[u] = __ldg(w0 + (int64_t)(c + u) * 4);
        wb[u] = __ldg(w1 + (int64_t)(c + u) * 4);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c + u < c1) step(wa[u], wb[u], c + u);
  }
  // cross-warp K reduction in warp order
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      red[warp][m * 16 + g][n * 8 + 2 * t] = acc[m][n][0];
      red[warp][m * 16 + g][n * 8 + 2 * t + 1] = acc[m][n][1];
      red[warp][m * 16 + g + 8][n * 8 + 2 * t] = acc[m][n][2];
      red[warp][m * 16 + g + 8][n * 8 + 2 * t + 1] = acc[m][n][3];
    }
  if (rms) {  // the 4 lanes t of a row in a fixed shuffle tree, then per warp
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v = ss[m][h];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (t == 0) rsq[warp][m * 16 + g + 8 * h] = v;
      }
  }
  __syncthreads();
  // rstd of row r from the warps' partial sums in warp order (deterministic)
  auto rstd = [&](int r) {
    float v = rsq[0][r];
#pragma unroll
    for (int wi = 1; wi < kGvWarps; ++wi) v += rsq[wi][r];
    return rsqrtf(v / (float)K + rms_eps);
  };
  if (gated) {
    for (int e = threadIdx.x; e < M * 8; e += kGvWarps * 32) {
      const int r = e >> 3, f = e & 7;
      float gv = red[0][r][f], uv = red[0][r][8 + f];
#pragma unroll
      for (int wi = 1; wi < kGvWarps; ++wi) {
        gv += red[wi][r][f];
        uv += red[wi][r][8 + f];
      }
      if (rms) {
        const float rs = rstd(r);
        gv *= rs;
        uv *= rs;
      }
      reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)r * ldc + o0 + f] = f2bf(silu_mul(gv, uv));
    }
    return;
  }
  for (int e = threadIdx.x; e < M * kGvN; e += kGvWarps * 32) {
    const int r = e / kGvN, f = e - r * kGvN;
    const int feat = n0 + f;
    if (feat >= N) continue;
    float v = red[0][r][f];
#pragma unroll
    for (int wi = 1; wi < kGvWarps; ++wi) v += red[wi][r][f];
    if (rms) v *= rstd(r);
    if (bias) v += bf2f(bias[feat]);
    if (act == 1) v = fmaxf(v, 0.f);
    if (residual) v += bf2f(residual[(int64_t)r * ldr + feat]);
    if (out_f32)
      reinterpret_cast<float*>(out)[(int64_t)r * ldc + feat] = v;
    else
      reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)r * ldc + feat] = f2bf(v);
  }
}

int preload_gemv() {
  return preload_fn(gemv_kernel<1, 2>) + preload_fn(gemv_kernel<2, 2>) + preload_fn(gemv_kernel<3, 2>) +
         preload_fn(gemv_kernel<4, 2>) + preload_fn(gemv_kernel<1, 4>) + preload_fn(gemv_kernel<2, 4>) +
         preload_fn(gemv_kernel<3, 4>) +
         preload_fn(gemv_kernel<4, 4>) + preload_fn(gemv_kernel<1, 8>) + preload_fn(gemv_kernel<2, 8>) +
         preload_fn(gemv_kernel<3, 8>) + preload_fn(gemv_kernel<4, 8>);
}

}  // namespace ms

static int gemv_impl(const void* x, int64_t ldx, const void* w, int64_t w_gstride, const void* bias,
                     const void* residual, int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K,
                     int act, int G, float rms_eps, void* stream) {
  if (M < 0 || N < 1 || K < 1 || G < 1 || ldx < K || ldc < (act == 2 ? N / 2 : N)) return MS_ERR_VALUE;
  if (M == 0) return MS_OK;
  if (!x || !w || !out) return MS_ERR_VALUE;
  if (act < 0 || act > 2) return MS_ERR_VALUE;
  if (act == 2 && (N % 128 || bias || residual || out_f32)) return MS_ERR_UNSUPPORTED;
  if (M > 64 || K % 32 || ldx % 8 || w_gstride % 8) return MS_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) return MS_ERR_UNSUPPORTED;
  if (residual && ldr < N) return MS_ERR_VALUE;
  const dim3 grid((N + ms::kGvN - 1) / ms::kGvN, G);
  cudaStream_t st = (cudaStream_t)stream;
  const auto* xb = (const __nv_bfloat16*)x;
  const auto* wb = (const __nv_bfloat16*)w;
  const auto* bb = (const __nv_bfloat16*)bias;
  const auto* rb = (const __nv_bfloat16*)residual;
#define MS_GV(MT, NW) \
  ms::launch(ms::gemv_kernel<MT, NW>, grid, dim3(NW * 32), 0, st, 1, xb, ldx, wb, bb, rb, ldr, out, ldc, out_f32, M, N, K, act, w_gstride, rms_eps)
  const int mt = (M + 15) / 16;
  if (ms::coresident()) {
    switch (mt) {
      case 1: return MS_GV(1, 2);
      case 2: return MS_GV(2, 2);
      case 3: return MS_GV(3, 2);
      default: return MS_GV(4, 2);
    }
  }
  // 8 warps only for long K: at K = 768 they measured slower (gate/up 12.5 vs
  // 10.5 us per 3-drafter call, QKV 6.6 vs 5.6; tools/draft_breakdown.py)
  if (K > 1024) {
    switch (mt) {
      case 1: return MS_GV(1, 8);
      case 2: return MS_GV(2, 8);
      case 3: return MS_GV(3, 8);
      default: return MS_GV(4, 8);
    }
  }
  switch (mt) {
    case 1: return MS_GV(1, 4);
    case 2: return MS_GV(2, 4);
    case 3: return MS_GV(3, 4);
    default: return MS_GV(4, 4);
  }
#undef MS_GV
}

extern "C" int ms_gemv_grouped(const void* x, int64_t ldx, const void* w, int64_t w_gstride, const void* bias,
                               const void* residual, int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N,
                               int K, int act, int G, void* stream) {
  return gemv_impl(x, ldx, w, w_gstride, bias, residual, ldr, out, ldc, out_f32, M, N, K, act, G, -1.f, stream);
}

extern "C" int ms_gemv_rms_grouped(const void* x, int64_t ldx, const void* w, int64_t w_gstride,
                                   const void* residual, int64_t ldr, void* out, int64_t ldc, int out_f32, int M,
                                   int N, int K, int act, int G, float eps, void* stream) {
  if (!(eps >= 0.f)) return MS_ERR_VALUE;
  return gemv_impl(x, ldx, w, w_gstride, nullptr, residual, ldr, out, ldc, out_f32, M, N, K, act, G, eps, stream);
}

extern "C" int ms_gemv(const void* x, int64_t ldx, const void* w, const void* bias, const void* residual,
                       int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K, int act,
                       void* stream) {
  return ms_gemv_grouped(x, ldx, w, 0, bias, residual, ldr, out, ldc, out_f32, M, N, K, act, 1, stream);
}
