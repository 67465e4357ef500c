// K2/K6 — KV-cache attention of Q consecutive query rows per request
// (Q = s+1 for the LLM verify forward, 1 for an SSM decode step, the catch-up
// length for an SSM's first step of a round), with the KV-cache append (K7)
// fused in.  Replaces the attention inside ModelOracle.next_dist
// (aggspec/oracles.py:19-26) for the draft (aggspec/oracles.py:148) and
// verify (aggspec/engine.py:294-296) positions.
//
// One CTA (4 warps) per (request, head[, query chunk]).  The request's K and
// V streams [T, D] are staged through shared memory in tiles of 64 keys with
// cp.async double buffering (16-byte copies, every thread issuing several in
// flight), so each K/V byte is read from HBM once for all the queries of the
// request — the kernel is HBM-bound on the KV cache.  Scores, online softmax
// and P·V run from shared memory in fp32.
//
// Batch invariance: a query's score/softmax/P·V arithmetic is fixed by its own
// position (same tile order, same per-tile reductions); other queries only add
// fully-masked tiles whose contribution is exactly zero.
#include "common.cuh"

namespace ms {

constexpr int kKT = 64;        // keys per tile
constexpr int kAThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int D, int QM>
struct AttnSmem {
  static constexpr int LD = D + 8;  // padded row: 16-byte row chunks land in distinct bank groups
  static constexpr int KV_BYTES = 2 * 2 * kKT * LD * 2;  // [K|V][buf][KT][LD] bf16
  static constexpr int Q_BYTES = QM * D * 4;
  static constexpr int P_BYTES = QM * kKT * 4;
  static constexpr int BYTES = KV_BYTES + Q_BYTES + P_BYTES + 3 * QM * 4;
};

template <int D, int QM>
__global__ void __launch_bounds__(kAThreads)
attention_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Qtot, int H,
                 const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                 __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, float scale,
                 int fuse_append, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  using S = AttnSmem<D, QM>;
  constexpr int LD = S::LD;
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_wait();
  pdl_trigger();
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem);  // [2][KT][LD]
  __nv_bfloat16* sV = sK + 2 * kKT * LD;                          // [2][KT][LD]
  float* sQ = reinterpret_cast<float*>(smem + S::KV_BYTES);        // [QM][D]
  float* sP = sQ + QM * D;                                         // [QM][KT]
  float* sCorr = sP + QM * kKT;                                    // [QM]
  float* sL = sCorr + QM;                                          // [QM]

  const int b = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = blockIdx.z * QM;
  const int Q = min(QM, Qtot - q0);
  const int pstart = start[b];
  const int p0 = pstart + q0;
  const int64_t cbase = ((int64_t)slot[b] * H + h) * T * D;
  __nv_bfloat16* K = kc + cbase;
  __nv_bfloat16* V = vc + cbase;
  const int HD = H * D;

  if (fuse_append) {
    // this request's new K/V rows for head h -> cache (single query chunk only)
    constexpr int V8 = D / 8;
    for (int e = tid; e < 2 * Qtot * V8; e += kAThreads) {
      const int kv = e >= Qtot * V8;
      const int e2 = e - kv * Qtot * V8;
      const int i = e2 / V8, c = e2 - i * V8;
      const int p = pstart + i;
      if (p < 0 || p >= T) continue;
      const bf16x8 val = *reinterpret_cast<const bf16x8*>(
          qkv + (int64_t)(b * Qtot + i) * ldq + (1 + kv) * HD + h * D + c * 8);
      *reinterpret_cast<bf16x8*>((kv ? V : K) + (int64_t)p * D + c * 8) = val;
    }
    __threadfence();
  }
  for (int e = tid; e < Q * D; e += kAThreads) {
    const int i = e / D, dd = e - i * D;
    sQ[e] = bf2f(qkv[(int64_t)(b * Qtot + q0 + i) * ldq + h * D + dd]) * scale;
  }
  __syncthreads();

  const int n_keys = min(p0 + Q, T);  // keys 0 .. p0+Q-1
  const int n_tiles = (n_keys + kKT - 1) / kKT;

  auto load_tile = [&](int tile, int buf) {
    constexpr int V8 = D / 8;
    const int t0 = tile * kKT;
    const int rows = min(kKT, n_keys - t0);
    for (int e = tid; e < 2 * kKT * V8; e += kAThreads) {
      const int kv = e >= kKT * V8;
      const int e2 = e - kv * kKT * V8;
      const int j = e2 / V8, c = e2 - j * V8;
      if (j < rows) {
        const __nv_bfloat16* src = (kv ? V : K) + (int64_t)(t0 + j) * D + c * 8;
        __nv_bfloat16* dst = (kv ? sV : sK) + (buf * kKT + j) * LD + c * 8;
        cp_async16(dst, src);
      }
    }
    cp_async_commit();
  };

  // per-query softmax state lives in the warp that owns query i (i % 4 == warp)
  constexpr int QW = (QM + 3) / 4;
  float m_r[QW], l_r[QW];
#pragma unroll
  for (int u = 0; u < QW; ++u) {
    m_r[u] = -INFINITY;
    l_r[u] = 0.f;
  }
  // P·V ownership: thread -> output dim d, queries i = g, g + NG, ...
  constexpr int NG = kAThreads / D;  // 1 (D=128) or 2 (D=64)
  constexpr int QT = (QM + NG - 1) / NG;
  const int d = tid % D;
  const int g = tid / D;
  float acc[QT];
#pragma unroll
  for (int u = 0; u < QT; ++u) acc[u] = 0.f;

  if (n_tiles > 0) load_tile(0, 0);
  for (int tile = 0; tile < n_tiles; ++tile) {
    const int buf = tile & 1;
    if (tile + 1 < n_tiles) {
      load_tile(tile + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int t0 = tile * kKT;
    // scores S[i][j] = q_i . k_j (fp32, sequential over d)
    const __nv_bfloat16* kt = sK + buf * kKT * LD;
    for (int e = tid; e < Q * kKT; e += kAThreads) {
      const int i = e / kKT, j = e - i * kKT;
      const int t = t0 + j;
      float sc = -INFINITY;
      if (t < n_keys && t <= p0 + i) {
        const float* qr = sQ + i * D;
        const __nv_bfloat16* kr = kt + j * LD;
        float a = 0.f;
#pragma unroll 4
        for (int c = 0; c < D / 8; ++c) {
          float kf[8];
          unpack8(*reinterpret_cast<const bf16x8*>(kr + c * 8), kf);
          const float4 qa = *reinterpret_cast<const float4*>(qr + c * 8);
          const float4 qb = *reinterpret_cast<const float4*>(qr + c * 8 + 4);
          a = fmaf(qa.x, kf[0], a);
          a = fmaf(qa.y, kf[1], a);
          a = fmaf(qa.z, kf[2], a);
          a = fmaf(qa.w, kf[3], a);
          a = fmaf(qb.x, kf[4], a);
          a = fmaf(qb.y, kf[5], a);
          a = fmaf(qb.z, kf[6], a);
          a = fmaf(qb.w, kf[7], a);
        }
        sc = a;
      }
      sP[i * kKT + j] = sc;
    }
    __syncthreads();
    // online softmax per query (warp `i % 4`), 64 keys = 2 per lane
#pragma unroll
    for (int u = 0; u < QW; ++u) {
      const int i = warp + 4 * u;
      if (i < Q) {
        const float v0 = sP[i * kKT + lane], v1 = sP[i * kKT + lane + 32];
        const float mx = warp_max(fmaxf(v0, v1));
        const float mn = fmaxf(m_r[u], mx);
        float e0 = 0.f, e1 = 0.f, corr = 1.f;
        if (mn != -INFINITY) {
          e0 = __expf(v0 - mn);
          e1 = __expf(v1 - mn);
          corr = __expf(m_r[u] - mn);
        }
        l_r[u] = l_r[u] * corr + warp_sum(e0 + e1);
        m_r[u] = mn;
        sP[i * kKT + lane] = e0;
        sP[i * kKT + lane + 32] = e1;
        if (lane == 0) sCorr[i] = corr;
      }
    }
    __syncthreads();
    // P·V from shared memory
    const __nv_bfloat16* vt = sV + buf * kKT * LD;
    const int kmax = min(kKT, n_keys - t0);
#pragma unroll
    for (int u = 0; u < QT; ++u) {
      const int i = g + NG * u;
      if (i < Q) acc[u] *= sCorr[i];
    }
    for (int j = 0; j < kmax; ++j) {
      const float v = bf2f(vt[j * LD + d]);
#pragma unroll
      for (int u = 0; u < QT; ++u) {
        const int i = g + NG * u;
        if (i < Q) acc[u] = fmaf(sP[i * kKT + j], v, acc[u]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < QW; ++u) {
    const int i = warp + 4 * u;
    if (i < Q && lane == 0) sL[i] = l_r[u];
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < QT; ++u) {
    const int i = g + NG * u;
    if (i < Q) out[(int64_t)(b * Qtot + q0 + i) * ldo + h * D + d] = f2bf(acc[u] / sL[i]);
  }
}

template <int D, int QM>
static int launch_attn(const void* qkv, int64_t ldq, int B, int Q, int H, const int32_t* slot,
                       const int32_t* start, int T, void* kc, void* vc, float scale, int fuse,
                       void* out, int64_t ldo, cudaStream_t st) {
  using S = AttnSmem<D, QM>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attention_kernel<D, QM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             S::BYTES) != cudaSuccess)
      return MS_ERR_CUDA;
    attr = true;
  }
  dim3 grid(B, H, (Q + QM - 1) / QM);
  return launch(attention_kernel<D, QM>, grid, dim3(kAThreads), S::BYTES, st, 1,
                (const __nv_bfloat16*)qkv, ldq, Q, H, slot, start, T, (__nv_bfloat16*)kc,
                (__nv_bfloat16*)vc, scale, fuse, (__nv_bfloat16*)out, ldo);
}

template <int D>
static int attention_d(const void* qkv, int64_t ldq, int B, int Q, int H, const int32_t* slot,
                       const int32_t* start, int T, void* kc, void* vc, float scale, int fuse,
                       void* out, int64_t ldo, cudaStream_t st) {
  if (Q <= 1) return launch_attn<D, 1>(qkv, ldq, B, Q, H, slot, start, T, kc, vc, scale, fuse, out, ldo, st);
  if (Q <= 2) return launch_attn<D, 2>(qkv, ldq, B, Q, H, slot, start, T, kc, vc, scale, fuse, out, ldo, st);
  if (Q <= 4) return launch_attn<D, 4>(qkv, ldq, B, Q, H, slot, start, T, kc, vc, scale, fuse, out, ldo, st);
  if (Q <= 8) return launch_attn<D, 8>(qkv, ldq, B, Q, H, slot, start, T, kc, vc, scale, fuse, out, ldo, st);
  return launch_attn<D, 16>(qkv, ldq, B, Q, H, slot, start, T, kc, vc, scale, fuse, out, ldo, st);
}

}  // namespace ms

extern "C" int ms_kv_append(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                            const int32_t* slot, const int32_t* start, int T, void* k_cache,
                            void* v_cache, void* stream);

extern "C" int ms_attention(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                            const int32_t* slot, const int32_t* start, int T, void* k_cache,
                            void* v_cache, float scale, int append, void* out, int64_t ldo,
                            void* stream) {
  if (B < 0 || Q < 1 || H < 1 || T < 1) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache || !out) return MS_ERR_VALUE;
  if (ldq % 8) return MS_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  int fuse = 0;
  if (append) {
    if (Q <= 16) {
      fuse = 1;  // one query chunk per (request, head): append inside the kernel
    } else {
      const int s = ms_kv_append(qkv, ldq, B, Q, H, D, slot, start, T, k_cache, v_cache, stream);
      if (s != MS_OK) return s;
    }
  }
  if (D == 64)
    return ms::attention_d<64>(qkv, ldq, B, Q, H, slot, start, T, k_cache, v_cache, scale, fuse, out, ldo, st);
  if (D == 128)
    return ms::attention_d<128>(qkv, ldq, B, Q, H, slot, start, T, k_cache, v_cache, scale, fuse, out, ldo, st);
  return MS_ERR_UNSUPPORTED;
}
