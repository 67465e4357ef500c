// K2/K6 — KV-cache attention of Q consecutive query rows per request
// (Q = s+1 for the LLM verify forward, 1 for an SSM decode step, the catch-up
// length for an SSM's first step of a round), with the KV-cache append (K7)
// fused in.  Replaces the attention inside ModelOracle.next_dist
// (aggspec/oracles.py:19-26) for the draft (aggspec/oracles.py:148) and
// verify (aggspec/engine.py:294-296) positions.
//
// One CTA (4 warps) per (request, head[, 16-query chunk]).  The request's K
// and V streams [T, D] are staged through shared memory in tiles of 64 keys
// with cp.async double buffering (16-byte copies, all threads issuing), so
// each K/V byte is read from HBM once for all the queries of the request: the
// kernel is bound by the KV-cache stream.  The (<= 16 queries) x (64 keys)
// score tile and the P·V product run on warp-level tensor-core MMAs
// (mma.m16n8k16 bf16 -> fp32; decode has far too few query rows for a
// 128-row tcgen05 tile): warp w owns keys 16w..16w+15 of every tile, keeps
// its own online-softmax state and output accumulator in registers, and the
// 4 warps are merged in warp order at the end.
//
// Grouped-query attention (Llama-2-70B: 64 query heads over 8 KV heads): the
// CTA is per (request, KV head[, chunk]) and its MMA rows are the flattened
// (position i, query head j of the group) pairs, row = i * G + j, so every K/V
// byte of a KV head is staged once for all G·Q query rows that read it.  With
// a RoPE table (Llama) the Q fragments are rotated in registers (the
// rotate-half partner of dim d, d + D/2, sits in the same thread's fragment
// of chunk c + D/32) and the call's fresh K rows are rotated while staged and
// appended; cached K rows are stored rotated.
//
// Batch invariance: a query row's arithmetic (its MMA rows, per-row quad
// reductions, tile order, warp-order merge) does not depend on the other
// rows; rows of other queries only add fully-masked keys that contribute
// exactly zero.
#include <atomic>

#include "common.cuh"

namespace ms {

constexpr int kKT = 64;  // keys per tile (16 per warp)
constexpr int kAThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// D(16x8) += A(16x16, row) * B(16x8, col), bf16 in, fp32 accumulate
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}

// NBUF-deep cp.async ring of 64-key K/V tiles (launch_attn picks the depth)
template <int D, int NBUF = 2>
struct AttnSmem {
  static constexpr int LD = D + 8;  // padded rows: fragment loads are bank-conflict free
  static constexpr int TILE = kKT * LD;                  // elements per K (or V) tile
  static constexpr int KV_BYTES = 2 * NBUF * TILE * 2;   // [K|V][buf] bf16
  static constexpr int MERGE_BYTES = 4 * 16 * (D + 3) * 4 + 2 * 16 * 4;  // per-warp (m, l, O, f) + row (m, L)
  static constexpr int BYTES = KV_BYTES > MERGE_BYTES ? KV_BYTES : MERGE_BYTES;
};

__device__ __forceinline__ uint32_t rope_pair_lo(uint32_t x, uint32_t y, float2 c0, float2 c1) {
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x));
  const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&y));
  return pack_bf16(a.x * c0.x - p.x * c0.y, a.y * c1.x - p.y * c1.y);
}
__device__ __forceinline__ uint32_t rope_pair_hi(uint32_t x, uint32_t y, float2 c0, float2 c1) {
  // x: dims d + D/2 (own), y: dims d (partner)
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x));
  const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&y));
  return pack_bf16(a.x * c0.x + p.x * c0.y, a.y * c1.x + p.y * c1.y);
}

template <int D, int NBUF, bool PAGED>
__global__ void __launch_bounds__(kAThreads)
attention_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Qtot, int Hq, int Hkv,
                 const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                 __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, float scale_log2,
                 int fuse_append, const float2* __restrict__ rope, __nv_bfloat16* __restrict__ out,
                 int64_t ldo, int n_kv, int kct, float* __restrict__ ws, int* __restrict__ counters, KVPage pg) {
  using S = AttnSmem<D, NBUF>;
  constexpr int LD = S::LD;
  constexpr int KC = D / 16;  // 16-dim chunks (MMA k-steps for Q.K^T)
  constexpr int NT = D / 8;   // 8-dim output tiles for P.V
  extern __shared__ __align__(16) uint8_t smem[];
  // (the programmatic-dependency wait comes after the cache prefetch below)
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem);  // [2][KT][LD]
  __nv_bfloat16* sV = sK + NBUF * S::TILE;                        // [NBUF][KT][LD]

  const int b = blockIdx.x, h = blockIdx.y;  // h: KV head
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;  // mma fragment coordinates
  const int G = Hq / Hkv;                  // query heads per KV head
  const int rows_tot = Qtot * G;           // flattened (position, group head) rows
  // blockIdx.z = (query-row chunk of 16, KV chunk of kct tiles)
  const int qc = blockIdx.z / n_kv, kvc = blockIdx.z - qc * n_kv;
  const int nqc = gridDim.z / n_kv;
  const int q0 = qc * 16;                  // first flattened row of this chunk
  const int Q = min(16, rows_tot - q0);    // rows in this chunk
  const int pstart = start[b];
  const int kv_slot = slot[b];
  // K/V row t's element offset: contiguous [slots, Hkv, T, D], or through the
  // block table (PAGED, a separate instantiation so the contiguous path keeps
  // its single multiply-add)
  const int64_t cbase = ((int64_t)kv_slot * Hkv + h) * T * D;
  auto krow = [&](int t) -> int64_t {
    if constexpr (PAGED) {
      return kv_row(pg, kv_slot, Hkv, h, T, t) * D;
    } else {
      return cbase + (int64_t)t * D;
    }
  };
  const int QD = Hq * D, KVD = Hkv * D;
  constexpr int V8 = D / 8;

  const int last_pos = pstart + (q0 + Q - 1) / G;
  const int n_keys = min(last_pos + 1, T);  // keys 0 .. last position of the chunk
  const int n_tiles_all = (n_keys + kKT - 1) / kKT;
  // split-KV: this CTA owns tiles [tile0, tile1) — fixed 64*kct-key chunks
  // from position 0, so a query's partition never depends on the other rows
  const int n_chunks = (n_tiles_all + kct - 1) / kct;
  if (kvc >= n_chunks) {  // nothing for this request here (uniform per CTA)
    pdl_wait();
    return;
  }
  const int tile0 = kvc * kct;
  const int n_tiles = min(n_tiles_all, tile0 + kct);

  // tile loader: thread -> fixed 16-byte column chunk `lc` and rows lr0 + p*LRS
  // (no per-element index arithmetic); the call's own rows (t >= pstart) come
  // straight from qkv (K rotated on the way when RoPE), older keys from the cache
  constexpr int LRS = kAThreads / V8;  // rows per pass
  constexpr int LNP = kKT / LRS;       // passes per tile
  const int lc = tid % V8, lr0 = tid / V8;
  const __nv_bfloat16* qkv_k = qkv + (int64_t)(b * Qtot) * ldq + QD + h * D + lc * 8;
  const __nv_bfloat16* qkv_v = qkv_k + KVD;
  const int lpc = lc < V8 / 2 ? lc + V8 / 2 : lc - V8 / 2;  // RoPE partner chunk
  // part 0: the rows cached by earlier calls (t < pstart) as cp.async,
  // issued BEFORE the programmatic-dependency wait (they do not depend on the
  // previous kernel: the KV stream's first latency overlaps its tail); part 1:
  // the rest of the tile (the call's own rows from qkv — K rotated when RoPE —
  // or from the cache when the caller appended; zeros past the keys) as
  // synchronous stores after the wait; part 2: both (steady-state prefetch)
  auto load_tile = [&](int tile, int buf, int part) {
    const int t0 = tile * kKT;
    __nv_bfloat16* dk = sK + buf * S::TILE + lc * 8;
    __nv_bfloat16* dv = sV + buf * S::TILE + lc * 8;
#pragma unroll
    for (int pp = 0; pp < LNP; ++pp) {
      const int j = lr0 + pp * LRS;
      const int t = t0 + j;
      const bool cached = t < n_keys && t < pstart;
      if (part == 0) {
        if (cached) {
          cp_async16(dk + j * LD, kc + krow(t) + lc * 8);
          cp_async16(dv + j * LD, vc + krow(t) + lc * 8);
        }
        continue;
      }
      if (part == 1 && cached) continue;
      if (t < n_keys) {
        const bool fresh = fuse_append && t >= pstart;
        const int64_t qrow = (int64_t)(t - pstart) * ldq;
        if (fresh && rope) {
          float fv[8], pf[8];
          unpack8(*reinterpret_cast<const bf16x8*>(qkv_k + qrow), fv);
          unpack8(*reinterpret_cast<const bf16x8*>(qkv_k + qrow + (lpc - lc) * 8), pf);
          rope8(fv, pf, rope + (int64_t)t * (D / 2), lc * 8, D / 2);
          *reinterpret_cast<bf16x8*>(dk + j * LD) = pack8(fv);
        } else if (part == 1) {
          *reinterpret_cast<uint4*>(dk + j * LD) =
              *reinterpret_cast<const uint4*>(fresh ? qkv_k + qrow : kc + krow(t) + lc * 8);
        } else {
          cp_async16(dk + j * LD, fresh ? qkv_k + qrow : kc + krow(t) + lc * 8);
        }
        if (part == 1)
          *reinterpret_cast<uint4*>(dv + j * LD) =
              *reinterpret_cast<const uint4*>(fresh ? qkv_v + qrow : vc + krow(t) + lc * 8);
        else
          cp_async16(dv + j * LD, fresh ? qkv_v + qrow : vc + krow(t) + lc * 8);
      } else {  // masked keys must be finite
        *reinterpret_cast<uint4*>(dk + j * LD) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dv + j * LD) = make_uint4(0, 0, 0, 0);
      }
    }
    if (part != 1) cp_async_commit();
  };

  float m_r[2] = {-INFINITY, -INFINITY};  // rows g, g+8 (log2 domain)
  float l_r[2] = {0.f, 0.f};
  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;

#pragma unroll
  for (int pp = 0; pp < NBUF - 1; ++pp) {
    if (tile0 + pp < n_tiles) load_tile(tile0 + pp, pp, 0);
    else cp_async_commit();  // empty group: keeps the wait count uniform
  }
  pdl_wait();
  pdl_trigger();
  for (int pp = 0; pp < NBUF - 1 && tile0 + pp < n_tiles; ++pp) load_tile(tile0 + pp, pp, 1);
  if (fuse_append && kvc == 0 && qc == 0) {
    // this request's new K/V rows for KV head h -> cache (K rotated when
    // RoPE); this kernel reads them back from qkv, so no fence is needed
    for (int e = tid; e < 2 * Qtot * V8; e += kAThreads) {
      const int kv = e >= Qtot * V8;
      const int e2 = e - kv * Qtot * V8;
      const int i = e2 / V8, c = e2 - i * V8;
      const int p = pstart + i;
      if (p < 0 || p >= T) continue;
      const __nv_bfloat16* row = qkv + (int64_t)(b * Qtot + i) * ldq + QD + kv * KVD + h * D;
      bf16x8 val = *reinterpret_cast<const bf16x8*>(row + c * 8);
      if (!kv && rope) {
        const int pc = c < V8 / 2 ? c + V8 / 2 : c - V8 / 2;
        float fv[8], pf[8];
        unpack8(val, fv);
        unpack8(*reinterpret_cast<const bf16x8*>(row + pc * 8), pf);
        rope8(fv, pf, rope + (int64_t)p * (D / 2), c * 8, D / 2);
        val = pack8(fv);
      }
      *reinterpret_cast<bf16x8*>((kv ? vc : kc) + krow(p) + c * 8) = val;
    }
  }

  // Q fragments (rows g, g+8 of the 16-row tile; flattened row -> position
  // fr / G, query head h*G + fr % G); the softmax scale log2(e)/sqrt(D) is
  // applied to the fp32 scores
  const int fr0 = q0 + g, fr1 = q0 + g + 8;
  const int pos0 = pstart + fr0 / G, pos1 = pstart + fr1 / G;
  uint32_t qa[KC][4];
  {
    const bool v0 = g < Q, v1 = g + 8 < Q;
    const uint32_t* q0p = reinterpret_cast<const uint32_t*>(
        qkv + (int64_t)(b * Qtot + (v0 ? fr0 / G : 0)) * ldq + (h * G + fr0 % G) * D);
    const uint32_t* q1p = reinterpret_cast<const uint32_t*>(
        qkv + (int64_t)(b * Qtot + (v1 ? fr1 / G : 0)) * ldq + (h * G + fr1 % G) * D);
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const int w = c * 8 + t4;  // 32-bit word: dims 2*t4 .. 2*t4+1 of chunk c
      qa[c][0] = v0 ? q0p[w] : 0u;      // (row g,   k 2t..2t+1)
      qa[c][1] = v1 ? q1p[w] : 0u;      // (row g+8, k 2t..2t+1)
      qa[c][2] = v0 ? q0p[w + 4] : 0u;  // (row g,   k 2t+8..)
      qa[c][3] = v1 ? q1p[w + 4] : 0u;  // (row g+8, k 2t+8..)
    }
    if (rope) {
      // fragment word u of chunk c holds dims c*16 + (u >= 2 ? 8 : 0) + 2*t4 (+1)
      // of row g (u even) / g+8 (u odd); its partner is chunk c + KC/2
      const float2* cs0 = rope + (int64_t)(v0 ? pos0 : 0) * (D / 2);
      const float2* cs1 = rope + (int64_t)(v1 ? pos1 : 0) * (D / 2);
#pragma unroll
      for (int c = 0; c < KC / 2; ++c) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2* cs = (u & 1) ? cs1 : cs0;
          const int d = c * 16 + (u >= 2 ? 8 : 0) + 2 * t4;
          const float2 c0 = cs[d], c1 = cs[d + 1];
          const uint32_t lo = qa[c][u], hi = qa[c + KC / 2][u];
          qa[c][u] = rope_pair_lo(lo, hi, c0, c1);
          qa[c + KC / 2][u] = rope_pair_hi(hi, lo, c0, c1);
        }
      }
    }
  }
  const int row_lim0 = g < Q ? pos0 : -1;      // last key position row g may see
  const int row_lim1 = g + 8 < Q ? pos1 : -1;

  for (int tile = tile0; tile < n_tiles; ++tile) {
    const int it = tile - tile0;
    const int buf = it % NBUF;
    // refill the buffer the previous iteration consumed, NBUF-1 tiles ahead
    if (tile + NBUF - 1 < n_tiles) load_tile(tile + NBUF - 1, (it + NBUF - 1) % NBUF, 2);
    else cp_async_commit();
    cp_async_wait<NBUF - 1>();
    __syncthreads();
    const int kbase = tile * kKT + warp * 16;  // this warp's 16 keys
    const __nv_bfloat16* kt = sK + buf * S::TILE + (warp * 16) * LD;
    const __nv_bfloat16* vt = sV + buf * S::TILE + (warp * 16) * LD;
    // S = Q K^T for two 8-key n-tiles
    float s[2][4];
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
      const __nv_bfloat16* kr = kt + (n * 8 + g) * LD + 2 * t4;
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + c * 16);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + c * 16 + 8);
        mma16816(s[n], qa[c], b0, b1);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) s[n][e] *= scale_log2;
    }
    // causal / length mask, online softmax (rows g and g+8; the 4 lanes of a
    // quad hold a row's 16 keys)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < 2; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + n * 8 + 2 * t4 + (e & 1);
        const int lim = (e < 2) ? row_lim0 : row_lim1;
        if (key > lim || key >= n_keys) s[n][e] = -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], s[n][e]);
      }
    }
    float corr[2], psum[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r]);
      corr[r] = (mn == -INFINITY) ? 1.f : exp2f(m_r[r] - mn);
      m_r[r] = mn;
      psum[r] = 0.f;
    }
#pragma unroll
    for (int n = 0; n < 2; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const float p = (m_r[r] == -INFINITY || s[n][e] == -INFINITY) ? 0.f : exp2f(s[n][e] - m_r[r]);
        s[n][e] = p;
        psum[r] += p;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 1);
      psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 2);
      l_r[r] = l_r[r] * corr[r] + psum[r];
    }
    // P as the A operand straight from the score accumulators, split into
    // bf16 hi + lo parts (P = hi + lo to ~2^-16) so P.V keeps fp32-like accuracy
    uint32_t pa[4], pl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float x0 = s[u >> 1][2 * (u & 1)], x1 = s[u >> 1][2 * (u & 1) + 1];
      const __nv_bfloat162 hi = __floats2bfloat162_rn(x0, x1);
      const float2 hf = __bfloat1622float2(hi);
      pa[u] = *reinterpret_cast<const uint32_t*>(&hi);
      pl[u] = pack_bf16(x0 - hf.x, x1 - hf.y);
    }
    // O = O * corr + P V   (V fragments via ldmatrix.trans, two 8-dim tiles per load)
    const int lrow = lane & 15;              // key row within the warp's 16
    const int lcol = (lane >> 4) * 8;        // dim offset 0 / 8 within a 16-dim pair
#pragma unroll
    for (int n2 = 0; n2 < NT / 2; ++n2) {
      uint32_t vb[4];
      ldmatrix_x4_trans(vb, vt + lrow * LD + n2 * 16 + lcol);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        float* on = o[2 * n2 + u];
        on[0] *= corr[0];
        on[1] *= corr[0];
        on[2] *= corr[1];
        on[3] *= corr[1];
        mma16816(o[2 * n2 + u], pa, vb[2 * u], vb[2 * u + 1]);
        mma16816(o[2 * n2 + u], pl, vb[2 * u], vb[2 * u + 1]);
      }
    }
    __syncthreads();
  }
  // merge the 4 warps' (m, l, O) in warp order
  float* sm = reinterpret_cast<float*>(smem);  // [4][16] m, [4][16] l, [4][16][D] O, [4][16] f, [16] m, [16] L
  float* sl = sm + 4 * 16;
  float* so = sl + 4 * 16;
  float* sf = so + 4 * 16 * D;  // per-(warp, row) merge factor
  float* rm = sf + 4 * 16;      // per-row max
  float* rL = rm + 16;          // per-row sum
  if (t4 == 0) {
    sm[warp * 16 + g] = m_r[0];
    sm[warp * 16 + g + 8] = m_r[1];
    sl[warp * 16 + g] = l_r[0];
    sl[warp * 16 + g + 8] = l_r[1];
  }
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int c = n * 8 + 2 * t4;
    so[(warp * 16 + g) * D + c] = o[n][0];
    so[(warp * 16 + g) * D + c + 1] = o[n][1];
    so[(warp * 16 + g + 8) * D + c] = o[n][2];
    so[(warp * 16 + g + 8) * D + c + 1] = o[n][3];
  }
  __syncthreads();
  // per-row merge factors, once per row: f_w = exp2(m_w - m) / L (the 4 warps'
  // softmax states combined in warp order)
  if (tid < 16) {
    const int i = tid;
    float mxx = sm[i];
#pragma unroll
    for (int w = 1; w < 4; ++w) mxx = fmaxf(mxx, sm[w * 16 + i]);
    float fw[4], L = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = sm[w * 16 + i];
      fw[w] = mw == -INFINITY ? 0.f : exp2f(mw - mxx);
      L += sl[w * 16 + i] * fw[w];
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) sf[w * 16 + i] = fw[w] * inv;
    rm[i] = mxx;
    rL[i] = L;
  }
  __syncthreads();
  // this CTA's partial: (m, L, O = A / L) per query row.  With a workspace the
  // chunk merge below runs even for a single chunk, so a query's output goes
  // through the same arithmetic whatever the other rows' key counts are.
  if (ws == nullptr) {
    for (int e = tid; e < Q * D; e += kAThreads) {
      const int i = e / D, dd = e - i * D;
      float A = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) A += so[(w * 16 + i) * D + dd] * sf[w * 16 + i];
      const int fr = q0 + i;
      out[(int64_t)(b * Qtot + fr / G) * ldo + (h * G + fr % G) * D + dd] = f2bf(A);
    }
    return;
  }
  constexpr int PS = 16 * (D + 2);  // partial record: m[16], L[16], O[16][D]
  const int64_t unit = ((int64_t)b * Hkv + h) * nqc + qc;
  float* rec = ws + (unit * n_kv + kvc) * PS;
  for (int e = tid; e < 16 * D; e += kAThreads) {
    const int i = e / D, dd = e - i * D;
    float A = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) A += so[(w * 16 + i) * D + dd] * sf[w * 16 + i];
    __stcg(rec + 32 + e, A);
    if (dd == 0) {
      __stcg(rec + i, rm[i]);
      __stcg(rec + 16 + i, rL[i]);
    }
  }
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  if (tid == 0) {
    const int old = atomicAdd(counters + unit, 1);
    s_last = old == n_chunks - 1;
    if (s_last) counters[unit] = 0;  // leave zero for the next launch
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last chunk to finish merges all chunks in chunk order (deterministic)
  const float* recs = ws + unit * n_kv * PS;
  for (int e = tid; e < Q * D; e += kAThreads) {
    const int i = e / D;
    float mxx = -INFINITY;
    for (int cc = 0; cc < n_chunks; ++cc) mxx = fmaxf(mxx, __ldcg(recs + cc * PS + i));
    float L = 0.f, A = 0.f;
    for (int cc = 0; cc < n_chunks; ++cc) {
      const float mc = __ldcg(recs + cc * PS + i);
      const float wgt = mc == -INFINITY ? 0.f : __ldcg(recs + cc * PS + 16 + i) * exp2f(mc - mxx);
      L += wgt;
      A += wgt * __ldcg(recs + cc * PS + 32 + e);
    }
    const int fr = q0 + i;
    out[(int64_t)(b * Qtot + fr / G) * ldo + (h * G + fr % G) * D + (e - i * D)] = f2bf(A / L);
  }
}


// ---------------------------------------------------------------------------
// Row-split schedule for grouped-query attention (G = H / Hkv > 1, e.g.
// Llama-2-70B's 8 query heads per KV head): one CTA per (request, KV head, 96
// flattened (position, group head) rows), 12 warps = 6 row warps x 2 key
// groups.  Row warp r owns rows 16r..16r+15; key group j takes the 32-key
// tiles t with t % 2 == j, so each round stages 64 keys once for all of the
// KV head's query rows and the two groups' online softmax states are merged
// once at the end (group 0 then group 1).  The query tile (RoPE applied) sits
// in shared memory, so a thread holds little more than its O accumulator.
// One CTA per SM covers a verify of up to 12 positions.  (The previous one-group schedule —
// 4 warps, 180 registers, 64-key tiles walked serially — was issue-latency
// bound: one warp per scheduler, 0.6-1 TB/s at every context.)
// The schedule is fixed by G alone (never by Q or the cache length), so a
// row's arithmetic is the same in a Q=1 decode and a Q=s+1 verify (batch
// invariance: tiles beyond a row's keys are exact no-ops, and the key-group
// merge always runs).
// ---------------------------------------------------------------------------
constexpr int kRW = 6;                 // row warps: 96 flattened rows per CTA (Q <= 12 at G = 8)
constexpr int kRRows = 16 * kRW;
constexpr int kRThreads = 2 * 32 * kRW;  // row warps x 2 key groups
constexpr int kRKT = 32;               // keys per tile; a round = one tile per key group
// round buffers: NR-1 rounds (64 keys each) in flight ahead of the one being
// computed — a ~200-key verify context is fetched in one DRAM latency, and a
// long context keeps ~100 KB in flight per SM (registers already hold the
// CTA to one per SM, so the shared memory is free)
constexpr int kRNR = 4;
#ifndef MS_ATTN_PLO
#define MS_ATTN_PLO 0
#endif

template <int D>
struct RowsSmem {
  static constexpr int LD = D + 8;             // padded rows: conflict-free ldmatrix
  static constexpr int TILE = kRKT * LD;       // elements per K (or V) tile
  static constexpr int Q_ELEMS = kRRows * LD;  // the CTA's query rows
  static constexpr int KV_ELEMS = kRNR * 2 * 2 * TILE;  // [round buf][key group][K|V]
  static constexpr int MERGE_BYTES = kRW * 16 * (D + 2) * 4;  // key group 1's (O, m, l) per row
  static constexpr int KV_BYTES = KV_ELEMS * 2 > MERGE_BYTES ? KV_ELEMS * 2 : MERGE_BYTES;
  static constexpr int BYTES = Q_ELEMS * 2 + KV_BYTES;
};

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}

template <int D, bool PAGED>
__global__ void __launch_bounds__(kRThreads, 1)
attention_rows_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Qtot, int Hq, int Hkv,
                      const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                      __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, float scale_log2,
                      int fuse_append, const float2* __restrict__ rope, __nv_bfloat16* __restrict__ out,
                      int64_t ldo, int n_kv, int kct, float* __restrict__ ws, int* __restrict__ counters,
                      KVPage pg) {
  using S = RowsSmem<D>;
  constexpr int LD = S::LD;
  constexpr int KC = D / 16;
  constexpr int NT = D / 8;
  constexpr int V8 = D / 8;
  extern __shared__ __align__(16) uint8_t smem[];
  // (the programmatic-dependency wait comes after the cache prefetch below)
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem);  // [kRRows][LD]
  __nv_bfloat16* sKV = sQ + S::Q_ELEMS;                          // [kRNR][2][K|V][kRKT][LD]

  const int b = blockIdx.x, h = blockIdx.y;  // h: KV head
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rw = warp % kRW, kg = warp / kRW;  // row warp, key group
  const int g = lane >> 2, t4 = lane & 3;
  const int G = Hq / Hkv;
  const int rows_tot = Qtot * G;
  // blockIdx.z = (row chunk zr, cache-length chunk kvc of kct 64-key rounds)
  const int zr = blockIdx.z / n_kv, kvc = blockIdx.z - zr * n_kv;
  const int c0 = zr * kRRows;                 // first flattened row of the CTA
  const int crows = min(kRRows, rows_tot - c0);
  const int q0 = c0 + rw * 16;                // first row of this warp
  const int Q = max(0, min(16, rows_tot - q0));  // rows of this warp (0: idle)
  const int pstart = start[b];
  const int kv_slot = slot[b];
  // K/V row t's element offset: contiguous [slots, Hkv, T, D], or through the
  // block table (PAGED, a separate instantiation so the contiguous path keeps
  // its single multiply-add)
  const int64_t cbase = ((int64_t)kv_slot * Hkv + h) * T * D;
  auto krow = [&](int t) -> int64_t {
    if constexpr (PAGED) {
      return kv_row(pg, kv_slot, Hkv, h, T, t) * D;
    } else {
      return cbase + (int64_t)t * D;
    }
  };
  const int QD = Hq * D, KVD = Hkv * D;

  // keys 0 .. the CTA's last position; split over the cache length: this CTA
  // owns rounds [r0, r0 + kct) — fixed chunks from position 0, so a row's
  // partition never depends on the other rows
  const int n_keys = min(pstart + (c0 + crows - 1) / G + 1, T);
  const int n_rounds_all = (n_keys + 2 * kRKT - 1) / (2 * kRKT);
  const int n_chunks = (n_rounds_all + kct - 1) / kct;
  if (kvc >= n_chunks) {  // uniform per CTA (the unit's arrival count excludes it)
    pdl_wait();
    return;
  }
  const int r0 = kvc * kct;
  const int n_rounds = min(n_rounds_all, r0 + kct) - r0;

  constexpr int LRS = kRThreads / V8;   // key rows per pass
  const int lc = tid % V8, lr0 = tid / V8;
  const __nv_bfloat16* qkv_k = qkv + (int64_t)(b * Qtot) * ldq + QD + h * D + lc * 8;
  const __nv_bfloat16* qkv_v = qkv_k + KVD;
  const int lpc = lc < V8 / 2 ? lc + V8 / 2 : lc - V8 / 2;
  // round rd = keys 64rd .. 64rd+63: tile 2rd (key group 0), tile 2rd+1 (group 1).
  // part 0: the rows cached by earlier calls (t < pstart) as cp.async — they
  //         do not depend on the previous kernel, so the first rounds are
  //         requested BEFORE the programmatic-dependency wait (the KV stream's
  //         first DRAM latency overlaps the QKV GEMM's tail);
  // part 1: the rest of the round (the call's own rows, straight from qkv with
  //         K rotated when RoPE, or from the cache when the caller appended;
  //         zeros past the keys), synchronous stores, after the wait;
  // part 2: both, as cp.async where possible (the steady-state prefetch).
  auto load_round = [&](int rd, int rb, int part) {
    const int t0 = rd * 2 * kRKT;
    for (int j = lr0; j < 2 * kRKT; j += LRS) {
      const int t = t0 + j;
      __nv_bfloat16* dk = sKV + ((rb * 2 + j / kRKT) * 2) * S::TILE + (j % kRKT) * LD + lc * 8;
      __nv_bfloat16* dv = dk + S::TILE;
      const bool cached = t < n_keys && t < pstart;
      if (part == 0) {
        if (cached) {
          cp_async16(dk, kc + krow(t) + lc * 8);
          cp_async16(dv, vc + krow(t) + lc * 8);
        }
        continue;
      }
      if (part == 1 && cached) continue;
      if (t < n_keys) {
        const bool fresh = fuse_append && t >= pstart;
        const int64_t qrow = (int64_t)(t - pstart) * ldq;
        if (fresh && rope) {
          float fv[8], pf[8];
          unpack8(*reinterpret_cast<const bf16x8*>(qkv_k + qrow), fv);
          unpack8(*reinterpret_cast<const bf16x8*>(qkv_k + qrow + (lpc - lc) * 8), pf);
          rope8(fv, pf, rope + (int64_t)t * (D / 2), lc * 8, D / 2);
          *reinterpret_cast<bf16x8*>(dk) = pack8(fv);
        } else if (part == 1) {
          *reinterpret_cast<uint4*>(dk) = *reinterpret_cast<const uint4*>(fresh ? qkv_k + qrow : kc + krow(t) + lc * 8);
        } else {
          cp_async16(dk, fresh ? qkv_k + qrow : kc + krow(t) + lc * 8);
        }
        if (part == 1)
          *reinterpret_cast<uint4*>(dv) = *reinterpret_cast<const uint4*>(fresh ? qkv_v + qrow : vc + krow(t) + lc * 8);
        else
          cp_async16(dv, fresh ? qkv_v + qrow : vc + krow(t) + lc * 8);
      } else {
        *reinterpret_cast<uint4*>(dk) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dv) = make_uint4(0, 0, 0, 0);
      }
    }
    if (part != 1) cp_async_commit();
  };
#pragma unroll
  for (int pp = 0; pp < kRNR - 1; ++pp) {
    if (pp < n_rounds) load_round(r0 + pp, pp, 0);
    else cp_async_commit();  // empty group: keeps the wait count uniform
  }
  pdl_wait();
  pdl_trigger();
  for (int pp = 0; pp < kRNR - 1 && pp < n_rounds; ++pp) load_round(r0 + pp, pp, 1);

  if (fuse_append && zr == 0 && kvc == 0) {
    for (int e = tid; e < 2 * Qtot * V8; e += kRThreads) {
      const int kv = e >= Qtot * V8;
      const int e2 = e - kv * Qtot * V8;
      const int i = e2 / V8, c = e2 - i * V8;
      const int p = pstart + i;
      if (p < 0 || p >= T) continue;
      const __nv_bfloat16* row = qkv + (int64_t)(b * Qtot + i) * ldq + QD + kv * KVD + h * D;
      bf16x8 val = *reinterpret_cast<const bf16x8*>(row + c * 8);
      if (!kv && rope) {
        const int pc = c < V8 / 2 ? c + V8 / 2 : c - V8 / 2;
        float fv[8], pf[8];
        unpack8(val, fv);
        unpack8(*reinterpret_cast<const bf16x8*>(row + pc * 8), pf);
        rope8(fv, pf, rope + (int64_t)p * (D / 2), c * 8, D / 2);
        val = pack8(fv);
      }
      *reinterpret_cast<bf16x8*>((kv ? vc : kc) + krow(p) + c * 8) = val;
    }
  }

  // the CTA's query rows -> shared memory (row r = flattened row c0 + r:
  // position r / G, query head h*G + r % G), RoPE on 32-bit words (dims 2w,
  // 2w+1 paired with 2w+D/2, 2w+D/2+1); rows past the call are zero
  for (int e = tid; e < kRRows * (D / 4); e += kRThreads) {
    const int r = e / (D / 4), w = e - r * (D / 4);
    const int fr = c0 + r;
    uint32_t lo = 0u, hi = 0u;
    if (fr < rows_tot) {
      const uint32_t* qp =
          reinterpret_cast<const uint32_t*>(qkv + (int64_t)(b * Qtot + fr / G) * ldq + (h * G + fr % G) * D);
      lo = qp[w];
      hi = qp[w + D / 4];
      if (rope) {
        const float2* cs = rope + (int64_t)(pstart + fr / G) * (D / 2);
        const float2 cc0 = cs[2 * w], cc1 = cs[2 * w + 1];
        const uint32_t l2 = rope_pair_lo(lo, hi, cc0, cc1);
        hi = rope_pair_hi(hi, lo, cc0, cc1);
        lo = l2;
      }
    }
    uint32_t* qs = reinterpret_cast<uint32_t*>(sQ + r * LD);
    qs[w] = lo;
    qs[w + D / 4] = hi;
  }

  const int fr0 = q0 + g, fr1 = q0 + g + 8;
  const bool v0 = g < Q, v1 = g + 8 < Q;
  const int pos0 = pstart + fr0 / G, pos1 = pstart + fr1 / G;
  // keys every valid row of this warp sees (the warp's first row has the
  // smallest position): tiles below it need no causal mask
  const int warp_lim = pstart + q0 / G;

  float m_r[2] = {-INFINITY, -INFINITY};
  float l_r[2] = {0.f, 0.f};
  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  const int row_lim0 = v0 ? pos0 : -1;
  const int row_lim1 = v1 ? pos1 : -1;
  const int lrow = lane & 15;
  const int lcol = (lane >> 4) * 8;
  const __nv_bfloat16* qw = sQ + (rw * 16 + lrow) * LD + lcol;  // this lane's ldmatrix row

  for (int rd = 0; rd < n_rounds; ++rd) {
    const int rb = rd % kRNR;
    if (rd + kRNR - 1 < n_rounds) load_round(r0 + rd + kRNR - 1, (rd + kRNR - 1) % kRNR, 2);
    else cp_async_commit();
    cp_async_wait<kRNR - 1>();
    __syncthreads();  // (first round: also the query tile)
    const int kbase = ((r0 + rd) * 2 + kg) * kRKT;
    if (Q > 0 && kbase < n_keys) {  // warp-uniform
      const __nv_bfloat16* kt = sKV + ((rb * 2 + kg) * 2) * S::TILE;
      const __nv_bfloat16* vt = kt + S::TILE;
      float sc[4][4];
#pragma unroll
      for (int n = 0; n < 4; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
      for (int c = 0; c < KC; c += 2) {
        uint32_t qa0[4], qa1[4];
        ldmatrix_x4(qa0, qw + c * 16);
        ldmatrix_x4(qa1, qw + (c + 1) * 16);
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          uint32_t kb[4];  // keys n*8..n*8+7, dims c*16 .. c*16+31
          ldmatrix_x4(kb, kt + (n * 8 + (lane & 7)) * LD + c * 16 + (lane >> 3) * 8);
          mma16816(sc[n], qa0, kb[0], kb[1]);
          mma16816(sc[n], qa1, kb[2], kb[3]);
        }
      }
      float mx[2] = {-INFINITY, -INFINITY};
      if (kbase + kRKT - 1 <= warp_lim && kbase + kRKT <= n_keys) {
        // every key of the tile is visible to every valid row of the warp
        // (invalid rows carry zero queries and are never stored)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            sc[n][e] *= scale_log2;
            mx[e >> 1] = fmaxf(mx[e >> 1], sc[n][e]);
          }
      } else {
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = kbase + n * 8 + 2 * t4 + (e & 1);
            const int lim = (e < 2) ? row_lim0 : row_lim1;
            float v = sc[n][e] * scale_log2;
            if (key > lim || key >= n_keys) v = -INFINITY;
            sc[n][e] = v;
            mx[e >> 1] = fmaxf(mx[e >> 1], v);
          }
      }
      float corr[2], psum[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        const float mn = fmaxf(m_r[r], mx[r]);
        corr[r] = (mn == -INFINITY) ? 1.f : exp2f(m_r[r] - mn);
        m_r[r] = mn;
        psum[r] = 0.f;
      }
#pragma unroll
      for (int n = 0; n < 4; ++n) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = e >> 1;
          const float pv = (m_r[r] == -INFINITY || sc[n][e] == -INFINITY) ? 0.f : exp2f(sc[n][e] - m_r[r]);
          sc[n][e] = pv;
          psum[r] += pv;
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 1);
        psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 2);
        l_r[r] = l_r[r] * corr[r] + psum[r];
      }
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        o[n][0] *= corr[0];
        o[n][1] *= corr[0];
        o[n][2] *= corr[1];
        o[n][3] *= corr[1];
      }
      // O += P V over the tile's two 16-key blocks: P as bf16 (its fp32 row
      // sum is the normaliser), as flash-attention kernels do; MS_ATTN_PLO=1
      // adds the bf16 remainder P - bf16(P) as a second MMA (~fp32 P, 1.5x the
      // tensor work of this compute-latency-bound loop)
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        uint32_t pa[4];
#if MS_ATTN_PLO
        uint32_t pl[4];
#endif
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float x0 = sc[2 * kb + (u >> 1)][2 * (u & 1)], x1 = sc[2 * kb + (u >> 1)][2 * (u & 1) + 1];
          const __nv_bfloat162 hi = __floats2bfloat162_rn(x0, x1);
          pa[u] = *reinterpret_cast<const uint32_t*>(&hi);
#if MS_ATTN_PLO
          const float2 hf = __bfloat1622float2(hi);
          pl[u] = pack_bf16(x0 - hf.x, x1 - hf.y);
#endif
        }
#pragma unroll
        for (int n2 = 0; n2 < NT / 2; ++n2) {
          uint32_t vb[4];
          ldmatrix_x4_trans(vb, vt + (kb * 16 + lrow) * LD + n2 * 16 + lcol);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            mma16816(o[2 * n2 + u], pa, vb[2 * u], vb[2 * u + 1]);
#if MS_ATTN_PLO
            mma16816(o[2 * n2 + u], pl, vb[2 * u], vb[2 * u + 1]);
#endif
          }
        }
      }
    }
    __syncthreads();  // the round buffer is refilled by the next iteration's prefetch
  }
  cp_async_wait<0>();
  __syncthreads();
  // key group 1 hands its (O, m, l) to group 0 through the idle KV buffers;
  // group 0 merges (group 0 first, always — also when group 1 saw no key)
  float* mg = reinterpret_cast<float*>(sKV) + rw * 16 * (D + 2);
  if (kg == 1 && Q > 0) {
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int col = n * 8 + 2 * t4;
      *reinterpret_cast<float2*>(mg + g * (D + 2) + col) = make_float2(o[n][0], o[n][1]);
      *reinterpret_cast<float2*>(mg + (g + 8) * (D + 2) + col) = make_float2(o[n][2], o[n][3]);
    }
    if (t4 == 0) {
      mg[g * (D + 2) + D] = m_r[0];
      mg[g * (D + 2) + D + 1] = l_r[0];
      mg[(g + 8) * (D + 2) + D] = m_r[1];
      mg[(g + 8) * (D + 2) + D + 1] = l_r[1];
    }
  }
  __syncthreads();
  float f0[2] = {0.f, 0.f}, f1[2] = {0.f, 0.f}, Lr[2] = {0.f, 0.f}, mr2[2] = {-INFINITY, -INFINITY};
  if (kg == 0 && Q > 0) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float* mr = mg + (g + 8 * r) * (D + 2);
      const float m1 = mr[D], l1 = mr[D + 1];
      const float m = fmaxf(m_r[r], m1);
      const float a0 = m_r[r] == -INFINITY ? 0.f : exp2f(m_r[r] - m);
      const float a1 = m1 == -INFINITY ? 0.f : exp2f(m1 - m);
      const float L = l_r[r] * a0 + l1 * a1;
      const float inv = L > 0.f ? 1.f / L : 0.f;
      f0[r] = a0 * inv;
      f1[r] = a1 * inv;
      Lr[r] = L;
      mr2[r] = m;
    }
  }
  if (ws == nullptr) {
    if (kg == 1 || Q == 0) return;
    __nv_bfloat16* o0p = out + (int64_t)(b * Qtot + (v0 ? fr0 / G : 0)) * ldo + (h * G + (v0 ? fr0 % G : 0)) * D;
    __nv_bfloat16* o1p = out + (int64_t)(b * Qtot + (v1 ? fr1 / G : 0)) * ldo + (h * G + (v1 ? fr1 % G : 0)) * D;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int col = n * 8 + 2 * t4;
      const float2 p0 = *reinterpret_cast<const float2*>(mg + g * (D + 2) + col);
      const float2 p1 = *reinterpret_cast<const float2*>(mg + (g + 8) * (D + 2) + col);
      if (v0) *reinterpret_cast<uint32_t*>(o0p + col) =
          pack_bf16(o[n][0] * f0[0] + p0.x * f1[0], o[n][1] * f0[0] + p0.y * f1[0]);
      if (v1) *reinterpret_cast<uint32_t*>(o1p + col) =
          pack_bf16(o[n][2] * f0[1] + p1.x * f1[1], o[n][3] * f0[1] + p1.y * f1[1]);
    }
    return;
  }
  // split over the cache length: this chunk's record (m, L, A = O / L per
  // row); with a workspace the chunk merge runs even for one chunk, so a
  // row's output goes through the same arithmetic whatever its key count
  constexpr int PS = kRRows * (D + 2);
  const int nzr = gridDim.z / n_kv;
  const int64_t unit = ((int64_t)b * Hkv + h) * nzr + zr;
  float* rec = ws + (unit * n_kv + kvc) * PS;
  if (kg == 0 && Q > 0) {
    const int lr0 = rw * 16 + g, lr1 = lr0 + 8;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int col = n * 8 + 2 * t4;
      const float2 p0 = *reinterpret_cast<const float2*>(mg + g * (D + 2) + col);
      const float2 p1 = *reinterpret_cast<const float2*>(mg + (g + 8) * (D + 2) + col);
      __stcg(reinterpret_cast<float2*>(rec + 2 * kRRows + lr0 * D + col),
             make_float2(o[n][0] * f0[0] + p0.x * f1[0], o[n][1] * f0[0] + p0.y * f1[0]));
      __stcg(reinterpret_cast<float2*>(rec + 2 * kRRows + lr1 * D + col),
             make_float2(o[n][2] * f0[1] + p1.x * f1[1], o[n][3] * f0[1] + p1.y * f1[1]));
    }
    if (t4 == 0) {
      __stcg(rec + lr0, mr2[0]);
      __stcg(rec + lr1, mr2[1]);
      __stcg(rec + kRRows + lr0, Lr[0]);
      __stcg(rec + kRRows + lr1, Lr[1]);
    }
  }
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  if (tid == 0) {
    const int old = atomicAdd(counters + unit, 1);
    s_last = old == n_chunks - 1;
    if (s_last) counters[unit] = 0;  // zero for the next launch
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last chunk to finish merges all chunks in chunk order (deterministic):
  // per-(chunk, row) weights L_c * 2^(m_c - max) and 1 / sum in shared memory
  const float* recs = ws + unit * n_kv * PS;
  float* wsm = reinterpret_cast<float*>(sKV);  // [8][kRRows] weights, [kRRows] 1 / sum
  for (int r = tid; r < crows; r += kRThreads) {
    float mx = -INFINITY;
    for (int cc = 0; cc < n_chunks; ++cc) mx = fmaxf(mx, __ldcg(recs + cc * PS + r));
    float L = 0.f;
    for (int cc = 0; cc < n_chunks; ++cc) {
      const float mc = __ldcg(recs + cc * PS + r);
      const float wgt = mc == -INFINITY ? 0.f : __ldcg(recs + cc * PS + kRRows + r) * exp2f(mc - mx);
      wsm[cc * kRRows + r] = wgt;
      L += wgt;
    }
    wsm[8 * kRRows + r] = L > 0.f ? 1.f / L : 0.f;
  }
  __syncthreads();
  for (int e = tid; e < crows * (D / 2); e += kRThreads) {
    const int r = e / (D / 2), d2 = (e - r * (D / 2)) * 2;
    float ax = 0.f, ay = 0.f;
    for (int cc = 0; cc < n_chunks; ++cc) {
      const float wgt = wsm[cc * kRRows + r];
      const float2 v = __ldcg(reinterpret_cast<const float2*>(recs + cc * PS + 2 * kRRows + r * D + d2));
      ax += wgt * v.x;
      ay += wgt * v.y;
    }
    const float inv = wsm[8 * kRRows + r];
    const int fr = c0 + r;
    *reinterpret_cast<uint32_t*>(out + (int64_t)(b * Qtot + fr / G) * ldo + (h * G + fr % G) * D + d2) =
        pack_bf16(ax * inv, ay * inv);
  }
}

// KV chunk (in 64-key tiles) per CTA for the split-KV schedule: a function of
// the cache length T only (at most 8 chunks, at least 2 tiles each), so the
// partition never depends on the batch or on Q.
__host__ __device__ inline int kv_chunk_tiles(int T) {
  const int tiles = (T + kKT - 1) / kKT;
  const int c = (tiles + 7) / 8;
  return c < 2 ? 2 : c;
}

template <int D>
static int launch_attn(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, const int32_t* slot,
                       const int32_t* start, int T, void* kc, void* vc, const float2* rope, float scale,
                       int fuse, void* out, int64_t ldo, float* ws, int64_t ws_bytes, int* counters,
                       int n_counters, cudaStream_t st, KVPage pg) {
  // ring depth 2: deeper rings (3-4) measured slower — the extra shared
  // memory costs more resident CTAs than the hidden tile latency gains
  // (Llama-160M B=48 decode attention 13.8 -> 16 us, 70B verify 2.0 -> 3.0 ms)
  constexpr int NB = 2;
  using S = AttnSmem<D, NB>;
  using SR = RowsSmem<D>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attention_kernel<D, NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             S::BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(attention_kernel<D, NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             S::BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(attention_rows_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SR::BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(attention_rows_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SR::BYTES) != cudaSuccess)
      return MS_ERR_CUDA;
    attr = true;
  }
  const bool paged = pg.table != nullptr;
  const float scale_log2 = scale * 1.4426950408889634f;
  if (Hkv < H) {  // grouped-query: row-split schedule (chosen by G, never by Q)
    const int nzr = (Q * (H / Hkv) + kRRows - 1) / kRRows;
    int n_kvr = 1, kctr = (T + kKT - 1) / kKT;  // default: one CTA walks all its rounds
    if (ws) {  // split over the cache length: chunks of kv_chunk_tiles(T) 64-key rounds
      kctr = kv_chunk_tiles(T);
      n_kvr = ((T + kKT - 1) / kKT + kctr - 1) / kctr;
      const int64_t need = (int64_t)B * Hkv * nzr * n_kvr * kRRows * (D + 2) * 4;
      if (ws_bytes < need || n_counters < B * Hkv * nzr) return MS_ERR_VALUE;
    }
    dim3 grid(B, Hkv, nzr * n_kvr);
    return launch(paged ? attention_rows_kernel<D, true> : attention_rows_kernel<D, false>, grid,
                  dim3(kRThreads), SR::BYTES, st, 1, (const __nv_bfloat16*)qkv, ldq, Q, H, Hkv, slot, start, T,
                  (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, scale_log2, fuse, rope, (__nv_bfloat16*)out, ldo, n_kvr,
                  kctr, ws, counters, pg);
  }
  const int nqc = (Q * (H / Hkv) + 15) / 16;
  int n_kv = 1, kct = (T + kKT - 1) / kKT;  // default: one CTA walks all its keys
  if (ws) {
    kct = kv_chunk_tiles(T);
    n_kv = ((T + kKT - 1) / kKT + kct - 1) / kct;
    const int64_t need = (int64_t)B * Hkv * nqc * n_kv * 16 * (D + 2) * 4;
    if (ws_bytes < need || n_counters < B * Hkv * nqc) return MS_ERR_VALUE;
  }
  dim3 grid(B, Hkv, nqc * n_kv);
  return launch(paged ? attention_kernel<D, NB, true> : attention_kernel<D, NB, false>, grid, dim3(kAThreads),
                S::BYTES, st, 1, (const __nv_bfloat16*)qkv, ldq, Q, H, Hkv, slot, start, T, (__nv_bfloat16*)kc,
                (__nv_bfloat16*)vc, scale_log2, fuse, rope, (__nv_bfloat16*)out, ldo, n_kv, kct, ws,
                counters, pg);
}

// ---------------------------------------------------------------------------
// Co-resident decode attention (drafters' decode steps beside the verifier,
// ms_set_coresident): one query row per request (Q = 1), MHA, contiguous cache.
// One warp per (request, head), 2 warps (64 threads, <= 128 registers, no
// shared memory) per CTA — a CTA fits beside two verify-GEMM CTAs on an SM
// (2 x 224 threads x 128 registers + 64 x 128 = the 64K register file; the
// GEMMs leave ~17 KB of shared memory), so drafting no longer waits for GEMM
// CTAs to retire nor blocks the next one.  Lanes form groups of D/8 (one
// 16-byte chunk of a key row each): a warp streams 32 / (D/8) keys per step,
// each group keeps its own online softmax over its keys, the groups merge in
// a fixed shuffle tree at the end (deterministic; fp32 P.V).  The cached keys
// of the first steps are requested before the programmatic-dependency wait.
template <int D>
__global__ void __launch_bounds__(64, 8)
attention_decode_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int B, int H,
                        const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                        __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, float scale_log2,
                        int fuse_append, const float2* __restrict__ rope, __nv_bfloat16* __restrict__ out,
                        int64_t ldo) {
  constexpr int LPK = D / 8;    // lanes per key row
  constexpr int KPI = 32 / LPK;  // keys per warp step
  constexpr int U = 4;           // warp steps in flight
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x * 2 + warp;
  const bool live = pair < B * H;
  const int b = live ? pair / H : 0, h = live ? pair % H : 0;
  const int sub = lane / LPK, j = lane % LPK;  // key slot in a step, 16-byte chunk (dims 8j..8j+7)
  const int pstart = start[b];
  const int n_keys = min(pstart + 1, T);
  const int64_t base = ((int64_t)slot[b] * H + h) * T * D + j * 8;
  // cached rows (t < pstart) of the first U steps, before the dependency wait
  uint4 kr[U], vr[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int t = u * KPI + sub;
    if (live && t < pstart && t < n_keys) {
      kr[u] = *reinterpret_cast<const uint4*>(kc + base + (int64_t)t * D);
      vr[u] = *reinterpret_cast<const uint4*>(vc + base + (int64_t)t * D);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  const int QD = H * D;
  const __nv_bfloat16* qrow = qkv + (int64_t)b * ldq;
  float q[8], kf[8], vf[8];
  unpack8(*reinterpret_cast<const bf16x8*>(qrow + h * D + j * 8), q);
  // the call's own key / value (position pstart): K rotated, appended to the cache
  unpack8(*reinterpret_cast<const bf16x8*>(qrow + QD + h * D + j * 8), kf);
  unpack8(*reinterpret_cast<const bf16x8*>(qrow + 2 * QD + h * D + j * 8), vf);
  if (rope) {  // rotate-half partner dims d +- D/2 sit in lane j ^ (LPK / 2) of the group
    float pq[8], pk[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      pq[e] = __shfl_xor_sync(0xffffffffu, q[e], LPK / 2);
      pk[e] = __shfl_xor_sync(0xffffffffu, kf[e], LPK / 2);
    }
    rope8(q, pq, rope + (int64_t)pstart * (D / 2), j * 8, D / 2);
    rope8(kf, pk, rope + (int64_t)pstart * (D / 2), j * 8, D / 2);
  }
  const bf16x8 kfresh = pack8(kf);
  bf16x8 vfresh;
  if (fuse_append) {
    vfresh = *reinterpret_cast<const bf16x8*>(qrow + 2 * QD + h * D + j * 8);
    if (sub == 0 && pstart < T) {
      *reinterpret_cast<bf16x8*>(kc + base + (int64_t)pstart * D) = kfresh;
      *reinterpret_cast<bf16x8*>(vc + base + (int64_t)pstart * D) = vfresh;
    }
  }
  float m = -INFINITY, l = 0.f, acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  auto consume = [&](int t, const uint4& kraw, const uint4& vraw) {
    // t: this group's key (uniform within the group); invalid keys contribute nothing
    bool valid = t < n_keys;
    uint4 kk = kraw, vv = vraw;
    if (t == pstart) {
      if (fuse_append) {
        kk = *reinterpret_cast<const uint4*>(&kfresh);
        vv = *reinterpret_cast<const uint4*>(&vfresh);
      } else {
        kk = *reinterpret_cast<const uint4*>(kc + base + (int64_t)t * D);
        vv = *reinterpret_cast<const uint4*>(vc + base + (int64_t)t * D);
      }
    }
    float k8[8], v8[8];
    unpack8(*reinterpret_cast<const bf16x8*>(&kk), k8);
    float d = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) d = fmaf(q[e], k8[e], d);
#pragma unroll
    for (int o = 1; o < LPK; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (!valid) return;
    const float sc = d * scale_log2;
    const float mn = fmaxf(m, sc);
    const float corr = exp2f(m - mn);  // m = -inf at the first key: corr = 0
    const float pv = exp2f(sc - mn);
    unpack8(*reinterpret_cast<const bf16x8*>(&vv), v8);
    l = l * corr + pv;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = fmaf(pv, v8[e], acc[e] * corr);
    m = mn;
  };
  for (int t0 = 0; t0 < n_keys; t0 += U * KPI) {
    if (t0 > 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u * KPI + sub;
        if (t < pstart && t < n_keys) {
          kr[u] = *reinterpret_cast<const uint4*>(kc + base + (int64_t)t * D);
          vr[u] = *reinterpret_cast<const uint4*>(vc + base + (int64_t)t * D);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) consume(t0 + u * KPI + sub, kr[u], vr[u]);
  }
  // merge the KPI groups' (m, l, acc) in a fixed xor tree
#pragma unroll
  for (int o = LPK; o < 32; o <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float l2 = __shfl_xor_sync(0xffffffffu, l, o);
    const float mn = fmaxf(m, m2);
    const float a1 = m == -INFINITY ? 0.f : exp2f(m - mn);
    const float a2 = m2 == -INFINITY ? 0.f : exp2f(m2 - mn);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float x2 = __shfl_xor_sync(0xffffffffu, acc[e], o);
      acc[e] = acc[e] * a1 + x2 * a2;
    }
    l = l * a1 + l2 * a2;
    m = mn;
  }
  if (sub == 0) {
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= inv;
    *reinterpret_cast<bf16x8*>(out + (int64_t)b * ldo + h * D + j * 8) = pack8(acc);
  }
}

static std::atomic<int> g_coresident{0};
int coresident() { return g_coresident.load(std::memory_order_relaxed); }
int set_coresident(int on) { return g_coresident.exchange(on ? 1 : 0); }

int preload_attention() {
  int n = 0;
  n += preload_fn(attention_decode_kernel<64>) + preload_fn(attention_decode_kernel<128>);
  n += preload_fn(attention_kernel<64, 2, false>) + preload_fn(attention_kernel<128, 2, false>);
  n += preload_fn(attention_kernel<64, 2, true>) + preload_fn(attention_kernel<128, 2, true>);
  n += preload_fn(attention_rows_kernel<64, false>) + preload_fn(attention_rows_kernel<128, false>);
  n += preload_fn(attention_rows_kernel<64, true>) + preload_fn(attention_rows_kernel<128, true>);
  return n;
}

}  // namespace ms

extern "C" int ms_kv_append_paged(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                                  const int32_t* slot, const int32_t* start, int T, void* k_cache,
                                  void* v_cache, const void* rope, const int32_t* block_table, int max_blocks,
                                  int block_size, void* stream);

extern "C" int ms_attention_workspace_gqa(int B, int Q, int H, int Hkv, int D, int T, int64_t* ws_bytes,
                                          int* n_counters) {
  // split-KV scratch: MHA kernel (16-row query chunks) or, Hkv < H, the GQA
  // row-split kernel (96-row records; worth it only for long caches — at
  // decode contexts the records and the last-CTA merge outweigh the extra CTAs)
  if (B < 0 || Q < 1 || H < 1 || Hkv < 1 || H % Hkv || T < 1) return MS_ERR_VALUE;
  if (Hkv < H) {
    const int nzr = (Q * (H / Hkv) + ms::kRRows - 1) / ms::kRRows;
    const int kct = ms::kv_chunk_tiles(T);
    const int n_kv = ((T + ms::kKT - 1) / ms::kKT + kct - 1) / kct;
    if (ws_bytes) *ws_bytes = (int64_t)B * Hkv * nzr * n_kv * ms::kRRows * (D + 2) * 4;
    if (n_counters) *n_counters = B * Hkv * nzr;
    return MS_OK;
  }
  const int nqc = (Q * (H / Hkv) + 15) / 16;
  const int kct = ms::kv_chunk_tiles(T);
  const int n_kv = ((T + ms::kKT - 1) / ms::kKT + kct - 1) / kct;
  if (ws_bytes) *ws_bytes = (int64_t)B * Hkv * nqc * n_kv * 16 * (D + 2) * 4;
  if (n_counters) *n_counters = B * Hkv * nqc;
  return MS_OK;
}

extern "C" int ms_attention_workspace(int B, int Q, int H, int D, int T, int64_t* ws_bytes,
                                      int* n_counters) {
  return ms_attention_workspace_gqa(B, Q, H, H, D, T, ws_bytes, n_counters);
}

extern "C" int ms_attention_paged(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                                  const int32_t* slot, const int32_t* start, int T, void* k_cache,
                                  void* v_cache, const void* rope, float scale, int append, void* out,
                                  int64_t ldo, void* ws, int64_t ws_bytes, int* counters, int n_counters,
                                  const int32_t* block_table, int max_blocks, int block_size, void* stream) {
  if (B < 0 || Q < 1 || H < 1 || Hkv < 1 || T < 1) return MS_ERR_VALUE;
  if (H % Hkv) return MS_ERR_VALUE;
  if (block_table && (block_size < 1 || max_blocks < 1 || T > max_blocks * block_size)) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache || !out) return MS_ERR_VALUE;
  if (ldq % 8) return MS_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const ms::KVPage pg{block_table, max_blocks, block_size};
  int fuse = 0;
  if (append) {
    if (Q <= 16) {
      fuse = 1;  // appended inside the kernel by the first query chunk's CTA
    } else {
      const int s = ms_kv_append_paged(qkv, ldq, B, Q, H, Hkv, D, slot, start, T, k_cache, v_cache, rope,
                                       block_table, max_blocks, block_size, stream);
      if (s != MS_OK) return s;
    }
  }
  if (ms::coresident() && Q == 1 && Hkv == H && !block_table && !ws && (D == 64 || D == 128)) {
    const dim3 grid((B * H + 1) / 2);
    const float sl = scale * 1.4426950408889634f;
    auto* q = (const __nv_bfloat16*)qkv;
    auto* kc = (__nv_bfloat16*)k_cache;
    auto* vc = (__nv_bfloat16*)v_cache;
    auto* o = (__nv_bfloat16*)out;
    return D == 64 ? ms::launch(ms::attention_decode_kernel<64>, grid, dim3(64), 0, st, 1, q, ldq, B, H, slot, start,
                                T, kc, vc, sl, fuse, (const float2*)rope, o, ldo)
                   : ms::launch(ms::attention_decode_kernel<128>, grid, dim3(64), 0, st, 1, q, ldq, B, H, slot,
                                start, T, kc, vc, sl, fuse, (const float2*)rope, o, ldo);
  }
  if (D == 64)
    return ms::launch_attn<64>(qkv, ldq, B, Q, H, Hkv, slot, start, T, k_cache, v_cache, (const float2*)rope,
                               scale, fuse, out, ldo, (float*)ws, ws_bytes, counters, n_counters, st, pg);
  if (D == 128)
    return ms::launch_attn<128>(qkv, ldq, B, Q, H, Hkv, slot, start, T, k_cache, v_cache, (const float2*)rope,
                                scale, fuse, out, ldo, (float*)ws, ws_bytes, counters, n_counters, st, pg);
  return MS_ERR_UNSUPPORTED;
}

extern "C" int ms_attention_gqa(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                                const int32_t* slot, const int32_t* start, int T, void* k_cache,
                                void* v_cache, const void* rope, float scale, int append, void* out,
                                int64_t ldo, void* ws, int64_t ws_bytes, int* counters, int n_counters,
                                void* stream) {
  return ms_attention_paged(qkv, ldq, B, Q, H, Hkv, D, slot, start, T, k_cache, v_cache, rope, scale, append, out,
                            ldo, ws, ws_bytes, counters, n_counters, nullptr, 0, 0, stream);
}

extern "C" int ms_attention(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                            const int32_t* slot, const int32_t* start, int T, void* k_cache,
                            void* v_cache, float scale, int append, void* out, int64_t ldo,
                            void* ws, int64_t ws_bytes, int* counters, int n_counters,
                            void* stream) {
  return ms_attention_gqa(qkv, ldq, B, Q, H, H, D, slot, start, T, k_cache, v_cache, nullptr, scale, append,
                          out, ldo, ws, ws_bytes, counters, n_counters, stream);
}
