// K6 on tcgen05: grouped-query verify / decode attention of the Llama-2-70B
// verifier (head dim 128, G = H / Hkv query heads per KV head, Q <= 16 query
// positions per request, Q * G <= 128 flattened rows), one CTA per (request,
// KV head):
//
//   * the call's own K / V rows are appended to the cache (K rotated), then the
//     cache is read in 128-key chunks by TMA (two 64-dim boxes per operand,
//     128-byte swizzle), double-buffered;
//   * S = Q K^T on tcgen05 (M = 128 flattened rows — position i, group head j
//     -> row i * G + j, Q staged RoPE-rotated into a swizzled K-major tile —,
//     N = 128 keys, K = 128 dims), fp32 accumulator in TMEM;
//   * two key groups (warpgroups) take alternate chunks concurrently, each
//     with its own S / O accumulators in TMEM, P tile and softmax state; in a
//     group four warps own one TMEM lane = one row each: causal mask, online softmax
//     in the exp2 domain (running max / sum per row, the O accumulator in TMEM
//     rescaled in place when the max moves), P written back as bf16 into a
//     swizzled K-major tile;
//   * O += P V on tcgen05 with V as the MN-major operand (keys along K, dims
//     along N, straight from the TMA tile);
//   * the epilogue merges the two groups' (m, l, O) in group order through
//     shared memory, divides by the row sum and stores bf16.
//
// Every row's arithmetic depends only on its own query and the keys it sees
// (chunking fixed by key position, fixed per-row reduction orders): the
// verify rows of a request give the same logits whatever Q (batch
// invariance, the lossless property).  Replaces the attention inside
// ModelOracle.next_dist for the draft / verify positions (aggspec/oracles.py:
// 19-26, aggspec/engine.py:294-296).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "common.cuh"
#include "tc.cuh"

namespace ms {
namespace atc {

constexpr int kD = 128;       // head dim
constexpr int kRows = 128;    // MMA M: flattened (position, group head) rows
constexpr int kKeys = 128;    // keys per chunk (MMA N of S, K of P.V)
constexpr int kThreads = 256;  // two key groups (warpgroups) of 4 warps
constexpr int BLK = kRows * 64 * 2;  // one [128 x 64] bf16 swizzled block = 16 KB

struct Smem {
  // all tiles 1024-byte aligned (128-byte swizzle atoms); buffer / tile g
  // belongs to key group g (chunks ch with ch % 2 == g)
  static constexpr int Q_OFF = 0;                     // Q [128 rows x 128 dims] = 2 blocks
  static constexpr int K_OFF = Q_OFF + 2 * BLK;       // K [2 groups][128 keys x 128 dims]
  static constexpr int V_OFF = K_OFF + 4 * BLK;       // V [2 groups][128 keys x 128 dims]
  static constexpr int P_OFF = V_OFF + 4 * BLK;       // P [2 groups][128 rows x 128 keys]
  static constexpr int BAR_OFF = P_OFF + 4 * BLK;
  static constexpr int BYTES = BAR_OFF + 64 + 1024 + 1024;  // barriers, group 1 (m, l) per row, alignment slack
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#ifdef ATC_DEBUG
// bounded wait: report the barrier that never completed and trap
__device__ __forceinline__ void wait_dbg(uint64_t* bar, uint32_t parity, int tag) {
  const uint32_t a = tc::smem_u32(bar);
  for (long long it = 0; it < (1ll << 24); ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
  }
  printf("attention_tc: stuck at barrier %d parity %u block (%d,%d) thread %d\n", tag, parity, blockIdx.x, blockIdx.y,
         threadIdx.x);
  asm volatile("trap;");
}
#define MBW(bar, par, tag) wait_dbg(bar, par, tag)
#else
#define MBW(bar, par, tag) tc::mbar_wait(bar, par)
#endif

// byte offset of the 16-byte chunk `c` (0..7) of row r in a [rows x 64] bf16
// block with the 128-byte swizzle (chunk index XOR row % 8)
__device__ __forceinline__ int swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

// MN-major operand descriptor, 128-byte swizzle: 64-element MN atoms LBO
// bytes apart, 8-row K groups 1024 bytes apart
__device__ __forceinline__ uint64_t desc_mn_sw128(const void* base, uint32_t lbo) {
  const uint64_t addr = tc::smem_u32(base);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(kThreads, 1)
attention_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Qtot, int Hq, int Hkv,
                    const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                    __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, float scale_log2,
                    int fuse_append, const float2* __restrict__ rope, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm + Smem::Q_OFF;
  uint8_t* sK = sm + Smem::K_OFF;
  uint8_t* sV = sm + Smem::V_OFF;
  uint8_t* sP = sm + Smem::P_OFF;
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(sm + Smem::BAR_OFF);  // [2 groups]
  uint64_t* s_full = kv_full + 2;                                       // [2]
  uint64_t* pv_done = s_full + 2;                                       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);
  float* stat = reinterpret_cast<float*>(tmem_slot + 4);                // [128 rows][2]: group 1's (m, l)

  const int b = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int g = warp >> 2;          // key group
  const int gt = tid & 127;         // thread within the group = row (TMEM lane)
  const bool issuer = gt == 0;      // the group's TMA / MMA thread
  const int G = Hq / Hkv;
  const int rows_tot = Qtot * G;
  const int QD = Hq * kD, KVD = Hkv * kD;
  constexpr int V8 = kD / 8;

  if (tid == 0) {
    tc::prefetch_tmap(&tmK);
    tc::prefetch_tmap(&tmV);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&pv_done[i], 1);
    }
    tc::fence_barrier_init();
  }
  __syncwarp();
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);  // S0 | S1 | O0 | O1, 128 columns each
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem + g * 128, tO = tmem + 256 + g * 128;
  uint8_t* gK = sK + 2 * g * BLK;
  uint8_t* gV = sV + 2 * g * BLK;
  uint8_t* gP = sP + 2 * g * BLK;

  // the cache rows of earlier calls (keys < pstart) do not depend on the
  // previous kernel: chunks made only of them are requested before the
  // programmatic-dependency wait and the append (start / slot come from
  // earlier kernels, complete by then)
  const int pstart = start[b];
  const int kv_slot = slot[b];
  const int64_t row0 = ((int64_t)kv_slot * Hkv + h) * T;  // cache row of key 0
  const int n_keys = min(pstart + Qtot, T);
  const int n_chunks = (n_keys + kKeys - 1) / kKeys;
  auto load_chunk = [&](int ch) {  // the issuer of group ch % 2
    const int buf = ch & 1;
    tc::mbar_arrive_expect_tx(&kv_full[buf], 4 * BLK);
    const int y = (int)(row0 + ch * kKeys);
    const uint64_t pol = tc::policy_evict_first();
    for (int half = 0; half < 2; ++half) {
      tc::tma_load_2d(sK + (2 * buf + half) * BLK, &tmK, &kv_full[buf], half * 64, y, pol);
      tc::tma_load_2d(sV + (2 * buf + half) * BLK, &tmV, &kv_full[buf], half * 64, y, pol);
    }
  };
  const bool early = g < n_chunks && (g + 1) * kKeys <= pstart;  // this group's first chunk is all cache
  if (issuer && early) load_chunk(g);
  pdl_wait();
  pdl_trigger();

  // (1) the call's own K / V rows -> cache (K rotated); visible to the TMA
  // (async proxy) after the proxy fence + barrier
  if (fuse_append) {
    for (int e = tid; e < 2 * Qtot * V8; e += kThreads) {
      const int kv = e >= Qtot * V8;
      const int e2 = e - kv * Qtot * V8;
      const int i = e2 / V8, c = e2 - i * V8;
      const int p = pstart + i;
      if (p < 0 || p >= T) continue;
      const __nv_bfloat16* rowp = qkv + (int64_t)(b * Qtot + i) * ldq + QD + kv * KVD + h * kD;
      bf16x8 val = *reinterpret_cast<const bf16x8*>(rowp + c * 8);
      if (!kv && rope) {
        const int pc = c < V8 / 2 ? c + V8 / 2 : c - V8 / 2;
        float fv[8], pf[8];
        unpack8(val, fv);
        unpack8(*reinterpret_cast<const bf16x8*>(rowp + pc * 8), pf);
        rope8(fv, pf, rope + (int64_t)p * (kD / 2), c * 8, kD / 2);
        val = pack8(fv);
      }
      *reinterpret_cast<bf16x8*>((kv ? vc : kc) + (row0 + p) * kD + c * 8) = val;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  // (2) Q -> swizzled K-major tile (rows past the call are zero), RoPE applied
  for (int e = tid; e < kRows * V8; e += kThreads) {
    const int r = e / V8, c = e - r * V8;  // row, 16-byte chunk (dims 8c..8c+7)
    bf16x8 val;
    if (r < rows_tot) {
      const __nv_bfloat16* qp = qkv + (int64_t)(b * Qtot + r / G) * ldq + (h * G + r % G) * kD;
      val = *reinterpret_cast<const bf16x8*>(qp + c * 8);
      if (rope) {
        const int pc = c < V8 / 2 ? c + V8 / 2 : c - V8 / 2;
        float fv[8], pf[8];
        unpack8(val, fv);
        unpack8(*reinterpret_cast<const bf16x8*>(qp + pc * 8), pf);
        rope8(fv, pf, rope + (int64_t)(pstart + r / G) * (kD / 2), c * 8, kD / 2);
        val = pack8(fv);
      }
    } else {
      *reinterpret_cast<uint4*>(&val) = make_uint4(0, 0, 0, 0);
    }
    *reinterpret_cast<bf16x8*>(sQ + (c >> 3) * BLK + swz(r, c & 7)) = val;
  }
  tc::fence_proxy_async_smem();
  __syncthreads();

  constexpr uint32_t idS = tc::idesc_bf16(kRows, kKeys);
  constexpr uint32_t idPV = tc::idesc_bf16(kRows, kD) | (1u << 16);  // B (V) MN-major
  auto issue_S = [&](int ch) {  // the group's issuer: S = Q K_ch^T
    MBW(&kv_full[g], (ch >> 1) & 1, 1);
    tc::fence_after_sync();
#pragma unroll
    for (int k = 0; k < kD / 16; ++k) {
      const uint64_t ad = tc::smem_desc_sw128(sQ + (k >> 2) * BLK) + 2 * (k & 3);
      const uint64_t bd = tc::smem_desc_sw128(gK + (k >> 2) * BLK) + 2 * (k & 3);
      tc::mma_bf16(tS, ad, bd, idS, k > 0 ? 1u : 0u);
    }
    tc::mma_commit(&s_full[g]);
  };
  if (issuer && g < n_chunks) {
    if (!early) load_chunk(g);
    issue_S(g);
  }
  __syncwarp();  // the issuer lane diverged: reconverge before the aligned tcgen05.ld

  // softmax state of this thread's row (= TMEM lane gt) over its group's chunks
  const int r = gt;
  const int row_pos = r < rows_tot ? pstart + r / G : -1;  // last key this row may see
  float m_run = -INFINITY, l_run = 0.f;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  int it = 0;  // this group's chunk count so far
  for (int ch = g; ch < n_chunks; ch += 2, ++it) {
    MBW(&s_full[g], it & 1, 2);
    tc::fence_after_sync();
    const int kbase = ch * kKeys;
    // pass 1: masked max of this chunk
    float mx = -INFINITY;
#pragma unroll 1
    for (int c0 = 0; c0 < kKeys; c0 += 32) {
      uint32_t sv[32];
      tc::tmem_ld16(tS + lane_base + c0, *reinterpret_cast<uint32_t(*)[16]>(sv));
      tc::tmem_ld16(tS + lane_base + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int key = kbase + c0 + j;
        if (key <= row_pos && key < n_keys) mx = fmaxf(mx, __uint_as_float(sv[j]) * scale_log2);
      }
    }
    const float m_new = fmaxf(m_run, mx);
    const float corr = m_run == -INFINITY ? 0.f : (m_new == m_run ? 1.f : exp2f(m_run - m_new));
    // the group's previous P.V must be done before O is rescaled and P rewritten
    if (it > 0) {
      MBW(&pv_done[g], (it - 1) & 1, 3);
      tc::fence_after_sync();
      if (__any_sync(0xffffffffu, corr != 1.f)) {  // warp-uniform: the TMEM ops are warp-collective
#pragma unroll 1
        for (int c0 = 0; c0 < kD; c0 += 32) {
          uint32_t ov[32];
          tc::tmem_ld16(tO + lane_base + c0, *reinterpret_cast<uint32_t(*)[16]>(ov));
          tc::tmem_ld16(tO + lane_base + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(ov + 16));
          tc::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
          tmem_st16(tO + lane_base + c0, *reinterpret_cast<uint32_t(*)[16]>(ov));
          tmem_st16(tO + lane_base + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(ov + 16));
        }
        tmem_wait_st();
      }
    }
    // pass 2: P = exp2(s - m_new) (masked -> 0), row sum, P -> the group's swizzled tile
    float psum = 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < kKeys; c0 += 32) {
      uint32_t sv[32];
      tc::tmem_ld16(tS + lane_base + c0, *reinterpret_cast<uint32_t(*)[16]>(sv));
      tc::tmem_ld16(tS + lane_base + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
      tc::tmem_wait_ld();
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        float pv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int key = kbase + c0 + q4 * 8 + j;
          const bool vis = key <= row_pos && key < n_keys && m_new != -INFINITY;
          pv[j] = vis ? exp2f(__uint_as_float(sv[q4 * 8 + j]) * scale_log2 - m_new) : 0.f;
          psum += pv[j];
        }
        const int c = (c0 >> 3) + q4;  // 16-byte chunk (8 keys) within the 128 keys
        *reinterpret_cast<bf16x8*>(gP + (c >> 3) * BLK + swz(r, c & 7)) = pack8(pv);
      }
    }
    l_run = l_run * corr + psum;
    m_run = m_new;
    tc::fence_proxy_async_smem();  // P visible to the MMA (async proxy)
    tc::fence_before_sync();       // S reads and O stores ordered before the next MMAs
    asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");  // the group's 4 warps
    if (issuer) {
      tc::fence_after_sync();
#pragma unroll
      for (int k = 0; k < kKeys / 16; ++k) {
        const uint64_t ad = tc::smem_desc_sw128(gP + (k >> 2) * BLK) + 2 * (k & 3);
        // V rows 16k..16k+15 (2048 bytes per 16 keys), the two 64-dim boxes BLK apart
        const uint64_t bd = desc_mn_sw128(gV + k * 2048, BLK);
        tc::mma_bf16(tO, ad, bd, idPV, (it > 0 || k > 0) ? 1u : 0u);
      }
      tc::mma_commit(&pv_done[g]);
      if (ch + 2 < n_chunks) {
        // the group's K/V buffer is free once this P.V completes
        MBW(&pv_done[g], it & 1, 4);
        load_chunk(ch + 2);
        issue_S(ch + 2);
      }
    }
    __syncwarp();
  }
  // epilogue: group 1 hands its row statistics (m, l) to group 0 through shared
  // memory; group 0 reads both groups' O rows from TMEM (its warps own the same
  // TMEM lanes), merges them in group order, divides and stores
  const int nit = it;
  if (nit > 0) {
    MBW(&pv_done[g], (nit - 1) & 1, 5);
    tc::fence_after_sync();
  }
  if (g == 1) {
    stat[2 * r] = nit > 0 ? m_run : -INFINITY;
    stat[2 * r + 1] = nit > 0 ? l_run : 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();  // every P.V of both groups is complete
  if (g == 0) {
    tc::fence_after_sync();
    const float m1 = stat[2 * r], l1 = stat[2 * r + 1];
    const bool has1 = n_chunks > 1;  // group 1 wrote O1
    const float m = fmaxf(m_run, m1);
    const float a0 = m_run == -INFINITY ? 0.f : exp2f(m_run - m);
    const float a1 = (!has1 || m1 == -INFINITY) ? 0.f : exp2f(m1 - m);
    const float L = l_run * a0 + l1 * a1;
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const uint32_t tO1 = tmem + 384;
    __nv_bfloat16* op = out + (int64_t)(b * Qtot + (r < rows_tot ? r / G : 0)) * ldo + (h * G + r % G) * kD;
#pragma unroll 1
    for (int c0 = 0; c0 < kD; c0 += 16) {
      uint32_t o0[16], o1[16];
      tc::tmem_ld16(tO + lane_base + c0, o0);
      tc::tmem_ld16(tO1 + lane_base + c0, o1);
      tc::tmem_wait_ld();
      if (r < rows_tot) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float f[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x0 = nit > 0 ? __uint_as_float(o0[c * 8 + j]) : 0.f;
            const float x1 = has1 ? __uint_as_float(o1[c * 8 + j]) : 0.f;
            f[j] = (x0 * a0 + x1 * a1) * inv;
          }
          *reinterpret_cast<bf16x8*>(op + c0 + c * 8) = pack8(f);
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// the cache [rows, 128] bf16 as 2-D, box = [64 dims, 128 keys], 128-byte swizzle
static bool cache_tmap(CUtensorMap* m, const void* base, int64_t rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(kD * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)kKeys};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace atc

int preload_attention_tc() { return preload_fn(atc::attention_tc_kernel); }

}  // namespace ms

extern "C" int ms_attention_tc(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                               const int32_t* slot, const int32_t* start, int T, int n_slots, void* k_cache,
                               void* v_cache, const void* rope, float scale, int append, void* out, int64_t ldo,
                               void* stream) {
  using namespace ms;
  if (B < 0 || Q < 1 || H < 1 || Hkv < 1 || T < 1 || n_slots < 1 || H % Hkv) return MS_ERR_VALUE;
  if (D != atc::kD || Q * (H / Hkv) > atc::kRows || Q > 16) return MS_ERR_UNSUPPORTED;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache || !out || ldq % 8 || ldo % 8) return MS_ERR_VALUE;
  const int64_t rows = (int64_t)n_slots * Hkv * T;
  CUtensorMap tk, tv;
  if (!atc::cache_tmap(&tk, k_cache, rows) || !atc::cache_tmap(&tv, v_cache, rows)) return MS_ERR_CUDA;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(atc::attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             atc::Smem::BYTES) != cudaSuccess)
      return MS_ERR_CUDA;
    attr = true;
  }
  return launch(atc::attention_tc_kernel, dim3(B, Hkv), dim3(atc::kThreads), atc::Smem::BYTES,
                (cudaStream_t)stream, 1, tk, tv, (const __nv_bfloat16*)qkv, ldq, Q, H, Hkv, slot, start, T,
                (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, scale * 1.4426950408889634f, append,
                (const float2*)rope, (__nv_bfloat16*)out, ldo);
}
