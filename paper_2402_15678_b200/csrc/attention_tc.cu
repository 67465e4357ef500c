// K6 on tcgen05: grouped-query verify / decode attention of the Llama-2-70B
// verifier (head dim 128, G = H / Hkv query heads per KV head, Q <= 16 query
// positions per request, Q * G <= 128 flattened rows), one CTA per (request,
// KV head):
//
//   * the call's own K / V rows are appended to the cache (K rotated), then the
//     cache is read in 128-key chunks by TMA (two 64-dim boxes per operand,
//     128-byte swizzle); long caches: one producer warp per key group issues
//     its K (two buffers) and V (one buffer) loads as the buffers retire;
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
//     along N, straight from the TMA tile); in the online kernel P stays in
//     TMEM (bf16, over the consumed S columns) as the MMA's A operand;
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
constexpr int kThreadsOnline = kThreads + 64;  // online kernel: + one K / V producer warp per group
constexpr int BLK = kRows * 64 * 2;  // one [128 x 64] bf16 swizzled block = 16 KB

struct Smem {
  // all tiles 1024-byte aligned (128-byte swizzle atoms); buffers g* belong to
  // key group g (chunks ch with ch % 2 == g).  P lives in TMEM (aliased onto
  // the consumed S columns), which leaves room for two K buffers per group.
  static constexpr int Q_OFF = 0;                     // Q [128 rows x 128 dims] = 2 blocks
  static constexpr int K_OFF = Q_OFF + 2 * BLK;       // K [2 groups][2 buffers][128 keys x 128 dims]
  static constexpr int V_OFF = K_OFF + 8 * BLK;       // V [2 groups][128 keys x 128 dims]
  static constexpr int BAR_OFF = V_OFF + 4 * BLK;
  static constexpr int BYTES = BAR_OFF + 128 + 1024 + 1024;  // barriers, group 1 (m, l) per row, alignment slack
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

// D (TMEM) (+)= A (TMEM, M = 128 rows in lanes, K = 16 bf16 in 8 columns) x
// B (shared memory descriptor): the P.V step with P kept in TMEM
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

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

#ifdef ATC_PROF
// diagnostic build only (tools/atc_prof.py): thread 0's %globaltimer at each
// phase of the last launch, per CTA
__device__ unsigned long long g_atc_prof[4096][12];
#define PROF(i)                                                                       \
  do {                                                                                \
    if (threadIdx.x == 0) {                                                           \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_atc_prof[blockIdx.x * gridDim.y + blockIdx.y][i] = t_;                        \
    }                                                                                 \
  } while (0)
#else
#define PROF(i)
#endif

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

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

template <int D>  // head dim: 128, or 64 (prompt-prefill tiles of the small drafters)
__global__ void __launch_bounds__(kThreadsOnline, 1)
attention_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Qtot, int Hq, int Hkv,
                    const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                    __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, float scale_log2,
                    int fuse_append, const float2* __restrict__ rope, __nv_bfloat16* __restrict__ out, int64_t ldo,
                    const int32_t* __restrict__ block_table, int max_blocks, int bs) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm + Smem::Q_OFF;
  uint8_t* sK = sm + Smem::K_OFF;
  uint8_t* sV = sm + Smem::V_OFF;
  uint64_t* k_full = reinterpret_cast<uint64_t*>(sm + Smem::BAR_OFF);  // [2 groups][2 buffers]
  uint64_t* v_full = k_full + 4;                                       // [2]
  uint64_t* s_full = v_full + 2;                                       // [2]
  uint64_t* pv_done = s_full + 2;                                       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);
  float* stat = reinterpret_cast<float*>(tmem_slot + 4);                // [128 rows][2]: group 1's (m, l)

  PROF(0);
  const int b = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5;
  // warps 0-7: two key groups of 4 softmax warps; warps 8, 9: the K / V
  // producers of group 0 / 1 (lane 0 issues the group's TMA loads in chunk
  // order, each as soon as its buffer retires, so no softmax warp waits for
  // a buffer to free)
  const bool producer = warp >= 8;
  const int g = producer ? warp - 8 : warp >> 2;  // key group
  const int gt = tid & 127;         // thread within the group = row (TMEM lane)
  const bool issuer = !producer && gt == 0;        // the group's MMA thread
  const bool loader = producer && (tid & 31) == 0;  // the group's TMA thread
  const int G = Hq / Hkv;
  // query tile (prompt prefill: Qtot > 16 or Qtot * G > 128 — one CTA per
  // (request, KV head, Qt positions), the call's K / V appended beforehand):
  // positions q0 .. q0 + Qc - 1 of the call; decode / verify: one tile
  const int Qt = kRows / G;
  const int q0 = blockIdx.z * Qt;
  const int Qc = min(Qt, Qtot - q0);
  const int64_t qrow0 = (int64_t)blockIdx.x * Qtot + q0;  // qkv / out row of the tile's first position
  const int rows_tot = Qc * G;
  const int QD = Hq * D, KVD = Hkv * D;

  // start / slot come from kernels complete before the previous one (the
  // round's upload): read first, their latency hidden by the setup below
  const int pcall = start[b];       // position of the call's first query
  const int pstart = pcall + q0;    // ... and of this tile's
  const int kv_slot = slot[b];
  if (tid == 0) {
    tc::prefetch_tmap(&tmK);
    tc::prefetch_tmap(&tmV);
    for (int i = 0; i < 4; ++i) tc::mbar_init(&k_full[i], 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&v_full[i], 1);
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
  uint8_t* gV = sV + 2 * g * BLK;

  // the cache rows of earlier calls (keys < pstart) do not depend on the
  // previous kernel: chunks made only of them are requested before the
  // programmatic-dependency wait and the append (start / slot come from
  // earlier kernels, complete by then)
  const int64_t row0 = ((int64_t)kv_slot * Hkv + h) * T;  // cache row of key 0
  const int n_keys = min(pstart + Qc, T);
  const int n_chunks = (n_keys + kKeys - 1) / kKeys;
  // K and V of a chunk on separate barriers.  A group's chunks are ch = g +
  // 2i; K(ch) goes to the group's K buffer i % 2 (two per group: K(ch + 4) is
  // requested when S(ch) completes, two chunks ahead of its use), V(ch) to
  // the group's one V buffer (requested when P.V(ch - 2) retires)
  auto kbuf = [&](int ch) { return sK + (2 * (ch & 1) + ((ch >> 1) & 1)) * 2 * BLK; };
  auto kbar = [&](int ch) { return &k_full[2 * (ch & 1) + ((ch >> 1) & 1)]; };
  auto load_kv = [&](int ch, bool v) {  // the loader of group ch % 2
    uint64_t* bar = v ? &v_full[ch & 1] : kbar(ch);
    uint8_t* dst = v ? sV + 2 * (ch & 1) * BLK : kbuf(ch);
    tc::mbar_arrive_expect_tx(bar, (D / 64) * BLK);
    const uint64_t pol = tc::policy_evict_first();
    if (!block_table) {
      const int y = (int)(row0 + ch * kKeys);
      for (int half = 0; half < D / 64; ++half)
        tc::tma_load_2d(dst + half * BLK, v ? &tmV : &tmK, bar, half * 64, y, pol);
    } else {  // paged (prefill tiles): one box of bs rows per block; blocks past
              // the table repeat its last block (finite rows, masked keys)
      const int nb = kKeys / bs;
      for (int j = 0; j < nb; ++j) {
        const int t = min(ch * kKeys + j * bs, T - bs);
        const int y = (int)(((int64_t)block_table[(int64_t)kv_slot * max_blocks + t / bs] * Hkv + h) * bs);
        for (int half = 0; half < D / 64; ++half)
          tc::tma_load_2d(dst + half * BLK + j * (BLK / nb), v ? &tmV : &tmK, bar, half * 64, y, pol);
      }
    }
  };
  // chunks made only of cache rows of earlier calls are requested before the
  // dependency wait; the others after the append below
  // (keys below pcall: earlier calls' rows; the call's own rows come from
  // the append, in this kernel or the one before it)
  const bool early = g < n_chunks && (g + 1) * kKeys <= pcall;  // this group's first chunk is all cache
  const bool early2 = g + 2 < n_chunks && (g + 3) * kKeys <= pcall;
  if (loader && early) {
    load_kv(g, false);
    load_kv(g, true);
  }
  if (loader && early2) load_kv(g + 2, false);
  pdl_wait();
  pdl_trigger();

  // (1) the call's own K / V rows -> cache (K rotated) and (2) Q -> the
  // swizzled K-major tile (RoPE applied, rows past the call zero).  A unit is
  // one row's dims {8j..8j+7} and {64+8j..64+8j+7} — a RoPE pair, one (cos,
  // sin) run; each thread issues every load of its units (kQU of Q, at most
  // one of the append: 2 * Qtot * 8 <= 256) before using any, so the staging
  // costs one global latency.  The appended rows are visible to the TMA
  // (async proxy) after the proxy fence + barrier.
  constexpr int UPR = D / 16;  // staging units per row (a unit: 8 dims and their rotate-half partners)
  constexpr int kQU = kRows * UPR / kThreads;
  const int n_app = fuse_append ? 2 * Qtot * UPR : 0;
  bf16x8 ux0[kQU + 1], ux1[kQU + 1];
  float2 ucs[kQU + 1][8];
  auto unit = [&](int u, const __nv_bfloat16*& src, __nv_bfloat16*& dst, int& r, int& j, int& p, bool& rot) {
    src = nullptr;
    dst = nullptr;
    rot = false;
    if (u < kQU) {  // Q unit: row r = e / 8
      const int e = tid + u * kThreads;
      r = e / UPR;
      j = e % UPR;
      p = pstart + r / G;
      if (r < rows_tot) {
        src = qkv + (qrow0 + r / G) * ldq + (h * G + r % G) * D + 8 * j;
        rot = rope != nullptr;
      }
    } else if (tid < n_app) {  // append unit: K rows, then V rows
      const int kv = tid >= Qtot * UPR;
      const int e2 = tid - kv * Qtot * UPR;
      const int i = e2 / UPR;
      j = e2 % UPR;
      p = pstart + i;
      r = -1;
      if (p >= 0 && p < T) {
        src = qkv + (int64_t)(b * Qtot + i) * ldq + QD + kv * KVD + h * D + 8 * j;
        dst = (kv ? vc : kc) + (row0 + p) * D + 8 * j;
        rot = !kv && rope != nullptr;
      }
    }
  };
  if (!producer) {  // the producers take no staging units
  #pragma unroll
    for (int u = 0; u <= kQU; ++u) {
      const __nv_bfloat16* src;
      __nv_bfloat16* dst;
      int r, j, p;
      bool rot;
      unit(u, src, dst, r, j, p, rot);
      if (src) {
        ux0[u] = *reinterpret_cast<const bf16x8*>(src);
        ux1[u] = *reinterpret_cast<const bf16x8*>(src + D / 2);
        if (rot) {
  #pragma unroll
          for (int k = 0; k < 8; ++k) ucs[u][k] = rope[(int64_t)p * (D / 2) + 8 * j + k];
        }
      }
    }
  #pragma unroll
    for (int u = 0; u <= kQU; ++u) {
      const __nv_bfloat16* src;
      __nv_bfloat16* dst;
      int r, j, p;
      bool rot;
      unit(u, src, dst, r, j, p, rot);
      bf16x8 v0, v1;
      if (src) {
        v0 = ux0[u];
        v1 = ux1[u];
        if (rot) {
          float f0[8], f1[8];
          unpack8(v0, f0);
          unpack8(v1, f1);
  #pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float2 t = ucs[u][k];
            const float a = f0[k], c = f1[k];
            f0[k] = a * t.x - c * t.y;
            f1[k] = c * t.x + a * t.y;
          }
          v0 = pack8(f0);
          v1 = pack8(f1);
        }
      } else {
        *reinterpret_cast<uint4*>(&v0) = make_uint4(0, 0, 0, 0);
        v1 = v0;
      }
      if (u < kQU) {
        constexpr int H2 = D / 2;  // the partner dims D/2 + 8j: block H2 / 64, 16-byte chunk (H2 % 64) / 8 + j
        *reinterpret_cast<bf16x8*>(sQ + swz(r, j)) = v0;
        *reinterpret_cast<bf16x8*>(sQ + (H2 >> 6) * BLK + swz(r, ((H2 & 63) >> 3) + j)) = v1;
      } else if (dst) {
        *reinterpret_cast<bf16x8*>(dst) = v0;
        *reinterpret_cast<bf16x8*>(dst + D / 2) = v1;
      }
    }
  }
  if (fuse_append) asm volatile("fence.proxy.async.global;" ::: "memory");
  tc::fence_proxy_async_smem();
  __syncthreads();
  PROF(1);

  constexpr uint32_t idS = tc::idesc_bf16(kRows, kKeys);
  constexpr uint32_t idPV = tc::idesc_bf16(kRows, D) | (1u << 16);  // B (V) MN-major
  auto issue_S = [&](int ch) {  // the group's issuer: S = Q K_ch^T
    MBW(kbar(ch), (ch >> 2) & 1, 1);
    tc::fence_after_sync();
    uint8_t* gK = kbuf(ch);
#pragma unroll
    for (int k = 0; k < D / 16; ++k) {
      const uint64_t ad = tc::smem_desc_sw128(sQ + (k >> 2) * BLK) + 2 * (k & 3);
      const uint64_t bd = tc::smem_desc_sw128(gK + (k >> 2) * BLK) + 2 * (k & 3);
      tc::mma_bf16(tS, ad, bd, idS, k > 0 ? 1u : 0u);
    }
    tc::mma_commit(&s_full[g]);
  };
  if (loader && g < n_chunks) {
    if (!early) {
      load_kv(g, false);
      load_kv(g, true);
    }
    if (g + 2 < n_chunks && !early2) load_kv(g + 2, false);
    // then every later chunk of the group in order: K(ch + 4) into the K
    // buffer S(ch) retires, V(ch + 2) into the V buffer P.V(ch) retires
    for (int ch = g, i = 0; ch + 2 < n_chunks; ch += 2, ++i) {
      MBW(&s_full[g], i & 1, 8);
      if (ch + 4 < n_chunks) load_kv(ch + 4, false);
      MBW(&pv_done[g], i & 1, 9);
      load_kv(ch + 2, true);
    }
  }
  if (issuer && g < n_chunks) issue_S(g);
  __syncwarp();  // the issuer / loader lanes diverged: reconverge before the aligned tcgen05.ld

  // softmax state of this thread's row (= TMEM lane gt) over its group's chunks
  const int r = gt;
  const int row_pos = r < rows_tot ? pstart + r / G : -1;  // last key this row may see
  float m_run = -INFINITY, l_run = 0.f;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  int it = 0;  // this group's chunk count so far
  for (int ch = g; !producer && ch < n_chunks; ch += 2, ++it) {
    MBW(&s_full[g], it & 1, 2);
    tc::fence_after_sync();
    if (it == 4) PROF(4);
    if (it == 8) PROF(5);
    const int kbase = ch * kKeys;
    // Warps whose TMEM lane quadrant holds no query row (rows_tot <= 64 at the
    // benchmark's Q * G) skip the softmax: their P / O rows are never stored
    // (MMA rows are independent).  A working thread loads its row's 128 S
    // values with one TMEM wait, takes the max as 8 independent chains (max
    // is exact: the same m as a sequential scan), rescales O in two 64-column
    // batches and forms P from two 64-key re-reads, the sums in key order —
    // bitwise the same P, l and O as the one-chain loop it replaced, with the
    // per-chunk softmax 3.6 -> 2.1 us (tools/atc_prof_online.py).
    const bool wvalid = (warp & 3) * 32 < rows_tot;  // warp-uniform
    float psum = 0.f, m_new = m_run, corr = 1.f;
    if (wvalid) {
      // keys j <= lim of this chunk are visible to the row; a chunk every row
      // of the warp sees whole (all but the last) skips the per-key masks
      const bool qrow = r < rows_tot;
      const int lim = min(row_pos, n_keys - 1) - kbase;
      const bool wfull = __all_sync(0xffffffffu, !qrow || lim >= kKeys - 1);
      uint32_t sv[kKeys];
#pragma unroll
      for (int c0 = 0; c0 < kKeys; c0 += 16) tc::tmem_ld16(tS + lane_base + c0, *reinterpret_cast<uint32_t(*)[16]>(sv + c0));
      tc::tmem_wait_ld();
      if (it == 4) PROF(2);
      // pass 1: masked max of the raw scores, then one scale (rounding is
      // monotone: max(s) * c == max(s * c) for c > 0)
      float m8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) m8[j] = -INFINITY;
      if (wfull) {
#pragma unroll
        for (int j = 0; j < kKeys; ++j) m8[j & 7] = fmaxf(m8[j & 7], __uint_as_float(sv[j]));
      } else {
#pragma unroll
        for (int j = 0; j < kKeys; ++j)
          if (j <= lim) m8[j & 7] = fmaxf(m8[j & 7], __uint_as_float(sv[j]));
      }
      const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) *
                       scale_log2;
      m_new = fmaxf(m_run, mx);
      if (it == 4) PROF(3);
      corr = m_run == -INFINITY ? 0.f : (m_new == m_run ? 1.f : exp2f(m_run - m_new));
      // the group's previous P.V must be done before O is rescaled and P rewritten
      if (it > 0) {
        MBW(&pv_done[g], (it - 1) & 1, 3);
        tc::fence_after_sync();
        if (it == 4) PROF(6);
        // warp-uniform (the TMEM ops are warp-collective); rows past the call
        // are never stored and do not trigger it
        if (__any_sync(0xffffffffu, qrow && corr != 1.f)) {
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 64) {
            uint32_t ov[64];
#pragma unroll
            for (int c1 = 0; c1 < 64; c1 += 16) tc::tmem_ld16(tO + lane_base + c0 + c1, *reinterpret_cast<uint32_t(*)[16]>(ov + c1));
            tc::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 64; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
#pragma unroll
            for (int c1 = 0; c1 < 64; c1 += 16) tmem_st16(tO + lane_base + c0 + c1, *reinterpret_cast<uint32_t(*)[16]>(ov + c1));
          }
          tmem_wait_st();
        }
      }
      if (it == 4) PROF(8);
      // pass 2: P = exp2(s - m_new) (masked -> 0), row sum in key order; S
      // re-read from TMEM in two 64-key halves and P (bf16, keys 2c / 2c + 1
      // in column c) stored over the consumed S columns 0..63 — the P.V MMA
      // reads it from TMEM
#pragma unroll 1
      for (int h0 = 0; h0 < kKeys; h0 += 64) {
        uint32_t sh[64];
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16)
          tc::tmem_ld16(tS + lane_base + h0 + c0, *reinterpret_cast<uint32_t(*)[16]>(sh + c0));
        tc::tmem_wait_ld();
        uint32_t pw[32];
        if (wfull) {  // every key visible, m_new finite
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float pv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              pv[j] = ex2_ftz(__uint_as_float(sh[c * 8 + j]) * scale_log2 - m_new);
              psum += pv[j];
            }
            const bf16x8 b8 = pack8(pv);
            const uint4 u = *reinterpret_cast<const uint4*>(&b8);
            pw[4 * c] = u.x; pw[4 * c + 1] = u.y; pw[4 * c + 2] = u.z; pw[4 * c + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float pv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const bool vis = h0 + c * 8 + j <= lim && m_new != -INFINITY;
              const float e = ex2_ftz(__uint_as_float(sh[c * 8 + j]) * scale_log2 - m_new);
              pv[j] = vis ? e : 0.f;
              psum += pv[j];
            }
            const bf16x8 b8 = pack8(pv);
            const uint4 u = *reinterpret_cast<const uint4*>(&b8);
            pw[4 * c] = u.x; pw[4 * c + 1] = u.y; pw[4 * c + 2] = u.z; pw[4 * c + 3] = u.w;
          }
        }
        tmem_st16(tS + lane_base + (h0 >> 1), *reinterpret_cast<uint32_t(*)[16]>(pw));
        tmem_st16(tS + lane_base + (h0 >> 1) + 16, *reinterpret_cast<uint32_t(*)[16]>(pw + 16));
        if (it == 4 && h0 == 0) PROF(10);
      }
      tmem_wait_st();
    }
    l_run = l_run * corr + psum;
    m_run = m_new;
    tc::fence_before_sync();  // P stores (TMEM) and O stores ordered before the next MMAs
    asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");  // the group's 4 warps
    if (it == 4) PROF(11);
    if (issuer) {
      tc::fence_after_sync();
      MBW(&v_full[g], (ch >> 1) & 1, 6);
      tc::fence_after_sync();
#pragma unroll
      for (int k = 0; k < kKeys / 16; ++k) {
        // A = P from TMEM (8 columns per 16 keys); V rows 16k..16k+15 (2048
        // bytes per 16 keys), the two 64-dim boxes BLK apart
        const uint64_t bd = desc_mn_sw128(gV + k * 2048, BLK);
        mma_bf16_ts(tO, tS + 8 * k, bd, idPV, (it > 0 || k > 0) ? 1u : 0u);
      }
      tc::mma_commit(&pv_done[g]);
      // S(ch + 2) after the P.V that reads P from the same columns (the MMAs
      // of one thread run in issue order); K(ch + 2) landed an iteration ago
      if (ch + 2 < n_chunks) issue_S(ch + 2);
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
  if (!producer && g == 1) {
    stat[2 * r] = nit > 0 ? m_run : -INFINITY;
    stat[2 * r + 1] = nit > 0 ? l_run : 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();  // every P.V of both groups is complete
  if (!producer && g == 0) {
    tc::fence_after_sync();
    const float m1 = stat[2 * r], l1 = stat[2 * r + 1];
    const bool has1 = n_chunks > 1;  // group 1 wrote O1
    const float m = fmaxf(m_run, m1);
    const float a0 = m_run == -INFINITY ? 0.f : exp2f(m_run - m);
    const float a1 = (!has1 || m1 == -INFINITY) ? 0.f : exp2f(m1 - m);
    const float L = l_run * a0 + l1 * a1;
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const uint32_t tO1 = tmem + 384;
    __nv_bfloat16* op = out + (qrow0 + (r < rows_tot ? r / G : 0)) * ldo + (h * G + r % G) * D;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 16) {
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
  PROF(9);
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

// Short caches (T <= kShortKeys = 384, the benchmark's verify contexts): the
// whole context in one pass, no online rescaling, 16 warps.
//
//   * every K / V chunk is requested by TMA at kernel entry, before the
//     programmatic-dependency wait (the rows of earlier calls do not depend on
//     the previous kernel); the call's own K / V rows are written into the
//     landed tiles from registers (and to the cache), the (cos, sin) rows of
//     RoPE are read before the wait too;
//   * S = Q K^T for every needed 128-key chunk in TMEM columns 0..383;
//   * four warps per TMEM lane quadrant take the 32-key groups g = part (mod
//     4) of every row: masked max (exchanged through shared memory), then
//     P = exp2(s - m) as bf16 over the consumed K tiles and the partial row
//     sums (each warp's keys in order, then parts 0 + 1 + 2 + 3);
//   * one P.V MMA chain over the keys up to the last visible one into O
//     (TMEM columns 384..511); the epilogue scales by 1 / sum, stages the bf16
//     rows in shared memory and stores them coalesced.
//
// The key -> warp assignment and the reduction orders depend only on key
// positions, so a row's arithmetic does not depend on Q (batch invariance);
// P.V steps past a row's last visible key add exact zeros.
constexpr int kShortKeys = 384;
constexpr int kShortThreads = 512;

struct SmemShort {
  static constexpr int Q_OFF = 0;                 // Q [128 rows x 128 dims]: 2 blocks; later the exchange arrays
  static constexpr int K_OFF = Q_OFF + 2 * BLK;   // K [384 keys x 128 dims]: 6 blocks; then P; then the O rows
  static constexpr int V_OFF = K_OFF + 6 * BLK;   // V [384 keys x 128 dims]: 6 blocks
  static constexpr int BAR_OFF = V_OFF + 6 * BLK;
  static constexpr int BYTES = BAR_OFF + 64 + 1024;  // barriers, alignment slack
};

__global__ void __launch_bounds__(kShortThreads, 1)
attention_tc_short_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                          const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int Qtot, int Hq, int Hkv,
                          const int32_t* __restrict__ slot, const int32_t* __restrict__ start, int T,
                          __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, float scale_log2,
                          int fuse_append, const float2* __restrict__ rope, __nv_bfloat16* __restrict__ out,
                          int64_t ldo, const int32_t* __restrict__ block_table, int max_blocks, int bs) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm + SmemShort::Q_OFF;
  uint8_t* sK = sm + SmemShort::K_OFF;
  uint8_t* sV = sm + SmemShort::V_OFF;
  uint8_t* sP = sK;                                                          // after S is complete
  uint8_t* sO = sK;                                                          // after P.V is complete
  float* red = reinterpret_cast<float*>(sQ);                                 // [4 parts][128 rows]: max, then sum
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(sm + SmemShort::BAR_OFF);  // [3 chunks]
  uint64_t* s_full = kv_full + 3;
  uint64_t* pv_done = s_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

  const int b = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int pstart = start[b];
  const int kv_slot = slot[b];
  const int G = Hq / Hkv;
  const int rows_tot = Qtot * G;
  const int QD = Hq * kD, KVD = Hkv * kD;
  const int64_t row0 = ((int64_t)kv_slot * Hkv + h) * T;  // contiguous: cache row of key 0
  // cache row of key t (paged: pool block table[slot][t / bs], row t % bs)
  auto cache_row = [&](int t) -> int64_t {
    if (!block_table) return row0 + t;
    return ((int64_t)block_table[(int64_t)kv_slot * max_blocks + t / bs] * Hkv + h) * bs + t % bs;
  };
  const int n_keys = min(pstart + Qtot, T);
  const int n_chunks = n_keys > 0 ? (n_keys + kKeys - 1) / kKeys : 0;
  const int n_steps = (n_keys + 15) / 16;  // 16-key P.V steps up to the last key
  PROF(0);

  // every needed K / V chunk now: the rows of earlier calls do not depend on
  // the previous kernel, the rows this call appends are overwritten in shared
  // memory below.  Paged: one box of bs rows per block, blocks holding a key
  // below 16 * n_steps (the P.V range; the rest of the chunk is masked)
  if (warp == 0) {
    const int nb_c = block_table ? kKeys / bs : 1;  // boxes per chunk and operand half
    const int need = block_table ? (16 * n_steps + bs - 1) / bs : n_chunks;
    if (tid == 0) {
      tc::prefetch_tmap(&tmK);
      tc::prefetch_tmap(&tmV);
      for (int i = 0; i < 3; ++i) tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(s_full, 1);
      tc::mbar_init(pv_done, 1);
      tc::fence_barrier_init();
      for (int c = 0; c < n_chunks; ++c)
        tc::mbar_arrive_expect_tx(&kv_full[c], 4 * BLK / nb_c * (min(need, (c + 1) * nb_c) - c * nb_c));
    }
    __syncwarp();
    const uint64_t pol = tc::policy_evict_first();
    for (int i = tid; i < need; i += 32) {  // box i: chunk i / nb_c
      const int c = i / nb_c;
      const int y = (int)(block_table ? cache_row(i * bs) : row0 + c * kKeys);
      const int off = (i - c * nb_c) * (BLK / nb_c);
      for (int half = 0; half < 2; ++half) {
        tc::tma_load_2d(sK + (2 * c + half) * BLK + off, &tmK, &kv_full[c], half * 64, y, pol);
        tc::tma_load_2d(sV + (2 * c + half) * BLK + off, &tmV, &kv_full[c], half * 64, y, pol);
      }
    }
  }
  __syncwarp();
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);  // S: columns 0..383, O: 384..511

  // staging units: one row's dims {8j..8j+7} and {64+8j..64+8j+7} (a RoPE
  // pair); kQU of Q per thread, at most one of the append (2 * Qtot * 8 <= 256)
  constexpr int kQU = kRows * 8 / kShortThreads;
  const int n_app = fuse_append ? 2 * Qtot * 8 : 0;
  auto unit = [&](int u, bool& live, int& r, int& j, int& p, int& i, int& kv, bool& rot) {
    live = false;
    rot = false;
    kv = 0;
    if (u < kQU) {
      const int e = tid + u * kShortThreads;
      r = e >> 3;
      j = e & 7;
      i = r / G;
      p = pstart + i;
      live = r < rows_tot;
      rot = live && rope != nullptr;
    } else if (tid < n_app) {
      kv = tid >= Qtot * 8;
      const int e2 = tid - kv * Qtot * 8;
      i = e2 >> 3;
      j = e2 & 7;
      p = pstart + i;
      r = -1;
      live = p >= 0 && p < T;
      rot = live && !kv && rope != nullptr;
    }
  };
  float2 ucs[kQU + 1][8];  // the (cos, sin) rows: constant, read before the dependency wait
#pragma unroll
  for (int u = 0; u <= kQU; ++u) {
    bool live, rot;
    int r, j, p, i, kv;
    unit(u, live, r, j, p, i, kv, rot);
    if (rot) {
#pragma unroll
      for (int k = 0; k < 8; ++k) ucs[u][k] = rope[(int64_t)p * (kD / 2) + 8 * j + k];
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + kShortKeys;
  PROF(1);
  pdl_wait();
  pdl_trigger();
  PROF(2);

  bf16x8 ux0[kQU + 1], ux1[kQU + 1];
#pragma unroll
  for (int u = 0; u <= kQU; ++u) {
    bool live, rot;
    int r, j, p, i, kv;
    unit(u, live, r, j, p, i, kv, rot);
    if (live) {
      const __nv_bfloat16* src = u < kQU ? qkv + (int64_t)(b * Qtot + i) * ldq + (h * G + r % G) * kD + 8 * j
                                         : qkv + (int64_t)(b * Qtot + i) * ldq + QD + kv * KVD + h * kD + 8 * j;
      ux0[u] = *reinterpret_cast<const bf16x8*>(src);
      ux1[u] = *reinterpret_cast<const bf16x8*>(src + 64);
    }
  }
#pragma unroll
  for (int u = 0; u <= kQU; ++u) {
    bool live, rot;
    int r, j, p, i, kv;
    unit(u, live, r, j, p, i, kv, rot);
    bf16x8 v0, v1;
    if (live) {
      v0 = ux0[u];
      v1 = ux1[u];
      if (rot) {
        float f0[8], f1[8];
        unpack8(v0, f0);
        unpack8(v1, f1);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 t = ucs[u][k];
          const float a = f0[k], c = f1[k];
          f0[k] = a * t.x - c * t.y;
          f1[k] = c * t.x + a * t.y;
        }
        v0 = pack8(f0);
        v1 = pack8(f1);
      }
    } else {
      *reinterpret_cast<uint4*>(&v0) = make_uint4(0, 0, 0, 0);
      v1 = v0;
    }
    if (u < kQU) {
      *reinterpret_cast<bf16x8*>(sQ + swz(r, j)) = v0;
      *reinterpret_cast<bf16x8*>(sQ + BLK + swz(r, j)) = v1;
    } else if (live) {
      __nv_bfloat16* dst = (kv ? vc : kc) + cache_row(p) * kD + 8 * j;
      *reinterpret_cast<bf16x8*>(dst) = v0;
      *reinterpret_cast<bf16x8*>(dst + 64) = v1;
      const int c = p / kKeys, rr = p - c * kKeys;  // and into its chunk's landed tile
      tc::mbar_wait(&kv_full[c], 0);
      uint8_t* t = (kv ? sV : sK) + 2 * c * BLK;
      *reinterpret_cast<bf16x8*>(t + swz(rr, j)) = v0;
      *reinterpret_cast<bf16x8*>(t + BLK + swz(rr, j)) = v1;
    }
  }
  if (fuse_append) asm volatile("fence.proxy.async.global;" ::: "memory");
  tc::fence_proxy_async_smem();
  __syncthreads();
  PROF(3);

  constexpr uint32_t idS = tc::idesc_bf16(kRows, kKeys);
  constexpr uint32_t idPV = tc::idesc_bf16(kRows, kD) | (1u << 16);  // B (V) MN-major
  if (tid == 0 && n_chunks > 0) {
    for (int c = 0; c < n_chunks; ++c) {
      tc::mbar_wait(&kv_full[c], 0);
      tc::fence_after_sync();
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint64_t ad = tc::smem_desc_sw128(sQ + (k >> 2) * BLK) + 2 * (k & 3);
        const uint64_t bd = tc::smem_desc_sw128(sK + (2 * c + (k >> 2)) * BLK) + 2 * (k & 3);
        tc::mma_bf16(tmem + c * kKeys, ad, bd, idS, k > 0 ? 1u : 0u);
      }
    }
    tc::mma_commit(s_full);
  }
  __syncwarp();

  const int q = warp & 3, part = warp >> 2;  // TMEM lane quadrant, key part (32-key groups part mod 4)
  const int r = q * 32 + (tid & 31);         // this thread's row = TMEM lane
  const int row_pos = r < rows_tot ? pstart + r / G : -1;
  const uint32_t lane_base = (uint32_t)(q * 32) << 16;
  const int n_grp = (n_keys + 31) / 32;      // groups holding a key < n_keys
  float m = -INFINITY, psum = 0.f;
  // Warps whose lane quadrant holds no query row skip both passes (their P /
  // O rows are never stored).  A warp takes its groups gi, gi + 4 two at a
  // time with one TMEM wait, takes the max of the raw scores and scales once
  // (rounding is monotone: the same m), and skips the per-key masks on groups
  // every row of the warp sees whole; P and the sums in the same key order —
  // bitwise the same results as the one-group-per-wait loop.
  const bool wvalid = q * 32 < rows_tot;  // warp-uniform
  const bool qrow = r < rows_tot;
  const int lim0 = min(row_pos, n_keys - 1);  // last key this row sees
  if (n_chunks > 0) {
    tc::mbar_wait(s_full, 0);
    tc::fence_after_sync();
    PROF(4);
    float mx = -INFINITY;
    if (wvalid) {
#pragma unroll 1
      for (int gi = part; gi < n_grp; gi += 8) {
        const bool two = gi + 4 < n_grp;  // warp-uniform
        uint32_t sv[64];
        tc::tmem_ld16(tmem + lane_base + gi * 32, *reinterpret_cast<uint32_t(*)[16]>(sv));
        tc::tmem_ld16(tmem + lane_base + gi * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
        if (two) {
          tc::tmem_ld16(tmem + lane_base + (gi + 4) * 32, *reinterpret_cast<uint32_t(*)[16]>(sv + 32));
          tc::tmem_ld16(tmem + lane_base + (gi + 4) * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 48));
        }
        tc::tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (t == 1 && !two) break;
          const int lim = lim0 - (gi + 4 * t) * 32;
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
          if (__all_sync(0xffffffffu, !qrow || lim >= 31)) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) m4[jj & 3] = fmaxf(m4[jj & 3], __uint_as_float(sv[t * 32 + jj]));
          } else {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (jj <= lim) m4[jj & 3] = fmaxf(m4[jj & 3], __uint_as_float(sv[t * 32 + jj]));
          }
          mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2);
        }
      }
    }
    red[part * kRows + r] = mx;
  }
  __syncthreads();  // (S complete: the Q region is free for the exchange)
  PROF(5);
  if (n_chunks > 0 && wvalid) {
    m = fmaxf(fmaxf(red[r], red[kRows + r]), fmaxf(red[2 * kRows + r], red[3 * kRows + r]));
#pragma unroll 1
    for (int gi = part; gi < n_grp; gi += 8) {
      const bool two = gi + 4 < n_grp;
      uint32_t sv[64];
      tc::tmem_ld16(tmem + lane_base + gi * 32, *reinterpret_cast<uint32_t(*)[16]>(sv));
      tc::tmem_ld16(tmem + lane_base + gi * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
      if (two) {
        tc::tmem_ld16(tmem + lane_base + (gi + 4) * 32, *reinterpret_cast<uint32_t(*)[16]>(sv + 32));
        tc::tmem_ld16(tmem + lane_base + (gi + 4) * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 48));
      }
      tc::tmem_wait_ld();
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (t == 1 && !two) break;
        const int g2 = gi + 4 * t;
        const int lim = lim0 - g2 * 32;
        const bool wfull = __all_sync(0xffffffffu, !qrow || lim >= 31);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float pv[8];
          if (wfull) {  // every key visible, m finite
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              pv[jj] = ex2_ftz(__uint_as_float(sv[t * 32 + q4 * 8 + jj]) * scale_log2 - m);
              psum += pv[jj];
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const bool vis = q4 * 8 + jj <= lim && m != -INFINITY;
              const float e = ex2_ftz(__uint_as_float(sv[t * 32 + q4 * 8 + jj]) * scale_log2 - m);
              pv[jj] = vis ? e : 0.f;
              psum += pv[jj];
            }
          }
          const int c8 = g2 * 4 + q4;  // 8-key chunk; P block = 64 keys
          *reinterpret_cast<bf16x8*>(sP + (c8 >> 3) * BLK + swz(r, c8 & 7)) = pack8(pv);
        }
      }
    }
  }
  tc::fence_proxy_async_smem();  // P visible to the MMA
  tc::fence_before_sync();
  __syncthreads();               // every max read before the sums overwrite them
  PROF(6);
  red[part * kRows + r] = psum;
  if (tid == 0 && n_chunks > 0) {
    tc::fence_after_sync();
    for (int k = 0; k < n_steps; ++k) {  // (P written for whole 32-key groups)
      const uint64_t ad = tc::smem_desc_sw128(sP + (k >> 2) * BLK) + 2 * (k & 3);
      // V rows 16k..16k+15 of chunk k / 8, the two 64-dim boxes BLK apart
      const uint64_t bd = desc_mn_sw128(sV + (k >> 3) * 2 * BLK + (k & 7) * 2048, BLK);
      tc::mma_bf16(tO, ad, bd, idPV, k > 0 ? 1u : 0u);
    }
    tc::mma_commit(pv_done);
  }
  __syncwarp();
  if (n_chunks > 0) tc::mbar_wait(pv_done, 0);
  tc::fence_after_sync();
  __syncthreads();  // the sums; P.V complete (the K / P region is free for the O rows)
  PROF(7);
  const float L = ((red[r] + red[kRows + r]) + red[2 * kRows + r]) + red[3 * kRows + r];
  const float inv = L > 0.f ? 1.f / L : 0.f;
  {  // this warp's 32 dims of its rows -> bf16 rows in shared memory (16-byte chunks XOR-swizzled by row)
    uint32_t o[32];
    tc::tmem_ld16(tO + lane_base + part * 32, *reinterpret_cast<uint32_t(*)[16]>(o));
    tc::tmem_ld16(tO + lane_base + part * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(o + 16));
    tc::tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float f[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) f[jj] = n_chunks > 0 ? __uint_as_float(o[c * 8 + jj]) * inv : 0.f;
      const int ch = part * 4 + c;  // 16-byte chunk of the 256-byte row
      *reinterpret_cast<bf16x8*>(sO + r * 256 + ((ch ^ (r & 15)) << 4)) = pack8(f);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  PROF(8);
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
  // coalesced stores: half a warp per row (16 lanes x 16 bytes)
  for (int e = tid; e < rows_tot * 16; e += kShortThreads) {
    const int rr = e >> 4, ch = e & 15;
    const bf16x8 v = *reinterpret_cast<const bf16x8*>(sO + rr * 256 + ((ch ^ (rr & 15)) << 4));
    *reinterpret_cast<bf16x8*>(out + (int64_t)(b * Qtot + rr / G) * ldo + (h * G + rr % G) * kD + ch * 8) = v;
  }
  PROF(9);
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

// the cache [rows, 128] bf16 as 2-D, box = [64 dims, box_rows keys], 128-byte swizzle
static bool cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int box_rows = kKeys, int D = kD) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(D * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace atc

int preload_attention_tc() {
  const int e = preload_fn(atc::attention_tc_kernel<128>) + preload_fn(atc::attention_tc_kernel<64>);
  return e ? e : preload_fn(atc::attention_tc_short_kernel);
}

}  // namespace ms

#ifdef ATC_PROF
extern "C" int ms_atc_prof_read(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, ms::atc::g_atc_prof, bytes) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int ms_attention_tc(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                               const int32_t* slot, const int32_t* start, int T, int n_slots, void* k_cache,
                               void* v_cache, const void* rope, float scale, int append, void* out, int64_t ldo,
                               const int32_t* block_table, int max_blocks, int block_size, void* stream) {
  using namespace ms;
  if (B < 0 || Q < 1 || H < 1 || Hkv < 1 || T < 1 || n_slots < 1 || H % Hkv) return MS_ERR_VALUE;
  // prompt prefill (more positions than one 128-row tile or 16): query tiles
  // of the online kernel; the K / V rows must already be in the cache.  Head
  // dim 128, or 64 for prefill tiles (the drafters' prompts)
  // append == 0 always takes this form (a prompt's rows must not depend on
  // how it was chunked)
  const bool tiles = Q * (H / Hkv) > atc::kRows || Q > 16 || !append;
  if (D != atc::kD && !(D == 64 && tiles)) return MS_ERR_UNSUPPORTED;
  if (tiles && append) return MS_ERR_UNSUPPORTED;  // (Q > 16 or Q * G > 128 with a fused append)
  if (block_table && (block_size < 16 || atc::kKeys % block_size || max_blocks < 1 || T != max_blocks * block_size))
    return MS_ERR_VALUE;
  // paged with a fused append: the one-pass kernel only (prefill tiles read
  // a paged cache the append kernel has written)
  if (block_table && !tiles && T > atc::kShortKeys) return MS_ERR_UNSUPPORTED;
  if (B == 0) return MS_OK;
  if (!qkv || !slot || !start || !k_cache || !v_cache || !out || ldq % 8 || ldo % 8) return MS_ERR_VALUE;
  // contiguous: n_slots slots of T rows per KV head; paged: n_slots pool blocks of block_size rows
  const int64_t rows = (int64_t)n_slots * Hkv * (block_table ? block_size : T);
  const int box = block_table ? block_size : atc::kKeys;
  CUtensorMap tk, tv;
  if (!atc::cache_tmap(&tk, k_cache, rows, box, D) || !atc::cache_tmap(&tv, v_cache, rows, box, D)) return MS_ERR_CUDA;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(atc::attention_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             atc::Smem::BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(atc::attention_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             atc::Smem::BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(atc::attention_tc_short_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             atc::SmemShort::BYTES) != cudaSuccess)
      return MS_ERR_CUDA;
    attr = true;
  }
  // the kernel is chosen by the cache length T, never by Q (batch invariance);
  // prefill tiles always take the online kernel
  if (T <= atc::kShortKeys && !tiles)
    return launch(atc::attention_tc_short_kernel, dim3(B, Hkv), dim3(atc::kShortThreads), atc::SmemShort::BYTES,
                  (cudaStream_t)stream, 1, tk, tv, (const __nv_bfloat16*)qkv, ldq, Q, H, Hkv, slot, start, T,
                  (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, scale * 1.4426950408889634f, append,
                  (const float2*)rope, (__nv_bfloat16*)out, ldo, block_table, max_blocks, block_size);
  const int qt = atc::kRows / (H / Hkv);
  return launch(D == 64 ? atc::attention_tc_kernel<64> : atc::attention_tc_kernel<128>, dim3(B, Hkv, (Q + qt - 1) / qt),
                dim3(atc::kThreadsOnline), atc::Smem::BYTES,
                (cudaStream_t)stream, 1, tk, tv, (const __nv_bfloat16*)qkv, ldq, Q, H, Hkv, slot, start, T,
                (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, scale * 1.4426950408889634f, append,
                (const float2*)rope, (__nv_bfloat16*)out, ldo, block_table, max_blocks, block_size);
}
