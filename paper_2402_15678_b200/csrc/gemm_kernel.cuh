// K1/K5/K8 — the linear layers of the SSM decode and the LLM verify forward on
// tcgen05 tensor cores (the kernel template; instantiated per token-tile width
// in gemm_inst*.cu so the build compiles them in parallel, host side in gemm.cu).
//
//   out[M, N] = epi( X[M, K] · W[N, K]^T )      X: tokens (bf16), W: weight (bf16)
//   epi(v)    = act(v + bias[n]) + residual[m, n]   -> bf16 or fp32
//   act 2 (gated SiLU, Llama's SwiGLU MLP): W = the gate and up projections
//   interleaved in 64-row blocks (rows 128t..128t+63 = gate rows 64t.., rows
//   128t+64.. = up rows 64t..), out[m, 64t + j] = silu(g) * u in fp32, one
//   bf16 rounding — the [M, 2F] gate/up activations never reach HBM.
//
// Decode/verify GEMMs have few token rows (M = B·(s+1) = 16..~300) against
// multi-GB weights: they are HBM-bound weight streams.  Layout "swap-AB": the
// weight tile is the MMA's M side (128 output features per CTA) and the token
// tile its N side (BN = 16..256), so a 16-row batch still issues full-height
// MMAs and TMEM holds a 128 x BN fp32 accumulator.
//
// Per CTA: warp 0 = TMA producer of the weight ring (128x64 tiles, 128B
// swizzle, mbarrier complete_tx; the first stages are issued before the
// programmatic-dependency wait, so weight streaming overlaps the previous
// kernel's tail), warp 6 = TMA producer of the token ring, warp 1 = TMEM
// allocator + single-thread tcgen05.mma issuer, warps 2-5 = epilogue
// (tcgen05.ld -> bias/act/residual -> global).  Split-K over the reduction
// dimension fills the 148 SMs: the `splits` CTAs of an output tile form one
// thread-block cluster and reduce their fp32 partial tiles through
// distributed shared memory (no global scratch, no extra launch), adding
// ranks in order — results are deterministic and, because the split count
// depends only on (N, K), identical for a token row whatever M is (batch
// invariance: a request's logits do not depend on what else is in the
// verify batch).
//
// (A tile-blocked weight layout — every 128 x 64 TMA tile one contiguous
// 16 KB run — measured no faster on the 70B shapes, profiles/
// r2_wblock_layout_ab.jsonl, and was not kept.)
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "tc.cuh"

namespace ms {

struct LinearParams {
  int M, N, K;
  const __nv_bfloat16* bias;      // [N] or null
  const __nv_bfloat16* residual;  // [M, ldr] or null
  int64_t ldr;
  void* out;                      // [M, ldc] bf16 or fp32
  int64_t ldc;
  int out_f32;
  int act;                        // 0 none, 1 relu, 2 gated SiLU (interleaved gate/up)
  int splits;
  int kb_total;                   // K / 64 (rounded up)
  int n_tiles;
  int sw, sx;                     // weight / token ring depths of this launch
  // tensor-parallel reduce-scatter fused into the epilogue: the fp32 value of
  // output (row m, feature f) is stored straight into the receive slot of the
  // rank owning f's column slice: tp_recv[f / tp_slice][(tp_rank * tp_rows +
  // m) * tp_slice + f % tp_slice] (peer memory over NVLink), tile by tile as
  // each CTA finishes, overlapping the transfer with other CTAs' mainloops
  float* const* tp_recv;
  int tp_rank, tp_slice, tp_rows;
  // RMSNorm folded across GEMMs (gains pre-multiplied into the consumer's
  // weight): a residual-writing split-K GEMM emits per-(row, tile) sums of
  // squares of the bf16 values it stores (rms_out[row * rms_ld + tile], a row's
  // partials contiguous); the next GEMM runs on the raw residual stream and
  // scales its fp32 accumulator by rstd[row] = rsqrt(sum_t rms_in[row * rms_ld
  // + t] / K + eps).
  float* rms_out;
  const float* rms_in;
  int rms_nparts;
  int64_t rms_ld;
  float rms_eps;
};

constexpr int kBM = 128;       // output features per CTA (MMA M)
constexpr int kBK = 64;        // bf16 elements per 128-byte swizzled row
constexpr int kThreads = 224;  // W producer, MMA, 4 epilogue warps, X producer

template <int BN>
struct LinearCfg {
  static constexpr int W_BYTES = kBM * kBK * 2;
  static constexpr int X_BYTES = BN * kBK * 2;
  static constexpr int MAX_SW = 14;
  static constexpr int MAX_SX = 6;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int PART_BYTES = BN * kBM * 4;  // fp32 partial tile for the split-K reduction
  static constexpr int NBAR = 2 * MAX_SW + 2 * MAX_SX + 1;  // mbarriers
  // Two decoupled TMA rings: the weight ring (HBM stream — its depth is the
  // bytes in flight that bound a weight stream by Little's law, ~6.5 TB/s x
  // ~2 us per GPU) and a shallow token ring (the X tile is re-read by every
  // CTA, an L2 hit).  Budget: ~210 KB at one CTA per SM, ~104 KB at two.
  __host__ __device__ static void rings_for(int budget, int* sw, int* sx) {
    int x = budget >= 150 * 1024 ? 4 : (X_BYTES <= 8192 ? 3 : 2);
    int w = (budget - x * X_BYTES) / W_BYTES;
    if (w < 3 && x > 2) {
      x = 2;
      w = (budget - x * X_BYTES) / W_BYTES;
    }
    *sw = w < 2 ? 2 : (w > MAX_SW ? MAX_SW : w);
    *sx = x > MAX_SX ? MAX_SX : x;
  }
  // the fp32 partial tile is staged in the (idle) ring smem only for the
  // split-K cluster reduction; the single-split gated epilogue exchanges
  // gate/up through smem as well
  // up half [BN][65] fp32, then the bf16 output tile [BN][64]
  static constexpr int O_OFF = BN * 65 * 4;
  static constexpr int GATED_EPI_BYTES = O_OFF + BN * 64 * 2;
  __host__ __device__ static int data_bytes(int sw, int sx, bool part) {
    const int pipe = sw * W_BYTES + sx * X_BYTES;
    int need = part ? PART_BYTES : GATED_EPI_BYTES;
    if (need < GATED_EPI_BYTES) need = GATED_EPI_BYTES;
    return pipe > need ? pipe : need;
  }
  __host__ __device__ static int smem(int sw, int sx, bool part) {
    return 1024 + data_bytes(sw, sx, part) + NBAR * 8 + 16 + BN * 4;
  }
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// tok: global output row; feat: feature within the row group grp.  Returns
// the value as stored (bf16-rounded for bf16 outputs).
__device__ __forceinline__ float epi_store(const LinearParams& p, int tok, int feat, float v, int grp = 0) {
  if (p.bias) v += bf2f(p.bias[(int64_t)grp * p.N + feat]);
  if (p.act == 1) v = fmaxf(v, 0.0f);
  if (p.residual) v += bf2f(p.residual[(int64_t)tok * p.ldr + feat]);
  if (p.tp_recv) {  // reduce-scatter: fp32 partial into the owning rank's receive slot
    const int dst = feat / p.tp_slice;
    p.tp_recv[dst][((int64_t)p.tp_rank * p.tp_rows + tok) * p.tp_slice + (feat - dst * p.tp_slice)] = v;
    return v;
  }
  if (p.out_f32) {
    reinterpret_cast<float*>(p.out)[(int64_t)tok * p.ldc + feat] = v;
    return v;
  }
  const __nv_bfloat16 b = f2bf(v);
  reinterpret_cast<__nv_bfloat16*>(p.out)[(int64_t)tok * p.ldc + feat] = b;
  return bf2f(b);
}

__device__ __forceinline__ void epi_bar128() { asm volatile("bar.sync 1, 128;" ::: "memory"); }


__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// float4 load from the shared memory of CTA `rank` of this cluster
__device__ __forceinline__ float4 ld_dsmem_f4(const float* local, int rank) {
  uint32_t a = tc::smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra) : "memory");
  return v;
}

template <int BN>
// minBlocks 2: two CTAs per SM must fit the register file (<= 146 registers
// per thread at 224 threads) — the decode / verify GEMMs run at two CTAs per
// SM, and a register-limited single CTA per SM cost 35-55% of their speed
// (tools/ab_lib_gemm.py, round 2)
__global__ void __launch_bounds__(kThreads, 2)
linear_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
              const LinearParams p) {
  using C = LinearCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  const int SW = p.sw, SX = p.sx;
  uint8_t* sX = smem + SW * C::W_BYTES;
  uint64_t* fullW = reinterpret_cast<uint64_t*>(smem + C::data_bytes(SW, SX, p.splits > 1));
  uint64_t* emptyW = fullW + C::MAX_SW;
  uint64_t* fullX = emptyW + C::MAX_SW;
  uint64_t* emptyX = fullX + C::MAX_SX;
  uint64_t* tmem_full = emptyX + C::MAX_SX;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  float* s_rstd = reinterpret_cast<float*>(tmem_slot + 4);  // [BN]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // cluster = the `splits` K-slices of one output tile; rank = split
  const int split = (int)(blockIdx.x % p.splits);
  const int tile_n = (int)(blockIdx.x / p.splits);
  const int n0 = tile_n * kBM;
  const int m0 = blockIdx.y * BN;
  // row group (grouped drafters): M rows of X / out and N rows of W per group
  const int grp = blockIdx.z;
  const int wrow = grp * p.N + n0, xrow = grp * p.M + m0, orow = grp * p.M + m0;
  const int kb0 = (int)((int64_t)split * p.kb_total / p.splits);
  const int kb1 = (int)((int64_t)(split + 1) * p.kb_total / p.splits);

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmW);
    tc::prefetch_tmap(&tmX);
    for (int s = 0; s < SW; ++s) {
      tc::mbar_init(&fullW[s], 1);
      tc::mbar_init(&emptyW[s], 1);
    }
    for (int s = 0; s < SX; ++s) {
      tc::mbar_init(&fullX[s], 1);
      tc::mbar_init(&emptyX[s], 1);
    }
    tc::mbar_init(tmem_full, 1);
    tc::fence_barrier_init();
  }
  __syncwarp();  // lane 0 of warp 0 diverged above: reconverge before the aligned barrier
  if (warp == 1) tc::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int nkb = kb1 - kb0;
  if (warp == 0) {
    if (lane == 0) {
      // weight producer: the first SW weight tiles do not depend on the previous
      // kernel — issued before the programmatic-dependency wait (PDL prefetch)
      const uint64_t pol_w = tc::policy_evict_first();  // weights stream through once
      const int pre = nkb < SW ? nkb : SW;
      for (int i = 0; i < pre; ++i) {
        tc::mbar_arrive_expect_tx(&fullW[i], C::W_BYTES);
        tc::tma_load_2d(sW + i * C::W_BYTES, &tmW, &fullW[i], (kb0 + i) * kBK, wrow, pol_w);
      }
      pdl_wait();
      pdl_trigger();
      for (int i = pre; i < nkb; ++i) {
        const int st = i % SW;
        tc::mbar_wait(&emptyW[st], ((i / SW) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&fullW[st], C::W_BYTES);
        tc::tma_load_2d(sW + st * C::W_BYTES, &tmW, &fullW[st], (kb0 + i) * kBK, wrow, pol_w);
      }
    } else {
      pdl_trigger();
    }
  } else if (warp == 6) {
    if (lane == 0) {
      // token producer (the X tile depends on the previous kernel)
      const uint64_t pol_x = tc::policy_evict_last();  // tokens are re-read by every tile
      pdl_wait();
      pdl_trigger();
      for (int i = 0; i < nkb; ++i) {
        const int st = i % SX;
        if (i >= SX) tc::mbar_wait(&emptyX[st], ((i / SX) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&fullX[st], C::X_BYTES);
        tc::tma_load_2d(sX + st * C::X_BYTES, &tmX, &fullX[st], (kb0 + i) * kBK, xrow, pol_x);
      }
    } else {
      pdl_trigger();
    }
  } else if (warp == 1) {
    pdl_trigger();
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(kBM, BN);
      for (int i = 0; i < nkb; ++i) {
        const int ws = i % SW, xs = i % SX;
        tc::mbar_wait(&fullW[ws], (i / SW) & 1);
        tc::mbar_wait(&fullX[xs], (i / SX) & 1);
        tc::fence_after_sync();
        const uint64_t ad = tc::smem_desc_sw128(sW + ws * C::W_BYTES);
        const uint64_t bd = tc::smem_desc_sw128(sX + xs * C::X_BYTES);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)  // +32 bytes along K per UMMA_K=16 step
          tc::mma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
        tc::mma_commit(&emptyW[ws]);
        tc::mma_commit(&emptyX[xs]);
      }
      tc::mma_commit(tmem_full);
    }
  } else {
    // ---------------- epilogue: warps 2..5, TMEM lane quadrant = warp % 4 ----------
    const int q = warp & 3;
    const int feat = n0 + q * 32 + lane;
    const bool feat_ok = feat < p.N;
    const int m_hi = min(BN, p.M - m0);  // valid token columns in this tile
    pdl_wait();  // residual / outputs are ordered after the previous kernel
    pdl_trigger();
    if (p.rms_in) {
      // folded RMSNorm: this tile's rows' rstd from the producer's partials
      // (fixed summation order), while the mainloop runs; one warp per row:
      // lanes take partials l, l+32, ... (coalesced), then a fixed shuffle tree
      for (int r = q; r < m_hi; r += 4) {
        const float* pr = p.rms_in + (int64_t)(orow + r) * p.rms_ld;
        float sq = 0.f;
        for (int t = lane; t < p.rms_nparts; t += 32) sq += pr[t];
        sq = warp_sum(sq);
        if (lane == 0) s_rstd[r] = rsqrtf(sq / (float)p.K + p.rms_eps);
      }
      epi_bar128();
    }
    tc::mbar_wait(tmem_full, 0);
    tc::fence_after_sync();
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);

    if (p.splits == 1 && p.act == 2) {
      // gated SiLU, one split (the pipeline smem is idle once tmem_full fired):
      // (1) the up warps (TMEM lanes 64..127) park the whole up half in smem,
      // (2) one barrier, the gate warps form silu(g) * u into a bf16 output
      // tile in smem, (3) one barrier, all four warps store the tile with
      // coalesced 16-byte writes.
      float* U = reinterpret_cast<float*>(smem);                                // [BN][65] fp32
      __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(smem + C::O_OFF);    // [BN][64] bf16
      const bool up = q >= 2;
      const int f = (q & 1) * 32 + lane;  // gate / up feature within the 64-wide half
      for (int c0 = 0; c0 < m_hi; c0 += 32) {
        uint32_t r[32];
        tc::tmem_ld16(trow + c0, *reinterpret_cast<uint32_t(*)[16]>(r));
        tc::tmem_ld16(trow + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
        tc::tmem_wait_ld();
        if (up) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < m_hi) U[(c0 + j) * 65 + f] = __uint_as_float(r[j]) * (p.rms_in ? s_rstd[c0 + j] : 1.f);
        }
      }
      epi_bar128();
      // the gate warps read their TMEM half after the barrier (re-loading is
      // cheaper than holding up to 256 columns in registers)
      if (!up) {
        for (int c0 = 0; c0 < m_hi; c0 += 32) {
          uint32_t r[32];
          tc::tmem_ld16(trow + c0, *reinterpret_cast<uint32_t(*)[16]>(r));
          tc::tmem_ld16(trow + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
          tc::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < m_hi)
              O[(c0 + j) * 64 + f] = f2bf(silu_mul(__uint_as_float(r[j]) * (p.rms_in ? s_rstd[c0 + j] : 1.f),
                                                   U[(c0 + j) * 65 + f]));
        }
      }
      epi_bar128();
      const int et = threadIdx.x - 64;  // 0..127
      __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)orow * p.ldc + tile_n * (kBM / 2);
      for (int e = et; e < m_hi * 8; e += 128) {
        const int row = e >> 3, ch = e & 7;
        *reinterpret_cast<uint4*>(ob + (int64_t)row * p.ldc + ch * 8) =
            *reinterpret_cast<const uint4*>(O + row * 64 + ch * 8);
      }
    } else if (p.splits == 1) {
      for (int c0 = 0; c0 < m_hi; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(trow + c0, r);
        tc::tmem_wait_ld();
        if (feat_ok) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < m_hi)
              epi_store(p, orow + c0 + j, feat, __uint_as_float(r[j]) * (p.rms_in ? s_rstd[c0 + j] : 1.f), grp);
        }
      }
    } else {
      // stage this split's fp32 partial tile in (now idle) pipeline smem,
      // layout P[token][feature] so a warp's 32 lanes write 32 consecutive words
      float* P = reinterpret_cast<float*>(smem);
      for (int c0 = 0; c0 < m_hi; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(trow + c0, r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) P[(c0 + j) * kBM + q * 32 + lane] = __uint_as_float(r[j]);
      }
    }
  }
  __syncwarp();  // producer / MMA roles ran on lane 0: reconverge before the aligned cluster / CTA barriers
  if (p.splits > 1) {
    pdl_wait();  // warps 0-1 also run the epilogue below (residual reads)
    // split-K reduction across the thread-block cluster through DSMEM: CTA
    // `split` reduces a 1/splits slice of the tile, adding the partials of
    // ranks 0..splits-1 in rank order (deterministic), then runs the epilogue.
    // Gated SiLU: a unit covers gate features f4..f4+3 and their up partners
    // f4+64.. of the same (staged) tile.
    cluster_sync_all();
    const int m_hi = min(BN, p.M - m0);
    const bool gated = p.act == 2;
    const int upr = (gated ? kBM / 2 : kBM) / 4;  // float4 units per token row
    const int units = m_hi * upr;
    const int u0 = (int)((int64_t)split * units / p.splits);
    const int u1 = (int)((int64_t)(split + 1) * units / p.splits);
    const float* P = reinterpret_cast<const float*>(smem);
    if (p.rms_out && !gated) {
      // residual producer of a folded RMSNorm: token-granular slices, one warp
      // per token row, lane l = features 4l..4l+3; the row's sum of squares of
      // the stored bf16 values over this tile's 128 features is a fixed-order
      // warp reduction written to its own (tile, row) slot — deterministic
      const int t0 = split * m_hi / p.splits, t1 = (split + 1) * m_hi / p.splits;
      const int f4 = lane * 4;
      const int feat = n0 + f4;
      const bool vec = (p.N % 4 == 0) && (p.ldc % 4 == 0) && (!p.residual || p.ldr % 4 == 0) && !p.tp_recv &&
                       !p.out_f32 && ((reinterpret_cast<uintptr_t>(p.out) & 7) == 0) &&
                       ((reinterpret_cast<uintptr_t>(p.residual) & 7) == 0) && !p.bias;
      if (vec && p.splits <= 4) {
        // RB rows per warp at once: every partial (DSMEM) and residual load of
        // the batch is issued before the first add — one latency per batch
        // instead of (splits + 1) per row; the same additions in the same
        // (rank) order and the same stores / sums of squares as epi_store
        constexpr int RB = 4;
        constexpr int W = kThreads / 32;
        for (int jb = t0 + warp; jb < t1; jb += W * RB) {
          float4 part[RB][4];
          uint2 res[RB];
#pragma unroll
          for (int i = 0; i < RB; ++i) {
            const int j = jb + i * W;
            if (j < t1) {
#pragma unroll
              for (int rk = 0; rk < 4; ++rk)
                if (rk < p.splits) part[i][rk] = ld_dsmem_f4(P + j * kBM + f4, rk);
              if (p.residual && feat < p.N)
                res[i] = *reinterpret_cast<const uint2*>(p.residual + (int64_t)(orow + j) * p.ldr + feat);
            }
          }
#pragma unroll
          for (int i = 0; i < RB; ++i) {
            const int j = jb + i * W;
            if (j >= t1) break;  // warp-uniform
            float4 acc = part[i][0];
#pragma unroll
            for (int rk = 1; rk < 4; ++rk)
              if (rk < p.splits) {
                acc.x += part[i][rk].x; acc.y += part[i][rk].y; acc.z += part[i][rk].z; acc.w += part[i][rk].w;
              }
            const float rs = p.rms_in ? s_rstd[j] : 1.f;
            float v4[4] = {acc.x * rs, acc.y * rs, acc.z * rs, acc.w * rs};
            float sq = 0.f;
            if (feat < p.N) {
              if (p.act == 1) {
#pragma unroll
                for (int t = 0; t < 4; ++t) v4[t] = fmaxf(v4[t], 0.0f);
              }
              if (p.residual) {
                const __nv_bfloat162* rr = reinterpret_cast<const __nv_bfloat162*>(&res[i]);
                const float2 r01 = __bfloat1622float2(rr[0]), r23 = __bfloat1622float2(rr[1]);
                v4[0] += r01.x; v4[1] += r01.y; v4[2] += r23.x; v4[3] += r23.y;
              }
              __nv_bfloat16 b[4];
#pragma unroll
              for (int t = 0; t < 4; ++t) b[t] = f2bf(v4[t]);
              uint2 pk;
              pk.x = (uint32_t)__bfloat16_as_ushort(b[0]) | ((uint32_t)__bfloat16_as_ushort(b[1]) << 16);
              pk.y = (uint32_t)__bfloat16_as_ushort(b[2]) | ((uint32_t)__bfloat16_as_ushort(b[3]) << 16);
              *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)(orow + j) * p.ldc + feat) = pk;
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float st = bf2f(b[t]);
                sq += st * st;
              }
            }
            sq = warp_sum(sq);
            if (lane == 0) p.rms_out[(int64_t)(orow + j) * p.rms_ld + tile_n] = sq;
          }
        }
      } else
      for (int j = t0 + warp; j < t1; j += kThreads / 32) {
        float4 acc = ld_dsmem_f4(P + j * kBM + f4, 0);
        for (int rk = 1; rk < p.splits; ++rk) {
          const float4 v = ld_dsmem_f4(P + j * kBM + f4, rk);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        const float rs = p.rms_in ? s_rstd[j] : 1.f;
        const float a4[4] = {acc.x * rs, acc.y * rs, acc.z * rs, acc.w * rs};
        float sq = 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (feat + t < p.N) {
            const float st = epi_store(p, orow + j, feat + t, a4[t], grp);
            sq += st * st;
          }
        sq = warp_sum(sq);
        if (lane == 0) p.rms_out[(int64_t)(orow + j) * p.rms_ld + tile_n] = sq;
      }
    } else if (!gated) {
      // batched for memory-level parallelism: each thread holds up to UB of
      // its units, issues every partial (DSMEM) and residual load first, then
      // computes and stores 4-wide — one latency per batch instead of one per
      // unit (the unbatched loop cost ~12 us on a 176-row O projection, half
      // of its mainloop)
      constexpr int UB = 8;
      const bool vec = (p.N % 4 == 0) && (p.ldc % 4 == 0) && (!p.residual || p.ldr % 4 == 0) && !p.tp_recv &&
                       ((reinterpret_cast<uintptr_t>(p.out) & (p.out_f32 ? 15 : 7)) == 0) &&
                       ((reinterpret_cast<uintptr_t>(p.residual) & 7) == 0) && !p.bias;
      // one unit's epilogue: rstd, act, residual, 4-wide store
      auto finish = [&](int u, const float4& acc, const uint2& res) {
        const int j = u / upr, f4 = (u - j * upr) * 4;
        const float rs = p.rms_in ? s_rstd[j] : 1.f;
        float a4[4] = {acc.x * rs, acc.y * rs, acc.z * rs, acc.w * rs};
        const int feat = n0 + f4;
        if (vec && feat < p.N) {
          if (p.act == 1) {
#pragma unroll
            for (int t = 0; t < 4; ++t) a4[t] = fmaxf(a4[t], 0.f);
          }
          if (p.residual) {
            const __nv_bfloat162* rr = reinterpret_cast<const __nv_bfloat162*>(&res);
            const float2 r01 = __bfloat1622float2(rr[0]), r23 = __bfloat1622float2(rr[1]);
            a4[0] += r01.x; a4[1] += r01.y; a4[2] += r23.x; a4[3] += r23.y;
          }
          if (p.out_f32) {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + (int64_t)(orow + j) * p.ldc + feat) =
                make_float4(a4[0], a4[1], a4[2], a4[3]);
          } else {
            uint2 pk;
            pk.x = pack_bf16x2(a4[0], a4[1]);
            pk.y = pack_bf16x2(a4[2], a4[3]);
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)(orow + j) * p.ldc + feat) = pk;
          }
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (feat + t < p.N) epi_store(p, orow + j, feat + t, a4[t], grp);
        }
      };
      if (p.splits <= 4) {
        // 4 units per thread with every rank's partial (DSMEM) and the residual
        // loaded before the first add: one latency per batch; the additions in
        // rank order as below
        constexpr int UW = 4;
        for (int ub = u0 + (int)threadIdx.x; ub < u1; ub += kThreads * UW) {
          float4 part[UW][4];
          uint2 res[UW];
#pragma unroll
          for (int i = 0; i < UW; ++i) {
            const int u = ub + i * kThreads;
            if (u < u1) {
              const int j = u / upr, f4 = (u - j * upr) * 4;
#pragma unroll
              for (int rk = 0; rk < 4; ++rk)
                if (rk < p.splits) part[i][rk] = ld_dsmem_f4(P + j * kBM + f4, rk);
              if (vec && p.residual && n0 + f4 < p.N)
                res[i] = *reinterpret_cast<const uint2*>(p.residual + (int64_t)(orow + j) * p.ldr + n0 + f4);
            }
          }
#pragma unroll
          for (int i = 0; i < UW; ++i) {
            const int u = ub + i * kThreads;
            if (u >= u1) continue;
            float4 acc = part[i][0];
#pragma unroll
            for (int rk = 1; rk < 4; ++rk)
              if (rk < p.splits) {
                acc.x += part[i][rk].x; acc.y += part[i][rk].y; acc.z += part[i][rk].z; acc.w += part[i][rk].w;
              }
            finish(u, acc, res[i]);
          }
        }
      } else
      for (int ub = u0 + (int)threadIdx.x; ub < u1; ub += kThreads * UB) {
        float4 acc[UB];
        uint2 res[UB];
#pragma unroll
        for (int i = 0; i < UB; ++i) {
          const int u = ub + i * kThreads;
          if (u < u1) {
            const int j = u / upr, f4 = (u - j * upr) * 4;
            acc[i] = ld_dsmem_f4(P + j * kBM + f4, 0);
            if (vec && p.residual && n0 + f4 < p.N)
              res[i] = *reinterpret_cast<const uint2*>(p.residual + (int64_t)(orow + j) * p.ldr + n0 + f4);
          }
        }
        for (int rk = 1; rk < p.splits; ++rk) {
#pragma unroll
          for (int i = 0; i < UB; ++i) {
            const int u = ub + i * kThreads;
            if (u < u1) {
              const int j = u / upr, f4 = (u - j * upr) * 4;
              const float4 v = ld_dsmem_f4(P + j * kBM + f4, rk);
              acc[i].x += v.x; acc[i].y += v.y; acc[i].z += v.z; acc[i].w += v.w;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < UB; ++i) {
          const int u = ub + i * kThreads;
          if (u < u1) finish(u, acc[i], res[i]);
        }
      }
    } else {
      for (int u = u0 + (int)threadIdx.x; u < u1; u += kThreads) {
        const int j = u / upr;
        const int f4 = (u - j * upr) * 4;
        const float rs = p.rms_in ? s_rstd[j] : 1.f;
        float4 acc = ld_dsmem_f4(P + j * kBM + f4, 0);
        for (int rk = 1; rk < p.splits; ++rk) {
          const float4 v = ld_dsmem_f4(P + j * kBM + f4, rk);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        const float a4[4] = {acc.x * rs, acc.y * rs, acc.z * rs, acc.w * rs};
        float4 up = ld_dsmem_f4(P + j * kBM + f4 + kBM / 2, 0);
        for (int rk = 1; rk < p.splits; ++rk) {
          const float4 v = ld_dsmem_f4(P + j * kBM + f4 + kBM / 2, rk);
          up.x += v.x; up.y += v.y; up.z += v.z; up.w += v.w;
        }
        const float u4[4] = {up.x * rs, up.y * rs, up.z * rs, up.w * rs};
        const int of = tile_n * (kBM / 2) + f4;  // output feature
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)(orow + j) * p.ldc + of;
#pragma unroll
        for (int t = 0; t < 4; ++t) o[t] = f2bf(silu_mul(a4[t], u4[t]));
      }
    }
    cluster_sync_all();  // peers may still be reading this CTA's smem
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// Launch one linear_kernel<BN> (host).  Ring depths per launch: ~210 KB of
// stages when the grid fits one CTA per SM, ~104 KB at two per SM, never more
// stages than k-blocks per CTA (so small drafter GEMMs leave shared memory
// for concurrent kernels).
template <int BN>
int launch_linear(const CUtensorMap& tw, const CUtensorMap& tx, LinearParams p, int m_tiles, cudaStream_t st,
                  int G) {
  using C = LinearCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    int sw, sx;
    C::rings_for(210 * 1024, &sw, &sx);
    if (cudaFuncSetAttribute(linear_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::smem(sw, sx, true)) != cudaSuccess)
      return MS_ERR_CUDA;
    attr_set = true;
  }
  const int grid = p.n_tiles * p.splits * m_tiles * G;
  const int kb_per_cta = (p.kb_total + p.splits - 1) / p.splits;
  const bool part = p.splits > 1;
  int sw, sx;
  C::rings_for(grid <= 148 ? 210 * 1024 : 104 * 1024, &sw, &sx);
  // the fp32 split-K staging tile may already rule out two CTAs per SM: then
  // take the deep single-CTA rings
  if (part && C::smem(sw, sx, part) > 113 * 1024) C::rings_for(210 * 1024, &sw, &sx);
  if (sw > kb_per_cta) sw = kb_per_cta < 2 ? 2 : kb_per_cta;
  if (sx > kb_per_cta) sx = kb_per_cta < 2 ? 2 : kb_per_cta;
  p.sw = sw;
  p.sx = sx;
  return launch(linear_kernel<BN>, dim3(p.n_tiles * p.splits, m_tiles, G), dim3(kThreads), C::smem(sw, sx, part),
                st, p.splits /* the split-K CTAs of a tile form one cluster */, tw, tx, p);
}

template <int BN>
int preload_linear() {
  return preload_fn(linear_kernel<BN>);
}

// Instantiated in gemm_inst*.cu (one translation unit per group of widths).
#define MS_LINEAR_WIDTHS(X) X(16) X(32) X(48) X(64) X(80) X(96) X(112) X(128) X(144) X(160) X(176) X(192) \
  X(208) X(224) X(240) X(256)
#define MS_LINEAR_DECLARE(BN)                                                                         \
  extern template int launch_linear<BN>(const CUtensorMap&, const CUtensorMap&, LinearParams, int,      \
                                        cudaStream_t, int);                                             \
  extern template int preload_linear<BN>();
#define MS_LINEAR_INSTANTIATE(BN)                                                                     \
  template int launch_linear<BN>(const CUtensorMap&, const CUtensorMap&, LinearParams, int, cudaStream_t, \
                                 int);                                                                  \
  template int preload_linear<BN>();

}  // namespace ms
