// K5 gate/up projection with more tiles than two CTAs per SM (the 70B verifier:
// 448 tiles of 128 rows = 1.51 waves of the 296 slots) as a persistent
// two-per-SM kernel: CTA c computes tiles c, c + P, ... (P = 2 x SMs), with a
// double-buffered TMEM accumulator so the gated epilogue of one tile runs
// while the TMA / MMA pipeline already streams the next.
//
// Why: a CTA's gated epilogue beside a co-resident CTA that is still
// streaming takes ~19 us at 112 token rows (TMEM reads and output stores queue
// behind the neighbour's weight stream; tools/epi_trace.py), and on the
// one-tile-per-CTA path it sits on each slot's critical path twice (first and
// second wave).  Here the first tile's epilogue overlaps the second tile's
// mainloop; the schedule (which CTA takes which tile) and every output's
// arithmetic are those of linear_kernel's one-split gated path — results are
// bitwise the same, a row's result never depends on M.
//
// The gate/up exchange goes through a 32-column chunk buffer (8 KB) instead of
// the whole-tile staging of linear_kernel (whose ring smem is busy here), and
// the gate warps store their outputs straight from registers.  Token tiles up
// to 128 columns (two accumulators fit the 256 TMEM columns of a CTA that
// shares the SM); wider tiles keep linear_kernel.
#pragma once
#include "gemm_kernel.cuh"

namespace ms {

template <int BN>
struct GatedCfg {
  static constexpr int W_BYTES = kBM * kBK * 2;
  static constexpr int X_BYTES = BN * kBK * 2;
  static constexpr int MAX_SW = 8;
  static constexpr int MAX_SX = 4;
  static constexpr int ACC = BN <= 32 ? 32 : BN <= 64 ? 64 : 128;
  static constexpr int TMEM_COLS = 2 * ACC;
  static constexpr int U_CHUNK = 32 * 64 * 4;  // one 32-column chunk of the up half, fp32
  // two chunk buffers (the up warps park chunk i + 1 while the gate warps
  // still read chunk i: one barrier per chunk) where two CTAs per SM still fit
  // beside the ring; BN = 128 keeps one (two barriers per chunk)
  static constexpr int U_BUFS = BN <= 112 ? 2 : 1;
  static constexpr int U_BYTES = U_BUFS * U_CHUNK;
  static constexpr int NBAR = 2 * MAX_SW + 2 * MAX_SX + 4;
  __host__ __device__ static void rings(int* sw, int* sx) {
    const int budget = 104 * 1024 - U_CHUNK;  // two CTAs per SM
    int x = X_BYTES <= 8192 ? 3 : 2;
    int w = (budget - x * X_BYTES) / W_BYTES;
    *sw = w < 2 ? 2 : (w > MAX_SW ? MAX_SW : w);
    *sx = x;
  }
  __host__ __device__ static int smem(int sw, int sx) {
    return 1024 + sw * W_BYTES + sx * X_BYTES + U_BYTES + NBAR * 8 + 16 + BN * 4;
  }
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 2)
linear_gated_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                    const LinearParams p) {
  using C = GatedCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int SW = p.sw, SX = p.sx;
  uint8_t* sW = smem;
  uint8_t* sX = smem + SW * C::W_BYTES;
  float* U = reinterpret_cast<float*>(sX + SX * C::X_BYTES);  // [32][64]
  uint64_t* fullW = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(U) + C::U_BYTES);
  uint64_t* emptyW = fullW + C::MAX_SW;
  uint64_t* fullX = emptyW + C::MAX_SW;
  uint64_t* emptyX = fullX + C::MAX_SX;
  uint64_t* tfull = emptyX + C::MAX_SX;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* s_rstd = reinterpret_cast<float*>(tmem_slot + 4);  // [BN]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int P = gridDim.x, c = blockIdx.x;
  const int m0 = blockIdx.y * BN;
  const int m_hi = min(BN, p.M - m0);
  const int nkb = p.kb_total;

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
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 128);
    }
    tc::fence_barrier_init();
  }
  __syncwarp();
  if (warp == 1) tc::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // weights do not depend on the previous kernel: the first SW tiles are
      // issued before the programmatic-dependency wait (PDL prefetch)
      const uint64_t pol_w = tc::policy_evict_first();
      int i = 0;
      bool waited = false;
      for (int t = c; t < p.n_tiles; t += P) {
        for (int kb = 0; kb < nkb; ++kb, ++i) {
          if (i == SW && !waited) {
            pdl_wait();
            pdl_trigger();
            waited = true;
          }
          const int st = i % SW;
          if (i >= SW) tc::mbar_wait(&emptyW[st], ((i / SW) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&fullW[st], C::W_BYTES);
          tc::tma_load_2d(sW + st * C::W_BYTES, &tmW, &fullW[st], kb * kBK, t * kBM, pol_w);
        }
      }
      if (!waited) {
        pdl_wait();
        pdl_trigger();
      }
    } else {
      pdl_trigger();
    }
  } else if (warp == 6) {
    if (lane == 0) {
      const uint64_t pol_x = tc::policy_evict_last();
      pdl_wait();
      pdl_trigger();
      int i = 0;
      for (int t = c; t < p.n_tiles; t += P) {
        for (int kb = 0; kb < nkb; ++kb, ++i) {
          const int st = i % SX;
          if (i >= SX) tc::mbar_wait(&emptyX[st], ((i / SX) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&fullX[st], C::X_BYTES);
          tc::tma_load_2d(sX + st * C::X_BYTES, &tmX, &fullX[st], kb * kBK, m0, pol_x);
        }
      }
    } else {
      pdl_trigger();
    }
  } else if (warp == 1) {
    pdl_trigger();
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(kBM, BN);
      int i = 0, s = 0;
      for (int t = c; t < p.n_tiles; t += P, ++s) {
        const int buf = s & 1;
        if (s >= 2) tc::mbar_wait(&tempty[buf], ((s >> 1) - 1) & 1);  // its previous epilogue drained it
        tc::fence_after_sync();
        const uint32_t acc = tmem + buf * C::ACC;
        for (int kb = 0; kb < nkb; ++kb, ++i) {
          const int ws = i % SW, xs = i % SX;
          tc::mbar_wait(&fullW[ws], (i / SW) & 1);
          tc::mbar_wait(&fullX[xs], (i / SX) & 1);
          tc::fence_after_sync();
          const uint64_t ad = tc::smem_desc_sw128(sW + ws * C::W_BYTES);
          const uint64_t bd = tc::smem_desc_sw128(sX + xs * C::X_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            tc::mma_bf16(acc, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          tc::mma_commit(&emptyW[ws]);
          tc::mma_commit(&emptyX[xs]);
        }
        tc::mma_commit(&tfull[buf]);
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5, TMEM lane quadrant = warp % 4 ----------
    const int q = warp & 3;
    const bool up = q >= 2;
    const int fu = (q & 1) * 32 + lane;  // gate / up feature within the 64-wide half
    pdl_wait();
    pdl_trigger();
    if (p.rms_in) {  // folded RMSNorm: the rows' rstd (as linear_kernel, fixed order)
      for (int r = q; r < m_hi; r += 4) {
        const float* pr = p.rms_in + (int64_t)(m0 + r) * p.rms_ld;
        float sq = 0.f;
        for (int u = lane; u < p.rms_nparts; u += 32) sq += pr[u];
        sq = warp_sum(sq);
        if (lane == 0) s_rstd[r] = rsqrtf(sq / (float)p.K + p.rms_eps);
      }
    }
    epi_bar128();
    int s = 0, chunk = 0;  // chunk: running count over tiles (U buffer = chunk % U_BUFS)
    for (int t = c; t < p.n_tiles; t += P, ++s) {
      const int buf = s & 1;
      tc::mbar_wait(&tfull[buf], (s >> 1) & 1);
      tc::fence_after_sync();
      const uint32_t trow = tmem + buf * C::ACC + ((uint32_t)(q * 32) << 16);
      __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)m0 * p.ldc + t * (kBM / 2) + fu;
      for (int c0 = 0; c0 < m_hi; c0 += 32, ++chunk) {
        float* Ub = U + (C::U_BUFS == 2 ? (chunk & 1) : 0) * (32 * 64);
        uint32_t r[32];
        tc::tmem_ld16(trow + c0, *reinterpret_cast<uint32_t(*)[16]>(r));
        tc::tmem_ld16(trow + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
        tc::tmem_wait_ld();
        if (up) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < m_hi) Ub[j * 64 + fu] = __uint_as_float(r[j]) * (p.rms_in ? s_rstd[c0 + j] : 1.f);
        }
        // with two buffers this one barrier also orders the gate warps' reads
        // of chunk - 2 (done before they arrived here) before its buffer is
        // rewritten (after it)
        epi_bar128();
        if (!up) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < m_hi)
              ob[(int64_t)(c0 + j) * p.ldc] =
                  f2bf(silu_mul(__uint_as_float(r[j]) * (p.rms_in ? s_rstd[c0 + j] : 1.f), Ub[j * 64 + fu]));
        }
        if (C::U_BUFS == 1) epi_bar128();  // U is rewritten by the next chunk
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&tempty[buf]);
    }
  }
  __syncwarp();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

template <int BN>
int launch_linear_gated(const CUtensorMap& tw, const CUtensorMap& tx, LinearParams p, int m_tiles, int P,
                        cudaStream_t st) {
  using C = GatedCfg<BN>;
  int sw, sx;
  C::rings(&sw, &sx);
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(linear_gated_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::smem(sw, sx)) != cudaSuccess)
      return MS_ERR_CUDA;
    attr_set = true;
  }
  p.sw = sw;
  p.sx = sx;
  return launch(linear_gated_kernel<BN>, dim3(P, m_tiles), dim3(kThreads), C::smem(sw, sx), st, 1, tw, tx, p);
}

template <int BN>
int preload_linear_gated() {
  return preload_fn(linear_gated_kernel<BN>);
}

#define MS_GATED_WIDTHS(X) X(16) X(32) X(48) X(64) X(80) X(96) X(112) X(128)
#define MS_GATED_DECLARE(BN)                                                                               \
  extern template int launch_linear_gated<BN>(const CUtensorMap&, const CUtensorMap&, LinearParams, int, int, \
                                              cudaStream_t);                                               \
  extern template int preload_linear_gated<BN>();
#define MS_GATED_INSTANTIATE(BN)                                                                        \
  template int launch_linear_gated<BN>(const CUtensorMap&, const CUtensorMap&, LinearParams, int, int, \
                                       cudaStream_t);                                                   \
  template int preload_linear_gated<BN>();

}  // namespace ms
