// ms_linear_wide — the compute-bound linear layer (prompt prefill, M >= 256
// token rows) on CTA pairs: tcgen05.mma.cta_group::2 with a 256-feature x
// BN-token tile per pair, persistent over tiles.
//
//   out[M, N] = epi( X[M, K] · W[N, K]^T ),  epi as ms_linear (bias, ReLU,
//   residual, gated SiLU over the 64-row interleaved gate/up weight, bf16 or
//   fp32 out)
//
// Swap-AB as in ms_linear: the weight is the MMA's M side.  A CTA pair (a
// 2-CTA cluster on one TPC) owns output tiles of 256 features x BN tokens:
// CTA r loads weight rows n0 + 128 r .. (its half of A) and token rows m0 +
// r BN/2 .. (its half of B) per 64-deep k-block, both TMA loads completing on
// the LEADER's full barrier; the leader's single MMA thread issues
// tcgen05.mma.cta_group::2 (M = 256, N = BN) reading both CTAs' shared
// memory, and each CTA's TMEM receives its 128 features x BN tokens.  So per
// SM the shared-memory operand traffic per MMA is halved against the 1-CTA
// 128-row MMA (the tensor pipe's pacing floor is met, B300_MICROARCH.md
// "tcgen05 floor"), and each CTA fetches only half of the token tile.
//
// Persistent: one pair per TPC (grid = 2 x pairs), pair c walks tiles c, c +
// P, ... with the token tiles of one weight tile consecutive (the pairs
// running at the same time share the weight tile through L2: weights are
// read ~once from HBM).  TMEM holds two accumulators (2 x BN columns): the
// epilogue of tile t (4 warps per CTA: tcgen05.ld -> smem -> 16-byte vector
// stores, residual read 16 bytes at a time) overlaps the mainloop of t + 1.
//
// Deterministic (fixed k order, no split-K); not the decode / verify path,
// whose per-row results must not depend on M (ms_linear's fixed split-K) —
// this kernel serves prompt prefill, where the greedy teacher and the
// speculative run share the same prefill.
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc.cuh"

namespace ms {
namespace pair {

constexpr int kBK = 64;
constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA (+ TMEM), warps 2..5 epilogue
constexpr int kStages = 6;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the pair leader's copy

struct Params {
  int M, N, K;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int64_t ldr;
  void* out;
  int64_t ldc;
  int out_f32;
  int act;
  int kb_total;
  int n_tiles, m_tiles;  // 256-feature tiles, BN-token tiles
};

template <int BN>
struct Cfg {
  static constexpr int W_BYTES = 128 * kBK * 2;        // this CTA's half of the weight tile
  static constexpr int X_BYTES = (BN / 2) * kBK * 2;   // this CTA's half of the token tile
  static constexpr int STAGE = W_BYTES + X_BYTES;
  static constexpr int EPI_BYTES = 32 * 129 * 4;       // [32 tokens][128 features] fp32 (+1 pad)
  static constexpr int SMEM = 1024 + kStages * STAGE + EPI_BYTES + (2 * kStages + 4) * 8 + 16;
};

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 2-CTA TMA: lands in this CTA's smem, completes tx bytes on the leader's barrier
__device__ __forceinline__ void tma_load_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar) & kPeerMask), "r"(x), "r"(y), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// arrive on `bar` (same offset) in both CTAs of the pair once the issued MMAs are done
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          tc::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// arrive on the pair leader's copy of `bar` (release at cluster scope)
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  uint32_t a = tc::smem_u32(bar), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(a));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = tc::smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    wide_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, const Params p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  float* epi = reinterpret_cast<float*>(smem + kStages * C::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::STAGE + C::EPI_BYTES);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [2] accumulator ready (both CTAs, from the leader's commit)
  uint64_t* tempty = tfull + 2;        // [2] accumulator drained (leader's copy: 8 epilogue-warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int total = p.n_tiles * p.m_tiles;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmW);
    tc::prefetch_tmap(&tmX);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 8);
    }
    tc::fence_barrier_init();
  }
  __syncwarp();
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "n"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_before_sync();
  cluster_sync();  // barriers and the TMEM address exist in both CTAs
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = tc::policy_evict_first();
      const uint64_t pol_x = tc::policy_evict_last();
      pdl_wait();
      int it = 0;
      for (int t = pair_id; t < total; t += n_pairs) {
        const int nt = t / p.m_tiles, mt = t - nt * p.m_tiles;
        const int wy = nt * 256 + (int)rank * 128, xy = mt * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < p.kb_total; ++kb, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          tc::mbar_wait(&empty[s], ph ^ 1);
          if (leader) tc::mbar_arrive_expect_tx(&full[s], 2 * C::STAGE);
          uint8_t* sb = stage_base + s * C::STAGE;
          tma_load_pair(sb, &tmW, &full[s], kb * kBK, wy, pol_w);
          tma_load_pair(sb + C::W_BYTES, &tmX, &full[s], kb * kBK, xy, pol_x);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(256, BN);
      int it = 0, j = 0;
      for (int t = pair_id; t < total; t += n_pairs, ++j) {
        const int a = j & 1;
        wait_cluster(&tempty[a], ((j >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t d = tmem + (uint32_t)(a * BN);
        for (int kb = 0; kb < p.kb_total; ++kb, ++it) {
          const int s = it % kStages;
          tc::mbar_wait(&full[s], (it / kStages) & 1);
          tc::fence_after_sync();
          uint8_t* sb = stage_base + s * C::STAGE;
          const uint64_t ad = tc::smem_desc_sw128(sb);
          const uint64_t bd = tc::smem_desc_sw128(sb + C::W_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) mma_pair(d, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          commit_pair(&empty[s]);
        }
        commit_pair(&tfull[a]);
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 (TMEM lane quadrant = warp % 4) -----------
    const int q = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    const bool gated = p.act == 2;
    pdl_wait();
    int j = 0;
    for (int t = pair_id; t < total; t += n_pairs, ++j) {
      const int a = j & 1;
      const int nt = t / p.m_tiles, mt = t - nt * p.m_tiles;
      const int f0 = nt * 256 + (int)rank * 128;  // this CTA's first weight row
      const int m0 = mt * BN;
      tc::mbar_wait(&tfull[a], (j >> 1) & 1);
      tc::fence_after_sync();
      const uint32_t trow = tmem + (uint32_t)(a * BN) + ((uint32_t)(q * 32) << 16);
      const int m_hi = min(BN, p.M - m0);
      for (int c0 = 0; c0 < m_hi; c0 += 32) {
        uint32_t r[32];
        tc::tmem_ld16(trow + c0, *reinterpret_cast<uint32_t(*)[16]>(r));
        tc::tmem_ld16(trow + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
        tc::tmem_wait_ld();
        if (c0 + 32 >= m_hi) {  // this warp is done with the accumulator: release it to the MMA
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) arrive_leader(&tempty[a]);
          __syncwarp();
        }
        // stage [32 tokens][128 features] fp32, feature = q*32 + lane
#pragma unroll
        for (int i = 0; i < 32; ++i) epi[i * 129 + q * 32 + lane] = __uint_as_float(r[i]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (gated) {
          // gate rows 0..63, up rows 64..127 of this CTA's weight half -> 64 outputs
          const int of0 = (f0 >> 1);  // output feature of gate row f0 (64-row interleave)
          for (int u = et; u < 32 * 8; u += 128) {  // (token, 8-feature group)
            const int i = u >> 3, g8 = (u & 7) * 8;
            const int tok = m0 + c0 + i;
            if (tok < p.M && of0 + g8 < p.N / 2) {
              float o[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = silu_mul(epi[i * 129 + g8 + e], epi[i * 129 + 64 + g8 + e]);
              *reinterpret_cast<bf16x8*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)tok * p.ldc + of0 + g8) =
                  pack8(o);
            }
          }
        } else {
          for (int u = et; u < 32 * 16; u += 128) {  // (token, 8-feature group)
            const int i = u >> 4, g8 = (u & 15) * 8;
            const int tok = m0 + c0 + i, f = f0 + g8;
            if (tok >= p.M || f >= p.N) continue;
            float o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = epi[i * 129 + g8 + e];
            const bool full8 = f + 8 <= p.N;
            if (p.bias) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (f + e < p.N) o[e] += bf2f(p.bias[f + e]);
            }
            if (p.act == 1) {
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = fmaxf(o[e], 0.f);
            }
            if (p.residual) {
              const __nv_bfloat16* rp = p.residual + (int64_t)tok * p.ldr + f;
              if (full8 && ((reinterpret_cast<uintptr_t>(rp) & 15) == 0)) {
                float rr[8];
                unpack8(*reinterpret_cast<const bf16x8*>(rp), rr);
#pragma unroll
                for (int e = 0; e < 8; ++e) o[e] += rr[e];
              } else {
                for (int e = 0; e < 8; ++e)
                  if (f + e < p.N) o[e] += bf2f(rp[e]);
              }
            }
            if (p.out_f32) {
              float* op = reinterpret_cast<float*>(p.out) + (int64_t)tok * p.ldc + f;
              for (int e = 0; e < 8; ++e)
                if (f + e < p.N) op[e] = o[e];
            } else {
              __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)tok * p.ldc + f;
              if (full8 && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
                *reinterpret_cast<bf16x8*>(op) = pack8(o);
              } else {
                for (int e = 0; e < 8; ++e)
                  if (f + e < p.N) op[e] = f2bf(o[e]);
              }
            }
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }
  __syncwarp();  // producer / MMA roles ran on lane 0: reconverge before the aligned cluster barrier
  tc::fence_before_sync();
  cluster_sync();  // the peer's MMAs / epilogue reads of this CTA's smem and TMEM are done
  if (warp == 1) {
    tc::fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN) : "memory");
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

static bool tmap(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

template <int BN>
static int launch_wide(const CUtensorMap& tw, const CUtensorMap& tx, const Params& p, cudaStream_t st) {
  using C = Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(wide_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess)
      return MS_ERR_CUDA;
    attr = true;
  }
  const int total = p.n_tiles * p.m_tiles;
  int pairs = sms() / 2;
  if (pairs > total) pairs = total;
  return launch(wide_kernel<BN>, dim3(2 * pairs), dim3(kThreads), C::SMEM, st, 1, tw, tx, p);
}

}  // namespace pair

int preload_wide() { return preload_fn(pair::wide_kernel<128>) + preload_fn(pair::wide_kernel<256>); }

}  // namespace ms

extern "C" int ms_linear_wide(const void* x, int64_t ldx, const void* w, const void* bias, const void* residual,
                              int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K, int act,
                              void* stream) {
  using namespace ms::pair;
  if (M < 0 || N < 1 || K < 1 || ldx < K || ldc < (act == 2 ? N / 2 : N)) return MS_ERR_VALUE;
  if (M == 0) return MS_OK;
  if (!x || !w || !out || act < 0 || act > 2) return MS_ERR_VALUE;
  if (act == 2 && (N % 128 || bias || residual || out_f32 || ldc % 8)) return MS_ERR_UNSUPPORTED;
  if (K % 8 || ldx % 8 || ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15))
    return MS_ERR_UNSUPPORTED;
  if (residual && ldr < N) return MS_ERR_VALUE;
  const int bn = M >= 256 ? 256 : 128;
  Params p;
  p.M = M; p.N = N; p.K = K;
  p.bias = (const __nv_bfloat16*)bias;
  p.residual = (const __nv_bfloat16*)residual;
  p.ldr = ldr;
  p.out = out; p.ldc = ldc; p.out_f32 = out_f32; p.act = act;
  p.kb_total = (K + kBK - 1) / kBK;
  p.n_tiles = (N + 255) / 256;
  p.m_tiles = (M + bn - 1) / bn;
  CUtensorMap tw, tx;
  if (!tmap(&tw, w, N, K, K, 128)) return MS_ERR_CUDA;
  if (!tmap(&tx, x, M, K, ldx, bn / 2)) return MS_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  return bn == 256 ? launch_wide<256>(tw, tx, p, st) : launch_wide<128>(tw, tx, p, st);
}
