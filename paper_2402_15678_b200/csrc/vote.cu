// K4 — weighted-majority vote over K drafts per request.
//
// Restates merge() + select_majority() (aggspec/voting.py:83-139) without
// building a trie: descending level by level, the weight of the child with
// token t under the chosen prefix is the fp64 sum, in draft order, of the
// weights of the drafts still on that prefix whose token at this level is t
// (merge adds `w[ssm_id]` to each node it passes, drafts in list order,
// voting.py:99-110).  The child minimising (-weight, token) is taken
// (voting.py:130) and the voted drafter is the smallest id among the leaf's
// contributors (voting.py:132).
//
// Mapping: one warp per request, lane k = draft k (K <= 32).  Drafts sharing a
// token are grouped with __match_any_sync; each lane of a group re-adds the
// group's weights in ascending k (the reference's summation order), so the
// fp64 sums are bit-identical to the reference's.  The winner is a warp
// argmax on (weight desc, token asc) — comparisons only, so exact.
#include "common.cuh"

namespace ms {

constexpr int kVoteWarps = 4;

__global__ void __launch_bounds__(kVoteWarps * 32)
vote_kernel(const int32_t* __restrict__ tokens, const double* __restrict__ weights,
            const int32_t* __restrict__ rank, int B, int K, int S,
            int32_t* __restrict__ path, int32_t* __restrict__ voted) {
  pdl_wait();
  pdl_trigger();
  const int lane = lane_id();
  const int b = blockIdx.x * kVoteWarps + (threadIdx.x >> 5);
  if (b >= B) return;  // warp-uniform
  const bool active = lane < K;
  const double w = active ? weights[lane] : 0.0;
  const int my_rank = active ? (rank ? rank[lane] : lane) : 0x7fffffff;
  const int32_t* tok = tokens + ((int64_t)b * K + (active ? lane : 0)) * S;
  unsigned alive = __ballot_sync(0xffffffffu, active);

  for (int l = 0; l < S; ++l) {
    const bool on = (alive >> lane) & 1u;
    const int t = on ? __ldg(tok + l) : 0;
    // group lanes by token among the alive drafts (inactive lanes get a mask
    // that is never read)
    const unsigned grp = __match_any_sync(0xffffffffu, on ? t : (int)0x80000000 + lane);
    const unsigned mine = grp & alive;
    // sequential fp64 sum over the group in ascending draft index
    double sum = 0.0;
    for (int k = 0; k < K; ++k) {
      const double wk = __shfl_sync(0xffffffffu, w, k);
      if ((mine >> k) & 1u) sum += wk;
    }
    // warp argmax on (sum desc, token asc); dead lanes never win
    double best_w = on ? sum : -__longlong_as_double(0x7ff0000000000000LL);
    int best_t = on ? t : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w2 = __shfl_xor_sync(0xffffffffu, best_w, o);
      const int t2 = __shfl_xor_sync(0xffffffffu, best_t, o);
      if (w2 > best_w || (w2 == best_w && t2 < best_t)) {
        best_w = w2;
        best_t = t2;
      }
    }
    alive &= __ballot_sync(0xffffffffu, on && t == best_t);
    if (lane == 0) path[(int64_t)b * S + l] = best_t;
  }
  // voted drafter = min rank among the survivors
  int r = ((alive >> lane) & 1u) ? my_rank : 0x7fffffff;
  int k = lane;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int r2 = __shfl_xor_sync(0xffffffffu, r, o);
    const int k2 = __shfl_xor_sync(0xffffffffu, k, o);
    if (r2 < r || (r2 == r && k2 < k)) {
      r = r2;
      k = k2;
    }
  }
  if (lane == 0) voted[b] = k;
}

int preload_vote() { return preload_fn(vote_kernel); }

}  // namespace ms

extern "C" int ms_vote(const int32_t* tokens, const double* weights, const int32_t* rank,
                       int B, int K, int S, int32_t* path, int32_t* voted, void* stream) {
  if (B < 0) return MS_ERR_VALUE;
  if (K < 1) return MS_ERR_VALUE;  // "at least one draft is required"
  if (S < 1) return MS_ERR_LENGTH;  // "draft sequences must be non-empty"
  if (K > 32 || S > 4096) return MS_ERR_UNSUPPORTED;
  if (B == 0) return MS_OK;
  if (!tokens || !weights || !path || !voted) return MS_ERR_VALUE;
  const int blocks = (B + ms::kVoteWarps - 1) / ms::kVoteWarps;
  return ms::launch(ms::vote_kernel, dim3(blocks), dim3(ms::kVoteWarps * 32), 0, (cudaStream_t)stream, 1,
                    tokens, weights, rank, B, K, S, path, voted);
}
