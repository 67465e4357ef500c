// K10 — stochastic (speculative-sampling) accept, bit-exact with the
// reference's verify() (aggspec/verification.py:29-77) on the same fp64
// distributions and the same uniforms.
//
//   position i: q = q_i(x_i), o = o_i(x_i), u = u_i
//               accept if q <= o, or if u >= 1 - o/q          (fp64, same ops)
//   first rejection at i: residual r = max(o_i - q_i, 0)
//               total = NumPy pairwise sum of r                (exact emulation)
//               total > 0 ? sample r/total : sample o_i, with u_{i+1}
//   all accepted: bonus = sample o_S with u_S
//   sample(p, u) = searchsorted(cumsum(p), u, 'right') clamped to V-1, the
//               cumsum sequential in fp64 (np.cumsum)
//
// The reference draws one uniform per considered position plus one for the
// resample / bonus; the host pre-draws S+1 uniforms (a PCG64 state peek) and
// afterwards advances the generator by n_draws, so the stream position
// matches the reference's exactly.
//
// Mapping: one CTA per request.  The accept scan is S scalar steps; the
// pairwise sum is evaluated on its fixed recursion tree (leaf blocks of <= 128
// elements in parallel, internal nodes in tree order), so it is bit-identical
// to NumPy's; the inverse-CDF scan is inherently sequential in fp64 and runs
// on one thread over shared-memory-staged chunks.
#include "common.cuh"

namespace ms {

constexpr int kSThreads = 256;
constexpr int kMaxLeaves = 1024;  // leaves of >= 64 elements: V <= 65536 (fits the OPT / Llama vocabularies)

// NumPy's pairwise sum of a[0..n) for n <= 128 (8 accumulators, 8-way unroll)
__device__ double np_pairwise_leaf(const double* a, int n) {
  if (n < 8) {  // sequential (inputs here are >= +0, so the start value's sign is moot)
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += a[i];
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  const int stop = n - (n % 8);
  for (int i = 8; i < stop; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (int i = stop; i < n; ++i) res += a[i];
  return res;
}

struct Leaf {
  int lo, n;
};

// Enumerate the leaves of NumPy's recursion in order (iterative DFS).
__device__ int np_pairwise_leaves(int n, Leaf* leaves) {
  int stack_lo[32], stack_n[32], sp = 0, cnt = 0;
  stack_lo[sp] = 0;
  stack_n[sp++] = n;
  while (sp > 0) {
    const int lo = stack_lo[--sp], m = stack_n[sp];
    if (m <= 128) {
      leaves[cnt++] = {lo, m};
    } else {
      int m2 = m / 2;
      m2 -= m2 % 8;
      stack_lo[sp] = lo + m2;  // right child after the left one (DFS order)
      stack_n[sp++] = m - m2;
      stack_lo[sp] = lo;
      stack_n[sp++] = m2;
    }
  }
  return cnt;
}

// Combine leaf sums following the recursion: sum(lo, n) = sum(left) + sum(right).
__device__ double np_pairwise_combine(int n, const double* leaf_sum) {
  // recursive descent with an explicit stack; leaves are consumed in DFS order
  struct Frame {
    int n;
    int state;
    double left;
  };
  Frame st[32];
  int sp = 0, next_leaf = 0;
  double ret = 0.0;
  st[sp++] = {n, 0, 0.0};
  while (sp > 0) {
    Frame& f = st[sp - 1];
    if (f.n <= 128) {
      ret = leaf_sum[next_leaf++];
      --sp;
      continue;
    }
    int m2 = f.n / 2;
    m2 -= m2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp++] = {m2, 0, 0.0};
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp++] = {f.n - m2, 0, 0.0};
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

// first j with sequential fp64 prefix sum of p > u, clamped to V-1 (thread 0
// scans shared-memory chunks the whole CTA stages)
__device__ int inverse_cdf_seq(const double* p, int V, double u, double* chunk, int* s_idx) {
  constexpr int CH = 1024;
  double c = 0.0;
  int found = -1;
  for (int base = 0; base < V; base += CH) {
    const int n = min(CH, V - base);
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) chunk[j] = p[base + j];
    __syncthreads();
    if (threadIdx.x == 0 && found < 0) {
      for (int j = 0; j < n; ++j) {
        c += chunk[j];
        if (c > u) {
          found = base + j;
          break;
        }
      }
    }
    if (threadIdx.x == 0) *s_idx = found;
    __syncthreads();
    if (*s_idx >= 0) break;
  }
  const int r = *s_idx;
  __syncthreads();
  return r < 0 ? V - 1 : r;
}

__global__ void __launch_bounds__(kSThreads)
accept_stochastic_kernel(const int32_t* __restrict__ draft, const double* __restrict__ q,
                         const double* __restrict__ o, const double* __restrict__ u,
                         const int32_t* __restrict__ remaining, int stop_token, int S, int V,
                         double* __restrict__ scratch, int32_t* __restrict__ n_acc_out,
                         int32_t* __restrict__ emitted, int32_t* __restrict__ n_emit_out,
                         int32_t* __restrict__ finished_out, int32_t* __restrict__ n_draws_out) {
  pdl_wait();
  pdl_trigger();
  __shared__ Leaf leaves[kMaxLeaves];
  __shared__ double leaf_sum[kMaxLeaves];
  __shared__ double chunk[1024];
  __shared__ int s_i, s_nleaves, s_idx;
  __shared__ double s_total;
  const int b = blockIdx.x;
  const int32_t* d = draft + (int64_t)b * S;
  const double* qb = q + (int64_t)b * S * V;
  const double* ob = o + (int64_t)b * (S + 1) * V;
  const double* ub = u + (int64_t)b * (S + 1);
  if (threadIdx.x == 0) {
    int i = 0;
    for (; i < S; ++i) {
      const int tok = d[i];
      // a token outside [0, V) never reads out of bounds: it carries no
      // probability on either side (the host API raises IndexError first,
      // as the reference's probs[tok] does)
      const bool in = tok >= 0 && tok < V;
      const double qq = in ? qb[(int64_t)i * V + tok] : 0.0;
      const double oo = in ? ob[(int64_t)i * V + tok] : 0.0;
      if (qq <= oo) continue;
      if (ub[i] >= 1.0 - oo / qq) continue;
      break;
    }
    s_i = i;
  }
  __syncthreads();
  const int i = s_i;
  int sample;
  if (i < S) {
    // residual of the rejected position
    double* r = scratch + (int64_t)b * V;
    const double* oi = ob + (int64_t)i * V;
    const double* qi = qb + (int64_t)i * V;
    for (int j = threadIdx.x; j < V; j += blockDim.x) r[j] = fmax(oi[j] - qi[j], 0.0);
    if (threadIdx.x == 0) s_nleaves = np_pairwise_leaves(V, leaves);
    __syncthreads();
    const int nl = s_nleaves;
    for (int l = threadIdx.x; l < nl; l += blockDim.x) leaf_sum[l] = np_pairwise_leaf(r + leaves[l].lo, leaves[l].n);
    __syncthreads();
    if (threadIdx.x == 0) s_total = np_pairwise_combine(V, leaf_sum);
    __syncthreads();
    const double total = s_total;
    if (total > 0.0) {
      for (int j = threadIdx.x; j < V; j += blockDim.x) r[j] = r[j] / total;
      __syncthreads();
      sample = inverse_cdf_seq(r, V, ub[i + 1], chunk, &s_idx);
    } else {
      sample = inverse_cdf_seq(oi, V, ub[i + 1], chunk, &s_idx);
    }
  } else {
    sample = inverse_cdf_seq(ob + (int64_t)S * V, V, ub[S], chunk, &s_idx);
  }
  if (threadIdx.x == 0) {
    // emitted = draft[:i] + [sample], then the remaining / stop-token commit
    const int n_em_full = i + 1;
    const int rem = remaining[b];
    int n_emit = min(n_em_full, max(rem, 0));
    bool stopped = false;
    int32_t* e = emitted + (int64_t)b * (S + 1);
    for (int j = 0; j <= S; ++j) {
      const int t = j < i ? d[j] : (j == i ? sample : -1);
      e[j] = t;
    }
    if (stop_token >= 0) {
      for (int j = 0; j < n_emit; ++j) {
        if (e[j] == stop_token) {
          n_emit = j + 1;
          stopped = true;
          break;
        }
      }
    }
    for (int j = n_emit; j <= S; ++j) e[j] = -1;
    n_acc_out[b] = i;
    n_emit_out[b] = n_emit;
    finished_out[b] = (stopped || rem - n_emit <= 0) ? 1 : 0;
    n_draws_out[b] = i < S ? i + 2 : S + 1;
  }
}

// K3 stochastic — one speculative model step's distribution and sample, the
// device form of ModelOracle.next_dist + ProbDist.sample
// (aggspec/oracles.py:146-150, aggspec/core.py:74-78) for a transformer
// whose distribution is softmax(logits):
//   p = exp(l - max) / sum(exp(l - max)) in fp64 over the fp32 logits, the
//   sum NumPy's pairwise sum (the oracle adapter's softmax64,
//   oracle/model_oracle.py), then sample = searchsorted(cumsum(p), u,
//   'right') clamped to V-1 with the sequential fp64 cumsum.
// One CTA per row; the row's probabilities are kept (probs) — the draft
// distribution the verifier's K10 needs, or the target distribution.
__global__ void __launch_bounds__(kSThreads)
softmax_sample_kernel(const float* __restrict__ logits, int64_t ldl, int V, const double* __restrict__ u,
                      int64_t ldu, double* __restrict__ probs, int64_t ldp, int32_t* __restrict__ tok) {
  pdl_wait();
  pdl_trigger();
  __shared__ Leaf leaves[kMaxLeaves];
  __shared__ double leaf_sum[kMaxLeaves];
  __shared__ double chunk[1024];
  __shared__ float s_red[kSThreads / 32];
  __shared__ int s_nleaves, s_idx;
  __shared__ double s_total;
  const int r = blockIdx.x;
  const float* l = logits + (int64_t)r * ldl;
  double* p = probs + (int64_t)r * ldp;
  // max over the fp32 logits (exact in any order)
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < V; j += blockDim.x) mx = fmaxf(mx, l[j]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mx;
  if (threadIdx.x == 0) s_nleaves = np_pairwise_leaves(V, leaves);
  __syncthreads();
  mx = s_red[0];
  for (int w = 1; w < kSThreads / 32; ++w) mx = fmaxf(mx, s_red[w]);
  const double m64 = (double)mx;
  for (int j = threadIdx.x; j < V; j += blockDim.x) p[j] = exp((double)l[j] - m64);
  __syncthreads();
  const int nl = s_nleaves;
  for (int k = threadIdx.x; k < nl; k += blockDim.x) leaf_sum[k] = np_pairwise_leaf(p + leaves[k].lo, leaves[k].n);
  __syncthreads();
  if (threadIdx.x == 0) s_total = np_pairwise_combine(V, leaf_sum);
  __syncthreads();
  const double total = s_total;
  for (int j = threadIdx.x; j < V; j += blockDim.x) p[j] = p[j] / total;
  if (!u) return;
  __syncthreads();
  const int t = inverse_cdf_seq(p, V, u[(int64_t)r * ldu], chunk, &s_idx);
  if (threadIdx.x == 0) tok[r] = t;
}

// The voted drafter's distributions of each request: out[b] = q[voted[b]][b]
// (q [K][B][S][V] fp64 -> out [B][S][V]), the draft_dists select_majority
// attaches (aggspec/voting.py:133-139).
__global__ void gather_voted_kernel(const double* __restrict__ q, const int32_t* __restrict__ voted, int B,
                                    int64_t SV, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  const double* src = q + ((int64_t)voted[b] * B + b) * SV;
  double* dst = out + (int64_t)b * SV;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < SV; j += (int64_t)gridDim.x * blockDim.x)
    dst[j] = src[j];
}

int preload_accept_stochastic() {
  return preload_fn(accept_stochastic_kernel) + preload_fn(softmax_sample_kernel) + preload_fn(gather_voted_kernel);
}

}  // namespace ms

extern "C" int ms_accept_stochastic(const int32_t* draft, const double* q, const double* o,
                                    const double* uniforms, const int32_t* remaining, int stop_token,
                                    int B, int S, int V, double* scratch, int32_t* n_acc,
                                    int32_t* emitted, int32_t* n_emit, int32_t* finished,
                                    int32_t* n_draws, void* stream) {
  if (B < 0 || V < 1) return MS_ERR_VALUE;
  if (S < 1) return MS_ERR_VALUE;  // "draft must contain at least one token"
  if (V > ms::kMaxLeaves * 64) return MS_ERR_UNSUPPORTED;
  if (B == 0) return MS_OK;
  if (!draft || !q || !o || !uniforms || !remaining || !scratch || !n_acc || !emitted || !n_emit ||
      !finished || !n_draws)
    return MS_ERR_VALUE;
  return ms::launch(ms::accept_stochastic_kernel, dim3(B), dim3(ms::kSThreads), 0, (cudaStream_t)stream, 1,
                    draft, q, o, uniforms, remaining, stop_token, S, V, scratch, n_acc, emitted, n_emit,
                    finished, n_draws);
}

extern "C" int ms_softmax_sample(const float* logits, int64_t ldl, int R, int V, const double* uniforms,
                                 int64_t ldu, double* probs, int64_t ldp, int32_t* tok, void* stream) {
  if (R < 0 || V < 1 || ldl < V || ldp < V) return MS_ERR_VALUE;
  if (V > ms::kMaxLeaves * 64) return MS_ERR_UNSUPPORTED;
  if (R == 0) return MS_OK;
  if (!logits || !probs || (uniforms && !tok)) return MS_ERR_VALUE;
  return ms::launch(ms::softmax_sample_kernel, dim3(R), dim3(ms::kSThreads), 0, (cudaStream_t)stream, 1, logits,
                    ldl, V, uniforms, ldu, probs, ldp, tok);
}

extern "C" int ms_gather_voted(const double* q, const int32_t* voted, int K, int B, int S, int V, double* out,
                               void* stream) {
  if (K < 1 || B < 0 || S < 1 || V < 1) return MS_ERR_VALUE;
  if (B == 0) return MS_OK;
  if (!q || !voted || !out) return MS_ERR_VALUE;
  const int64_t SV = (int64_t)S * V;
  int gx = (int)((SV + 255) / 256);
  gx = gx > 64 ? 64 : gx;
  return ms::launch(ms::gather_voted_kernel, dim3(gx, B), dim3(256), 0, (cudaStream_t)stream, 1, q, voted, B, SV,
                    out);
}
