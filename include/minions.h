/*
 * minions.h — C ABI of libminions.so, the sm_100a speculate-vote-verify hot path.
 *
 * Every entry point takes DEVICE pointers owned by the caller, plain integer
 * sizes and a cudaStream_t passed as `void*` (NULL = legacy default stream),
 * launches stream-ordered work, allocates nothing and returns an int status
 * (MS_OK = 0, negative = error).  Negative codes map onto the reference's
 * exception classes (see paper_2402_15678_b200/_native.py):
 *
 *   MS_ERR_VALUE          -> ValueError            (aggspec argument errors)
 *   MS_ERR_LENGTH         -> LengthMismatch        (aggspec/voting.py:11)
 *   MS_ERR_DIST_MISMATCH  -> DistMismatch          (aggspec/verification.py:13)
 *   MS_ERR_UNSUPPORTED    -> NotImplementedError   (shape outside the kernel's range)
 *   MS_ERR_CUDA           -> RuntimeError          (launch failure)
 *
 * Reference interfaces each entry point replaces are cited per function;
 * paths are relative to /root/reference/pkg/src.
 */
#ifndef MINIONS_H_
#define MINIONS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MS_OK = 0,
  MS_ERR_VALUE = -1,
  MS_ERR_LENGTH = -2,
  MS_ERR_DIST_MISMATCH = -3,
  MS_ERR_UNSUPPORTED = -4,
  MS_ERR_CUDA = -5,
};

/* ---- library ---------------------------------------------------------- */

/* ABI version (major*100 + minor). */
int ms_version(void);
/* Human-readable message for a status code. */
const char* ms_strerror(int status);
/* Number of kernels launched through this library since load / last reset. */
int64_t ms_launch_count(void);
/* Load every kernel of the library now (instead of lazily at first launch:
 * the tensor-parallel peer protocol runs spin-waiting kernels concurrently
 * with other streams' kernels, and a lazy load can block behind them). */
int ms_preload(void);
void ms_reset_launch_count(void);

/* ---- K4: weighted-majority vote ---------------------------------------
 * Replaces merge() + select_majority() (aggspec/voting.py:83-139) as called
 * per request by SpeculationEngine._do_draft_batch (aggspec/engine.py:262-276).
 *
 *   tokens  [B, K, S] int32   draft k of request b (draft order = k)
 *   weights [K]       fp64    weight of draft k (summed in draft order)
 *   rank    [K]       int32   rank of draft k's drafter id among the ids
 *                             (voted = min id among the leaf contributors);
 *                             NULL = identity (ids 0..K-1 in draft order)
 *   path    [B, S]    int32   majority path (out)
 *   voted   [B]       int32   draft index of the voted drafter (out)
 * Limits: 1 <= K <= 32, 1 <= S <= 4096, B >= 0.
 */
int ms_vote(const int32_t* tokens, const double* weights, const int32_t* rank,
            int B, int K, int S, int32_t* path, int32_t* voted, void* stream);

/* ---- K9: greedy accept + commit ----------------------------------------
 * Replaces verify() on point-mass dists (aggspec/verification.py:29-77) plus the
 * append / remaining / stop-token commit of _do_verify_batch
 * (aggspec/engine.py:297-313).
 *
 *   draft      [B, S]   int32  voted draft tokens
 *   tgt_argmax [B, S+1] int32  target argmax at each of the s+1 positions
 *   remaining  [B]      int32  max_new_tokens - len(generated)
 *   stop_token          int    -1 = none
 *   n_acc      [B]      int32  accepted_count (out; untruncated, feeds the ACR)
 *   emitted    [B, S+1] int32  tokens appended (out; -1 padded after n_emit)
 *   n_emit     [B]      int32  len(use) after budget / stop truncation (out)
 *   finished   [B]      int32  1 if the request finished this round (out)
 *   kv_len     [B]      int32  in/out or NULL: += n_acc + 1 when not finished
 * Limits: 1 <= S <= 4096.
 */
int ms_accept_greedy(const int32_t* draft, const int32_t* tgt_argmax,
                     const int32_t* remaining, int stop_token, int B, int S,
                     int32_t* n_acc, int32_t* emitted, int32_t* n_emit,
                     int32_t* finished, int32_t* kv_len, void* stream);

/* ---- K8 (unfused form): row argmax over logits --------------------------
 * Builds the greedy target "distributions" of aggspec/engine.py:294-296:
 * argmax over V with first-index tie-break, as ProbDist.point_mass(argmax)
 * of np.argmax (aggspec/core.py:81-85).
 *   logits [R, ld] (fp32 if is_bf16 == 0, else bf16), first V columns used
 *   out    [R] int32
 *   ws     unused (kept for ABI stability; may be NULL) — one CTA per row
 */
int ms_argmax_rows(const void* logits, int is_bf16, int R, int V, int64_t ld,
                   int32_t* out, void* ws, void* stream);

/* argmax + accept in one call: logits [B, S+1, V]; tgt_argmax_ws [B*(S+1)]
 * int32 receives the target argmax, argmax_ws [B*(S+1)] uint64 scratch. */
int ms_accept_greedy_logits(const int32_t* draft, const void* logits, int is_bf16,
                            int V, const int32_t* remaining, int stop_token, int B,
                            int S, int32_t* tgt_argmax_ws, void* argmax_ws, int32_t* n_acc,
                            int32_t* emitted, int32_t* n_emit, int32_t* finished,
                            int32_t* kv_len, void* stream);

/* ---- K1/K5/K8: linear layer on tcgen05 tensor cores ---------------------
 * The projection GEMMs of the SSM decode step and the LLM verification
 * forward, i.e. the compute behind ModelOracle.next_dist
 * (aggspec/oracles.py:19-26) as called by draft_sequence (aggspec/oracles.py:148)
 * and the target loop of _do_verify_batch (aggspec/engine.py:294-296).
 *
 *   out[m, n] = act(sum_k x[m, k] * w[n, k] + bias[n]) + residual[m, n]
 *   x [M, ldx] bf16, w [N, K] bf16 (nn.Linear layout), bias [N] bf16 or NULL,
 *   residual [M, ldr] bf16 or NULL, out [M, ldc] bf16 (out_f32 = 0) or fp32,
 *   act 0 = identity, 1 = ReLU, 2 = gated SiLU (Llama SwiGLU MLP): w holds the
 *   gate and up projections interleaved in 64-row blocks (rows 128t..128t+63 =
 *   gate rows 64t.., rows 128t+64..128t+127 = up rows 64t..) and
 *   out [M, N/2] = silu(gate) * up, bf16, no bias / residual, N % 128 == 0.
 * Schedule: one CTA per (128-feature tile, split, token tile); the `splits`
 * CTAs of a tile (0 = ms_linear_splits(N, K), max 8) form a thread-block
 * cluster and reduce their fp32 partials through distributed shared memory in
 * rank order — deterministic and batch invariant (a row's result does not
 * depend on M: the partition depends only on N and K).
 * Limits: K % 8 == 0, ldx % 8 == 0, x and w 16-byte aligned.
 */
int ms_linear(const void* x, int64_t ldx, const void* w, const void* bias,
              const void* residual, int64_t ldr, void* out, int64_t ldc, int out_f32,
              int M, int N, int K, int act, int splits, void* stream);
/* ms_linear with the RMSNorm folded across GEMMs (the norm's gain is
 * pre-multiplied into the consumer's weight, so no normalised activation is
 * written): rms_out != NULL — a residual-writing split-K GEMM (bf16 out,
 * splits >= 2) also writes, per 128-feature tile t and row m, the sum of
 * squares of the bf16 values it stored: rms_out[m * rms_ld + t] (a row's
 * partials contiguous); rms_in != NULL — the GEMM runs on the raw residual
 * stream x and scales its fp32 accumulator by rstd[m] = rsqrt(sum_{t <
 * rms_nparts} rms_in[m * rms_ld + t] / K + eps) before the epilogue (bias / activation / gated SiLU / residual).
 * Fixed summation orders: deterministic and batch invariant. */
int ms_linear_rms(const void* x, int64_t ldx, const void* w, const void* bias, const void* residual,
                  int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K, int act,
                  int splits, const float* rms_in, int rms_nparts, float rms_eps, float* rms_out,
                  int64_t rms_ld, void* stream);
/* Compute-bound linear layer for prompt prefill (M >= 256 token rows; any M
 * accepted): same contract as ms_linear (bias / ReLU / residual / gated SiLU
 * with N % 128 == 0, bf16 or fp32 out), on CTA pairs — tcgen05.mma
 * cta_group::2 over a 256-feature x 256-token tile (128 tokens when M < 256),
 * persistent over tiles with a double-buffered TMEM accumulator.  Full-K
 * accumulation in k order: deterministic; NOT split like ms_linear, so the
 * decode / verify path (whose per-row results must not depend on M) keeps
 * ms_linear.  Replaces the prefill GEMMs' cuBLAS calls.
 * Limits: K % 8 == 0, ldx % 8 == 0, x and w 16-byte aligned. */
int ms_linear_wide(const void* x, int64_t ldx, const void* w, const void* bias, const void* residual,
                   int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K, int act,
                   void* stream);
/* Low-latency projection for M <= 64 token rows (the drafters' decode steps):
 * same contract as ms_linear (bias / ReLU / residual, bf16 or fp32 out), one
 * CTA per 16 output features, K split over 4 warps reduced in shared memory,
 * warp-level MMAs fed by 16-byte global loads; no TMEM, clusters or scratch.
 * Deterministic; a row's result does not depend on M.  K % 32 == 0. */
int ms_gemv(const void* x, int64_t ldx, const void* w, const void* bias, const void* residual,
            int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K, int act,
            void* stream);
/* Default split-K factor for an [N, K] weight (cluster path). */
int ms_linear_splits(int N, int K);
/* Schedule of one-split gated ms_linear GEMMs with more output tiles than two
 * CTAs per SM (the 70B gate/up): 1 (default) = persistent two-per-SM CTAs with a
 * double-buffered TMEM accumulator (gemm_gated.cuh; bitwise the same outputs),
 * 0 = one tile per CTA.  Read at launch; returns the previous value. */
int ms_set_gated_persistent(int on);

/* ---- decoder pieces around the GEMMs (OPT-style, pre-LN) ----------------
 * Token + learned-position embedding of R = B*Q rows: row r = b*Q + i is at
 * position start[b] + i; out[r] = tok_emb[tok[r]] + pos_emb[pos + pos_offset]
 * (pos_emb may be NULL).  bf16 [R, d].
 */
int ms_embed(const int32_t* tok, const int32_t* start, int Q, const void* tok_emb,
             const void* pos_emb, int pos_offset, int R, int d, void* out, void* stream);

/* LayerNorm (fp32 statistics) into out [R, ldo]: output row r normalises input
 * row rows[r] (rows == NULL: row r) of x [*, ldx] bf16. */
int ms_layernorm(const void* x, int64_t ldx, const int32_t* rows, const void* gamma,
                 const void* beta, float eps, int R, int d, void* out, int64_t ldo, void* stream);
/* RMSNorm (Llama): out = x * rsqrt(mean(x^2) + eps) * gamma, fp32 statistics,
 * one bf16 rounding; rows as in ms_layernorm. */
int ms_rmsnorm(const void* x, int64_t ldx, const int32_t* rows, const void* gamma, float eps,
               int R, int d, void* out, int64_t ldo, void* stream);

/* Gated SiLU of a gate/up GEMM's fp32 output gu [M, ldg] (N columns, 64-row
 * interleaved weight: tile t = 64 gate then 64 up columns) into out [M, ldo]
 * bf16, N/2 columns: silu(g) * u in fp32, one rounding — the ms_linear act=2
 * epilogue for prompt-prefill GEMMs run on cuBLAS. */
int ms_gated_silu(const float* gu, int64_t ldg, int M, int N, void* out, int64_t ldo, void* stream);

/* KV-cache append: rows r = b*Q + i of qkv [B*Q, ldq] (layout [q | k | v],
 * each H*D wide) are written at position start[b] + i of cache slot slot[b];
 * caches are [slots, H, T, D] bf16.  Positions outside [0, T) are skipped. */
int ms_kv_append(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                 const int32_t* slot, const int32_t* start, int T, void* k_cache,
                 void* v_cache, void* stream);
/* Grouped-query form: qkv row layout [q (H*D) | k (Hkv*D) | v (Hkv*D)], caches
 * [slots, Hkv, T, D]; with rope != NULL (float2 [>= T, D/2] of (cos, sin) of
 * position p times frequency i, Llama rotate-half pairing i <-> i + D/2) the K
 * rows are rotated at their absolute position before they are stored. */
int ms_kv_append_gqa(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                     const int32_t* slot, const int32_t* start, int T, void* k_cache,
                     void* v_cache, const void* rope, void* stream);

/* Causal attention of Q query rows per request over the KV cache: query i of
 * request b (row b*Q + i of qkv) is at position start[b] + i and attends to
 * cache positions 0..start[b] + i.  With append != 0 the K/V columns of the Q
 * rows are first written into the cache (fused into the kernel when Q <= 16,
 * else an ms_kv_append launch precedes it).  out [B*Q, ldo] bf16, head h at
 * columns h*D.. .  Deterministic and batch invariant (fixed key partition,
 * fixed merge order).  Limits: D in {64, 128}. */
int ms_attention(const void* qkv, int64_t ldq, int B, int Q, int H, int D,
                 const int32_t* slot, const int32_t* start, int T, void* k_cache,
                 void* v_cache, float scale, int append, void* out, int64_t ldo,
                 void* ws, int64_t ws_bytes, int* counters, int n_counters, void* stream);
/* With ws != NULL the KV range is split into fixed 128-key chunks, one CTA each
 * (more CTAs in flight on the KV stream); the last chunk of a (request, head)
 * merges the chunk partials in chunk order.  ws / counters sizes: */
int ms_attention_workspace(int B, int Q, int H, int D, int T, int64_t* ws_bytes, int* n_counters);
/* Split-KV scratch for grouped-query attention (Hkv < H: the row-split kernel's records). */
int ms_attention_workspace_gqa(int B, int Q, int H, int Hkv, int D, int T, int64_t* ws_bytes,
                               int* n_counters);
/* Grouped-query attention with optional RoPE (Llama-2: H = 64 query heads over
 * Hkv = 8 KV heads): layouts as in ms_kv_append_gqa; query head h reads KV head
 * h / (H / Hkv).  One CTA per (request, KV head, 16 flattened (position, head)
 * rows), so a KV head's keys are staged once for all its query heads; Q is
 * rotated in registers, the call's own K rows while staged / appended.  The
 * workspace of ms_attention_workspace(B, Q, H, D, T) suffices. */
int ms_attention_gqa(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                     const int32_t* slot, const int32_t* start, int T, void* k_cache,
                     void* v_cache, const void* rope, float scale, int append, void* out,
                     int64_t ldo, void* ws, int64_t ws_bytes, int* counters, int n_counters,
                     void* stream);

/* ---- round glue ------------------------------------------------------------
 * After an SSM decode step's argmax tok[B]: drafts[b, k, j] = tok[b] (the token
 * list draft_sequence builds, aggspec/oracles.py:146-152) and next_tok[b] =
 * tok[b] (NULL: not written).  With teacher != NULL (fidelity-injection bench
 * mode), the token is replaced by teacher[b, ctx_len[b] + j] (a target greedy
 * continuation, absolute positions, ld_teacher per row; -1 = none) when
 * hash(seed, req_key[b], k, position) < fidelity — the device analogue of the
 * PerturbedOracle fidelity knob (aggspec/oracles.py:108-132).
 */
int ms_draft_commit(const int32_t* tok, const int32_t* ctx_len, int B, int j, int k,
                    int K, int S, const int32_t* teacher, int64_t ld_teacher,
                    const int32_t* req_key, float fidelity, uint64_t seed,
                    int32_t* drafts, int32_t* next_tok, void* stream);

/* Verifier input rows vin[b] = [last[b], path[b, 0..S-1]] ([B, S+1] int32):
 * the contexts ctx + tokens[:i] of aggspec/engine.py:294-296. */
int ms_pack_verify(const int32_t* last, const int32_t* path, int B, int S,
                   int32_t* vin, void* stream);

/* K3 stochastic — the device form of ModelOracle.next_dist + ProbDist.sample
 * (aggspec/oracles.py:146-150, aggspec/core.py:74-78) for a softmax model:
 * row r of logits [R, ldl] fp32 -> probs[r*ldp ..] fp64 = exp(l - max) / S,
 * S the NumPy pairwise sum of exp(l - max) (oracle/model_oracle.softmax64),
 * and, when uniforms != NULL, tok[r] = searchsorted(cumsum(p), u[r*ldu],
 * 'right') clamped to V-1 (sequential fp64 cumsum).  V <= 65536. */
int ms_softmax_sample(const float* logits, int64_t ldl, int R, int V, const double* uniforms, int64_t ldu,
                      double* probs, int64_t ldp, int32_t* tok, void* stream);
/* out[b] = q[voted[b]][b]: q [K][B][S][V] fp64 draft distributions -> the
 * voted drafter's [B][S][V] (select_majority's dists, aggspec/voting.py:133-139). */
int ms_gather_voted(const double* q, const int32_t* voted, int K, int B, int S, int V, double* out,
                    void* stream);
/* ---- K10: stochastic accept (speculative sampling) ------------------------
 * verify() of aggspec/verification.py:29-77 on general distributions, bit-exact
 * given the same fp64 probabilities and uniforms:
 *   draft [B, S] int32, q [B, S, V] fp64 (voted drafter's dists),
 *   o [B, S+1, V] fp64 (target dists), uniforms [B, S+1] fp64 — the next S+1
 *   doubles of each request's verify stream (the kernel uses n_draws of them),
 *   scratch [B, V] fp64.  Outputs as ms_accept_greedy plus n_draws [B] (the
 *   number of uniforms the reference consumed: i+2 on a rejection at i, S+1 on
 *   full acceptance), so the host advances its generator identically.
 * The residual normaliser is NumPy's pairwise sum (exact emulation) and the
 * inverse-CDF scan is sequential fp64 (np.cumsum + searchsorted 'right').
 * Limits: V <= 65536.
 */
int ms_accept_stochastic(const int32_t* draft, const double* q, const double* o,
                         const double* uniforms, const int32_t* remaining, int stop_token,
                         int B, int S, int V, double* scratch, int32_t* n_acc,
                         int32_t* emitted, int32_t* n_emit, int32_t* finished,
                         int32_t* n_draws, void* stream);

/* ---- paged KV cache ------------------------------------------
 * K/V live in block pools [n_blocks, Hkv, block_size, D] bf16; block_table
 * [slots, max_blocks] int32 maps position t of a slot to pool block
 * table[slot][t / block_size], row t % block_size (T <= max_blocks *
 * block_size).  Same arithmetic as the contiguous entry points (bitwise):
 * only K/V row addresses change.  A host block manager
 * (paper_2402_15678_b200/paged.py) grows a sequence's blocks before a round
 * and frees the blocks past the accepted length after it — the KV of
 * rejected speculative tokens. */
int ms_attention_paged(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                       const int32_t* slot, const int32_t* start, int T, void* k_cache,
                       void* v_cache, const void* rope, float scale, int append, void* out,
                       int64_t ldo, void* ws, int64_t ws_bytes, int* counters, int n_counters,
                       const int32_t* block_table, int max_blocks, int block_size, void* stream);
int ms_kv_append_paged(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                       const int32_t* slot, const int32_t* start, int T, void* k_cache,
                       void* v_cache, const void* rope, const int32_t* block_table, int max_blocks,
                       int block_size, void* stream);

/* ---- grouped drafters -------------------------------------------------------
 * The K drafters of a round (same architecture, own weights) run as ONE
 * launch per op: G row groups, group k = drafter k, each with its own weights
 * (stacked [G, ...]) and its own KV-cache slots.  Rows of group g are rows
 * g*M .. g*M + M-1 of x / out (M rows per group).  Replaces the per-drafter
 * loop of draft_sequence calls in _do_draft_batch (aggspec/engine.py:262-276).
 *   ms_linear_grouped: W = [G*N, K] (group g's weight = rows g*N..), bias [G*N],
 *     cluster split-K schedule, otherwise as ms_linear.
 *   ms_gemv_grouped:   group g's weight at w + g*w_gstride elements.
 *   ms_embed_grouped / ms_rmsnorm_grouped: output row r uses table / gain
 *     number r / rpg (stride tstride / gstride elements).
 *   ms_draft_commit_grouped: tok [G*B] -> drafts[b, k, j] = tok[k*B + b] (with
 *     drafter k's fidelity[k], host array of G <= 8 floats), next_tok [G*B]. */
int ms_linear_grouped(const void* x, int64_t ldx, const void* w, const void* bias, const void* residual,
                      int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K, int act,
                      int splits, int G, void* stream);
int ms_gemv_grouped(const void* x, int64_t ldx, const void* w, int64_t w_gstride, const void* bias,
                    const void* residual, int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N,
                    int K, int act, int G, void* stream);
/* ms_gemv_grouped with each x row's RMSNorm folded in (the gain folded into w
 * beforehand, LlamaWeights.fold_norms): out = act(rstd[row] * (x . w^T)) (+
 * residual), rstd = rsqrt(mean_k x[row, k]^2 + eps) from the bf16 x values in
 * a fixed order — no RMSNorm kernel and no normalised activation in HBM.  The
 * grouped drafters' QKV and gate/up projections of a decode step. */
int ms_gemv_rms_grouped(const void* x, int64_t ldx, const void* w, int64_t w_gstride, const void* residual,
                        int64_t ldr, void* out, int64_t ldc, int out_f32, int M, int N, int K, int act, int G,
                        float eps, void* stream);
int ms_embed_grouped(const int32_t* tok, const int32_t* start, int Q, const void* tok_emb, int64_t tstride,
                     int rpg, const void* pos_emb, int pos_offset, int R, int d, void* out, void* stream);
int ms_rmsnorm_grouped(const void* x, int64_t ldx, const int32_t* rows, const void* gamma, int64_t gstride,
                       int rpg, float eps, int R, int d, void* out, int64_t ldo, void* stream);
int ms_draft_commit_grouped(const int32_t* tok, const int32_t* ctx_len, int B, int j, int G, int S,
                            const int32_t* teacher, int64_t ld_teacher, const int32_t* req_key,
                            const float* fidelity, uint64_t seed, int32_t* drafts, int32_t* next_tok,
                            void* stream);

/* ---- tensor-parallel verify over peer memory -----------------
 * Symmetric buffers: ms_ipc_alloc cudaMallocs `bytes` (zeroed) and exports a
 * CUDA IPC handle (ms_ipc_handle_size() bytes) that peers open with
 * ms_ipc_open.  Flag sets hold one int per rank; `epoch` is a device counter
 * per flag set (ms_tp_signal bumps it and publishes it to slot `rank` of every
 * rank's flags with a system-scope release; waits acquire until every slot
 * reaches the local epoch, bounded: on timeout *err = 1 and the kernel
 * proceeds — no hang).  early != 0 releases the dependent kernel (PDL) before
 * the wait — only when every rank has its own GPU.  Pointer arrays (peer_*) are device arrays of the t
 * ranks' buffer addresses, rank order.  Replaces the NCCL allreduce of the
 * Megatron row-parallel projections with a fixed-order, batch-invariant sum. */
int ms_ipc_alloc(int64_t bytes, void** ptr, void* handle);
int ms_ipc_handle_size(void);
int ms_ipc_open(const void* handle, void** ptr);
int ms_ipc_close(void* ptr);
int ms_free(void* ptr);
int ms_tp_signal(int* const* peer_flags, int rank, int t, int* epoch, void* stream);
/* Two-shot sum after a row-parallel GEMM: waits for flag set `flags`, then
 * rank `rank` adds column slice [rank*d/t, (rank+1)*d/t) of the t fp32
 * partials parts[j] [R, ldp] in rank order (one bf16 rounding) and stores it
 * into every rank's residual stream xs[j] [R, ldx] bf16.  d % (4t) == 0. */
int ms_tp_reduce_gather(const float* const* parts, int64_t ldp, void* const* xs, int64_t ldx,
                        const int* flags, const int* epoch, int rank, int t, int R, int d,
                        int* err, int early, void* stream);
/* Fused GEMM -> reduce-scatter: out = x . w^T (+ residual, rank 0), fp32,
 * written straight into the receive slots of the rank owning each column
 * slice: recv[f / (N/t)][(rank * rows + m) * (N/t) + f % (N/t)] (recv: device
 * array of the t ranks' receive buffers) — peer stores issued as each output
 * tile completes, overlapped with the other tiles' math.  Cluster split-K. */
int ms_linear_tp_scatter(const void* x, int64_t ldx, const void* w, const void* residual, int64_t ldr,
                         int M, int N, int K, float* const* recv, int rank, int t, int rows, void* stream);
/* After the flags: sum the t local receive slots [t][rows_cap][slice] in rank
 * order, store the bf16 slice into every rank's residual stream xs[j]. */
int ms_tp_reduce_recv_gather(const float* recv, int rows_cap, int slice, void* const* xs, int64_t ldx,
                             const int* flags, const int* epoch, int rank, int t, int R, int* err,
                             int early, void* stream);
/* RMSNorm of x [R, ldx] (as ms_rmsnorm) after waiting for flag set `flags`
 * (every rank's slice of x has landed). */
int ms_rmsnorm_wait(const void* x, int64_t ldx, const void* gamma, float eps, int R, int d,
                    void* out, int64_t ldo, const int* flags, const int* epoch, int t, int* err,
                    int early, void* stream);
/* Vocab-parallel argmax: per row of this rank's logits slice [R, Vr] (global
 * ids v0..v0+Vr-1) a u64 key (order-preserving value | ~index, so the max key
 * is the first-index argmax; NaN never wins); combine waits for the flags and
 * takes the max key over the t ranks' keys -> out [R] int32 (every rank). */
int ms_tp_argmax_local(const float* logits, int64_t ld, int R, int Vr, int v0, uint64_t* out,
                       void* stream);
int ms_tp_argmax_combine(const uint64_t* const* peer, int t, int R, const int* flags,
                         const int* epoch, int32_t* out, int* err, int early, void* stream);

/* ---- fp32 verification mode (csrc/fp32.cu) ---------------------------------
 * The model forward behind ModelOracle.next_dist (aggspec/oracles.py:19-26)
 * with fp32 activations, fp32 KV cache and fp32 accumulation (weights: the
 * same bf16 tensors).  north_star: "accepted token sequences and vote results
 * bit-exact in the fp32 verification mode" — SpecEngine(precision="fp32")
 * reproduces the reference engine (aggspec/engine.py:252-330) driven by fp32
 * CPU oracles.  Plain SIMT kernels; every output depends only on its own row.
 *   ms_embed_f32:     out [R, d] = tok_emb[tok] (+ pos_emb[pos + pos_offset]).
 *   ms_norm_f32:      LayerNorm (rms = 0; two-pass mean / variance) or RMSNorm
 *                     (rms = 1, beta unused) of x rows (rows[r] or r).
 *   ms_linear_f32:    out = act(x . w^T + bias) (+ residual), x / out / residual
 *                     fp32, w bf16 [N, K]; act 0 none, 1 ReLU, 2 gated SiLU over
 *                     the 64-row interleaved gate/up weight (out [M, N/2]).
 *   ms_attention_f32: KV append (K rotated when rope != NULL; fp32 caches
 *                     [slots, Hkv, T, D]) + causal attention of the call's rows
 *                     (H query heads over Hkv KV heads, D <= 128); scale_q = 1
 *                     scales q before q.k (OPT), 0 scales the score (Llama). */
int ms_embed_f32(const int32_t* tok, const int32_t* start, int Q, const void* tok_emb,
                 const void* pos_emb, int pos_offset, int R, int d, float* out, void* stream);
int ms_norm_f32(const float* x, int64_t ldx, const int32_t* rows, const void* gamma, const void* beta,
                float eps, int rms, int R, int d, float* out, int64_t ldo, void* stream);
int ms_linear_f32(const float* x, int64_t ldx, const void* w, const void* bias, const float* residual,
                  int64_t ldr, float* out, int64_t ldo, int M, int N, int K, int act, void* stream);
int ms_attention_f32(const float* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D,
                     const int32_t* slot, const int32_t* start, int T, float* k_cache, float* v_cache,
                     const float* rope, float scale, int scale_q, float* out, int64_t ldo, void* stream);

/* Grouped-query attention of Q <= 16 query positions per request on tcgen05
 * (head dim 128, H % Hkv == 0 — multi-head G = 1 accepted —, Q * H / Hkv <=
 * 128 flattened rows): K / V read by TMA in
 * 128-key chunks, S = Q K^T and P V on tcgen05 with TMEM accumulators, K/V
 * append fused (append != 0).  T <= 384: one pass over the whole context;
 * longer caches: online softmax over chunks.  Cache: contiguous
 * [n_slots, Hkv, T, 128] (block_table NULL) or a paged pool of n_slots blocks
 * [n_slots, Hkv, block_size, 128] with block_table [slots, max_blocks]
 * (T = max_blocks * block_size <= 384, block_size a multiple of 16 dividing
 * 128).  Prompt prefill (append == 0, required when Q > 16 or Q * H / Hkv >
 * 128; head dim 128 or 64): the call's K / V rows already in the cache (e.g.
 * by ms_kv_append_paged) and the online kernel runs one CTA per (request, KV
 * head, 128 / G positions).  Replaces the attention inside ModelOracle.next_dist for the verify
 * positions (aggspec/oracles.py:19-26, aggspec/engine.py:294-296); same
 * contract as ms_attention_paged for those shapes (csrc/attention_tc.cu). */
int ms_attention_tc(const void* qkv, int64_t ldq, int B, int Q, int H, int Hkv, int D, const int32_t* slot,
                    const int32_t* start, int T, int n_slots, void* k_cache, void* v_cache, const void* rope,
                    float scale, int append, void* out, int64_t ldo, const int32_t* block_table,
                    int max_blocks, int block_size, void* stream);

/* Programmatic dependent launch (PDL) attribute for subsequent launches of
 * this process (default on; MS_PDL=0 in the environment turns it off); a
 * captured CUDA graph keeps the setting it was captured with.  Returns the
 * previous setting. */
int ms_set_pdl(int on);

/* Co-resident launch shapes (default off; the pipelined engine turns it on
 * around its drafter graphs): ms_gemv runs 64-thread CTAs (<= 128 registers)
 * and single-row MHA decode attention (Q = 1, contiguous cache) runs
 * 64-thread, shared-memory-free CTAs — each fits on an SM beside two
 * verify-GEMM CTAs (2 x 224 x 128 + 64 x 128 registers = 64K), so the
 * drafters of one group neither wait for nor displace the verifier of the
 * other.  Results differ in rounding from the default shapes.  A captured CUDA
 * graph keeps the setting it was captured with.  Returns the previous value. */
int ms_set_coresident(int on);

/* ---- SM partition for the pipelined schedule ------------------------------
 * Replaces: the reference's separate SSM / LLM executors of run_pipelined
 * (aggspec/engine.py:494-576 — drafting of one batch concurrent with the
 * verification of another); the paper places SSMs on their own devices.  On
 * one GPU: two green contexts splitting the SMs (draft_sms for the drafters,
 * the rest for the verifier), one stream each, returned as cudaStream_t
 * (void*).  The contexts live for the process.  MS_ERR_UNSUPPORTED when the
 * driver has no green contexts. */
int ms_sm_partition(int device, int draft_sms, int draft_priority, int verify_priority,
                    void** draft_stream, void** verify_stream, int* got_draft, int* got_verify);

#ifdef __cplusplus
}
#endif

#endif /* MINIONS_H_ */
