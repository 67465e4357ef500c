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
 *   ws     [R] uint64 scratch (contents clobbered)
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

#ifdef __cplusplus
}
#endif

#endif /* MINIONS_H_ */
