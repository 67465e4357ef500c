"""Verification (mirrors aggspec/verification.py) on the K8/K9 kernels.

`verify(draft_tokens, draft_dists, target_dists, rng)` keeps the reference's
signature, result type, errors and RNG consumption.  Greedy verification —
every draft and target distribution a point mass, which is what a greedy
drafter/target produces — runs `ms_accept_greedy` (csrc/accept.cu); general
distributions run `ms_accept_stochastic` (csrc/accept_stochastic.cu) on the
uniforms peeked from `rng`.  Either way the result equals the reference's on
the same inputs, and `rng` ends up advanced by exactly the number of uniforms
the reference draws (one per considered position plus one for the
correction/bonus, aggspec/verification.py:55-76).

The batched engine path calls `accept_batch` / `accept_batch_logits` on device
tensors: [B, S] voted drafts against [B, S+1] target argmaxes (or the raw
[B, S+1, V] logits), with the remaining-budget / stop-token commit of
aggspec/engine.py:300-313 fused in.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _dev
from . import _native
from .core import DistMismatch, ProbDist

__all__ = ["DistMismatch", "VerificationResult", "verify", "acceptance_rate", "accept_batch",
           "accept_batch_logits", "accept_batch_stochastic", "argmax_rows", "AcceptOut",
           "peek_uniforms"]


@dataclass(frozen=True)
class VerificationResult:
    accepted_count: int
    emitted: list[int]
    acceptance_rate: float


@dataclass
class AcceptOut:
    n_acc: torch.Tensor      # [B] int32 accepted_count (untruncated)
    emitted: torch.Tensor    # [B, S+1] int32, -1 after n_emit
    n_emit: torch.Tensor     # [B] int32 tokens committed this round
    finished: torch.Tensor   # [B] int32
    tgt_argmax: torch.Tensor | None = None  # [B, S+1] when computed from logits

    @classmethod
    def alloc(cls, B: int, S: int, device, with_argmax: bool = False) -> "AcceptOut":
        z = lambda *sh: torch.empty(sh, dtype=torch.int32, device=device)  # noqa: E731
        return cls(z(B), z(B, S + 1), z(B), z(B), z(B, S + 1) if with_argmax else None)


def accept_batch(draft: torch.Tensor, tgt_argmax: torch.Tensor, remaining: torch.Tensor,
                 stop_token: int | None = None, kv_len: torch.Tensor | None = None,
                 out: AcceptOut | None = None, stream=None) -> AcceptOut:
    """K9 on device tensors: draft [B, S], tgt_argmax [B, S+1], remaining [B]."""
    dev = _dev.require_cuda()
    B, S = draft.shape
    if tgt_argmax.shape != (B, S + 1):
        raise DistMismatch(f"expected target argmax [{B}, {S + 1}], got {tuple(tgt_argmax.shape)}")
    out = out or AcceptOut.alloc(B, S, dev)
    _native.call("ms_accept_greedy", _dev.ptr(draft, torch.int32, "draft"),
                 _dev.ptr(tgt_argmax, torch.int32, "tgt_argmax"),
                 _dev.ptr(remaining, torch.int32, "remaining"),
                 -1 if stop_token is None else int(stop_token), B, S,
                 _dev.ptr(out.n_acc), _dev.ptr(out.emitted), _dev.ptr(out.n_emit),
                 _dev.ptr(out.finished), _dev.ptr(kv_len, torch.int32, "kv_len"),
                 _dev.stream_ptr(stream))
    return out


def argmax_rows(logits: torch.Tensor, out: torch.Tensor | None = None,
                ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """K8 (unfused): first-index argmax of each row of [R, V] fp32/bf16 logits."""
    dev = _dev.require_cuda()
    if logits.dim() != 2 or logits.stride(1) != 1:
        raise ValueError("logits must be [R, V] with unit column stride")
    R, V = logits.shape
    if logits.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("logits must be fp32 or bf16")
    out = out if out is not None else torch.empty(R, dtype=torch.int32, device=dev)
    ws = ws if ws is not None else torch.empty(R, dtype=torch.int64, device=dev)
    _native.call("ms_argmax_rows", logits.data_ptr(), int(logits.dtype == torch.bfloat16), R, V,
                 logits.stride(0), _dev.ptr(out, torch.int32), _dev.ptr(ws, torch.int64),
                 _dev.stream_ptr(stream))
    return out


def accept_batch_logits(draft: torch.Tensor, logits: torch.Tensor, remaining: torch.Tensor,
                        stop_token: int | None = None, kv_len: torch.Tensor | None = None,
                        out: AcceptOut | None = None, ws: torch.Tensor | None = None,
                        stream=None) -> AcceptOut:
    """K8 + K9: draft [B, S] against target logits [B, S+1, V] (fp32 or bf16)."""
    dev = _dev.require_cuda()
    B, S = draft.shape
    if logits.dim() != 3 or logits.shape[:2] != (B, S + 1):
        raise DistMismatch(f"expected logits [{B}, {S + 1}, V], got {tuple(logits.shape)}")
    if logits.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("logits must be fp32 or bf16")
    V = logits.shape[2]
    out = out or AcceptOut.alloc(B, S, dev, with_argmax=True)
    if out.tgt_argmax is None:
        out.tgt_argmax = torch.empty((B, S + 1), dtype=torch.int32, device=dev)
    ws = ws if ws is not None else torch.empty(B * (S + 1), dtype=torch.int64, device=dev)
    _native.call("ms_accept_greedy_logits", _dev.ptr(draft, torch.int32, "draft"),
                 _dev.ptr(logits, None, "logits"), int(logits.dtype == torch.bfloat16), V,
                 _dev.ptr(remaining, torch.int32, "remaining"),
                 -1 if stop_token is None else int(stop_token), B, S,
                 _dev.ptr(out.tgt_argmax), _dev.ptr(ws, torch.int64), _dev.ptr(out.n_acc),
                 _dev.ptr(out.emitted), _dev.ptr(out.n_emit), _dev.ptr(out.finished),
                 _dev.ptr(kv_len, torch.int32, "kv_len"), _dev.stream_ptr(stream))
    return out


def accept_batch_stochastic(draft: torch.Tensor, q: torch.Tensor, o: torch.Tensor,
                            uniforms: torch.Tensor, remaining: torch.Tensor,
                            stop_token: int | None = None, out: AcceptOut | None = None,
                            scratch: torch.Tensor | None = None, stream=None):
    """K10 on device tensors: draft [B, S] int32, q [B, S, V] fp64, o [B, S+1, V]
    fp64, uniforms [B, S+1] fp64 (peeked from each request's verify stream).
    Returns (AcceptOut, n_draws [B] int32)."""
    dev = _dev.require_cuda()
    B, S = draft.shape
    V = q.shape[-1]
    if q.shape != (B, S, V) or o.shape != (B, S + 1, V):
        raise DistMismatch(f"expected q [{B}, {S}, V] and o [{B}, {S + 1}, V]")
    if uniforms.shape != (B, S + 1):
        raise ValueError(f"expected uniforms [{B}, {S + 1}]")
    out = out or AcceptOut.alloc(B, S, dev)
    n_draws = torch.empty(B, dtype=torch.int32, device=dev)
    scratch = scratch if scratch is not None else torch.empty((B, V), dtype=torch.float64, device=dev)
    _native.call("ms_accept_stochastic", _dev.ptr(draft, torch.int32, "draft"),
                 _dev.ptr(q, torch.float64, "q"), _dev.ptr(o, torch.float64, "o"),
                 _dev.ptr(uniforms, torch.float64, "uniforms"),
                 _dev.ptr(remaining, torch.int32, "remaining"),
                 -1 if stop_token is None else int(stop_token), B, S, V,
                 _dev.ptr(scratch, torch.float64), _dev.ptr(out.n_acc), _dev.ptr(out.emitted),
                 _dev.ptr(out.n_emit), _dev.ptr(out.finished), _dev.ptr(n_draws),
                 _dev.stream_ptr(stream))
    return out, n_draws


def peek_uniforms(rng: np.random.Generator, n: int) -> np.ndarray:
    """The next n doubles of rng without consuming them (PCG64 state peek)."""
    state = rng.bit_generator.state
    u = rng.random(n)
    rng.bit_generator.state = state
    return u


def verify(draft_tokens: Sequence[int], draft_dists: Sequence[ProbDist],
           target_dists: Sequence[ProbDist], rng: np.random.Generator) -> VerificationResult:
    """aggspec/verification.py:29-77 with the same checks and RNG consumption."""
    s = len(draft_tokens)
    if s < 1:
        raise ValueError("draft must contain at least one token")
    if len(draft_dists) != s:
        raise DistMismatch(f"expected {s} draft distributions, got {len(draft_dists)}")
    if len(target_dists) != s + 1:
        raise DistMismatch(f"expected {s + 1} target distributions, got {len(target_dists)}")
    V = draft_dists[0].vocab_size
    if any(d.vocab_size != V for d in (*draft_dists, *target_dists)):
        raise DistMismatch("draft and target distributions must share a vocabulary")
    # the reference reads probs.item(tok): negative tokens wrap, tokens outside
    # [-V, V) raise IndexError when (and only if) verification reaches them
    bad = next((i for i, t in enumerate(draft_tokens) if not -V <= int(t) < V), s)
    q_tok = [d.point_mass_token() for d in draft_dists]
    o_tok = [d.point_mass_token() for d in target_dists]
    dev = _dev.require_cuda()
    draft = torch.tensor([list(map(int, draft_tokens))], dtype=torch.int32, device=dev)
    rem = torch.tensor([s + 1], dtype=torch.int32, device=dev)
    if all(t is not None for t in (*q_tok, *o_tok)) and all(
            qt == int(t) for qt, t in zip(q_tok, draft_tokens)):
        # greedy fast path (K9): point masses on both sides
        tgt = torch.tensor([o_tok], dtype=torch.int32, device=dev)
        o = accept_batch(draft, tgt, rem)
        acc = int(o.n_acc[0])
        emitted = o.emitted[0, : acc + 1].tolist()
        rng.random(acc + 2 if acc < s else s + 1)  # uniforms the reference consumes
        return VerificationResult(acc, emitted, acc / s)
    # general speculative sampling (K10), bit-exact on the same fp64 dists / uniforms
    wrapped = [int(t) % V if -V <= int(t) < 0 else int(t) for t in draft_tokens]
    draft = torch.tensor([wrapped], dtype=torch.int32, device=dev)  # out-of-range: no probability
    qd = torch.from_numpy(np.stack([d.probs for d in draft_dists])[None]).to(dev)
    od = torch.from_numpy(np.stack([d.probs for d in target_dists])[None]).to(dev)
    u = torch.from_numpy(peek_uniforms(rng, s + 1)[None]).to(dev)
    o, n_draws = accept_batch_stochastic(draft, qd, od, u, rem)
    acc = int(o.n_acc[0])
    if acc >= bad < s:  # positions before `bad` all accepted: the reference reaches it
        rng.random(bad)
        raise IndexError(f"draft token {int(draft_tokens[bad])} outside the vocabulary of size {V}")
    emitted = list(draft_tokens[:acc]) + [int(o.emitted[0, acc])]
    rng.random(int(n_draws[0]))  # advance the stream exactly as the reference did
    return VerificationResult(acc, emitted, acc / s)


def acceptance_rate(result: VerificationResult, s: int) -> float:
    """accepted_count / s (aggspec/verification.py:80-82)."""
    return result.accepted_count / s
