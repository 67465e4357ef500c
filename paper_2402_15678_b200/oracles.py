"""The model plug-in boundary (mirrors aggspec/oracles.py:19-153).

* `ModelOracle` — the reference's runtime-checkable protocol: `vocab_size`,
  `context_cap`, `next_dist(context) -> ProbDist` (aggspec/oracles.py:19-26).
* `draft_sequence(oracle, context, s, rng)` — s autoregressive steps, same
  signature / errors / RNG use as aggspec/oracles.py:135-153.
* `GPUOracle` (alias `OPTOracle`) — a GPU model of either family (OPT or
  Llama-2, models.make_model on libminions kernels) behind that protocol, greedy: next_dist is the point mass on the first-index argmax.  It
  keeps a one-slot KV cache and feeds only the context suffix it has not seen,
  so the reference's per-position call pattern (draft_sequence, the verify
  loop of aggspec/engine.py:294-296) costs one decode step per call instead of
  a full forward.  This is the drop-in for code that drives models through
  the reference's protocol; the batched engine (engine.py) is the fast path.
"""
from __future__ import annotations

from typing import Protocol, Sequence, runtime_checkable

import numpy as np
import torch

from . import _dev
from . import _native
from .core import ContextTooLong, ProbDist
from .models import make_model
from .opt import KVCache

__all__ = ["ContextTooLong", "ModelOracle", "draft_sequence", "GPUOracle", "OPTOracle"]

DEFAULT_CONTEXT_CAP = 4096


@runtime_checkable
class ModelOracle(Protocol):
    vocab_size: int
    context_cap: int

    def next_dist(self, context: Sequence[int]) -> ProbDist: ...


def _check_context(oracle, context: Sequence[int]) -> None:
    if len(context) == 0:
        raise ValueError("context must be non-empty")
    if len(context) > oracle.context_cap:
        raise ContextTooLong(f"context length {len(context)} exceeds cap {oracle.context_cap}")


def draft_sequence(oracle: ModelOracle, context: Sequence[int], s: int,
                   rng: np.random.Generator) -> tuple[list[int], list[ProbDist]]:
    """Sample s tokens autoregressively; one `rng.random()` per step (ProbDist.sample)."""
    if s < 1:
        raise ValueError("s must be >= 1")
    ctx = list(context)
    toks: list[int] = []
    dists: list[ProbDist] = []
    for _ in range(s):
        d = oracle.next_dist(ctx)
        t = d.sample(rng)
        toks.append(t)
        dists.append(d)
        ctx.append(t)
    return toks, dists


class GPUOracle:
    """Greedy GPU model (OPT or Llama-2 weights) behind the ModelOracle protocol."""

    def __init__(self, weights, context_cap: int = 1024, device="cuda"):
        _dev.require_cuda()
        self.cfg = weights.cfg
        self.vocab_size = weights.cfg.vocab
        self.context_cap = context_cap
        self.model = make_model(weights, max_rows=context_cap, device=device)
        self.cache = KVCache(weights.cfg, 1, context_cap + 1, device)
        self.dev = torch.device(device)
        self._seen: list[int] = []  # tokens whose KV is cached
        self._slot = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._logits = torch.empty(1, self.vocab_size, device=self.dev)
        self._am = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._ws = torch.zeros(1, dtype=torch.int64, device=self.dev)

    def argmax_next(self, context: Sequence[int]) -> int:
        _check_context(self, context)
        ctx = [int(t) for t in context]
        # longest cached prefix (the last token is always re-fed)
        n = 0
        lim = min(len(self._seen), len(ctx) - 1)
        while n < lim and self._seen[n] == ctx[n]:
            n += 1
        feed = ctx[n:]
        toks = torch.tensor([feed], dtype=torch.int32, device=self.dev)
        start = torch.tensor([n], dtype=torch.int32, device=self.dev)
        rows = torch.tensor([len(feed) - 1], dtype=torch.int32, device=self.dev)
        self.model.forward(toks, start, self._slot, self.cache, self._logits, head_rows=rows)
        _native.call("ms_argmax_rows", self._logits.data_ptr(), 0, 1, self.vocab_size, self.vocab_size,
                     self._am.data_ptr(), self._ws.data_ptr(), _dev.stream_ptr())
        self._seen = ctx
        return int(self._am.item())

    def next_dist(self, context: Sequence[int]) -> ProbDist:
        p = np.zeros(self.vocab_size)
        p[self.argmax_next(context)] = 1.0
        return ProbDist(p)


OPTOracle = GPUOracle  # the name the OPT-only first version exported
