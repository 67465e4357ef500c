"""fp32 CPU ModelOracles over the model restatements — TEST INFRASTRUCTURE ONLY.

The reference's model plug-in point is the ModelOracle protocol
(aggspec/oracles.py:19-26: vocab_size, context_cap, next_dist(context) ->
ProbDist).  The reference ships only synthetic oracles (Markov / Dirichlet);
this adapter puts a transformer behind the protocol — opt_ref.forward or
llama_ref.forward over the same random-init weights the device uses — so the
UNMODIFIED reference engine (aggspec/engine.py:252-330, run_sequential /
run_pipelined at :619-671) can produce golden token streams and per-round
decisions (tests/golden/make_engine_golden.py), and so the reference arm of
bench.py can time the reference's own CPU path end to end.

mode "greedy": next_dist is the point mass on the first-index argmax of the
fp32 logits (the greedy contract).  mode "sample": the softmax in
fp64, p = exp(l - max) / sum(exp(l - max)) over the fp32 logits — the
distribution the device's stochastic path samples (paper_2402_15678_b200/
csrc/sample.cu mirrors this formula).

exact=True: the fp32 verification-mode contract (no bf16 rounding anywhere);
exact=False: the bf16 product contract.
"""
from __future__ import annotations

import sys
from importlib import import_module

import numpy as np
import torch

from . import llama_ref, opt_ref


def _prob_dist_cls():
    """aggspec.core.ProbDist when the reference is loaded (golden runs, the
    reference bench arm), else the package's restatement."""
    core = sys.modules.get("aggspec.core") or import_module("paper_2402_15678_b200.core")
    return core.ProbDist


class CPUModelOracle:
    def __init__(self, w: dict, cfg, exact: bool = True, mode: str = "greedy", context_cap: int = 4096,
                 fused_norm: bool = False):
        if mode not in ("greedy", "sample"):
            raise ValueError("mode must be 'greedy' or 'sample'")
        self.w = {k: v.float() for k, v in w.items()}  # converted once (forward's .float() is then a no-op)
        self.cfg = cfg
        self.exact, self.mode = exact, mode
        self.fused_norm = fused_norm
        self.vocab_size = cfg.vocab
        self.context_cap = context_cap
        self.calls = 0
        self.min_margin = float("inf")  # smallest top-1 minus top-2 logit seen (fp32 parity headroom)

    def logits(self, context) -> torch.Tensor:
        self.calls += 1
        if getattr(self.cfg, "family", "opt") == "llama":
            out = llama_ref.forward(self.w, self.cfg, context, last_only=True, fused_norm=self.fused_norm,
                                    exact=self.exact)
        else:
            out = opt_ref.forward(self.w, self.cfg, context, last_only=True, exact=self.exact)
        top = torch.topk(out[-1], 2).values
        self.min_margin = min(self.min_margin, float(top[0] - top[1]))
        return out[-1]

    def next_dist(self, context):
        if len(context) > self.context_cap:
            raise ValueError("context exceeds context_cap")
        lg = self.logits(context)
        P = _prob_dist_cls()
        if self.mode == "greedy":
            p = np.zeros(self.vocab_size)
            p[int(torch.argmax(lg))] = 1.0
            return P(p)
        return P(softmax64(lg.numpy()))


def softmax64(logits: np.ndarray) -> np.ndarray:
    """p = exp(l - max) / sum(exp(l - max)) in fp64 over fp32 logits."""
    l64 = np.asarray(logits, dtype=np.float32).astype(np.float64)
    e = np.exp(l64 - l64.max())
    return e / e.sum()
