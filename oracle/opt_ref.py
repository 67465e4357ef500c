"""fp32 PyTorch-CPU reference of the OPT-style decoder — TEST INFRASTRUCTURE ONLY.

The reference package has no model (its ModelOracle protocol,
aggspec/oracles.py:19-26, is the plug-in point), so model numerics are pinned
against this restatement rather than against the reference: parity of the
forward is "unpinned by the reference" and checked with a stated
tolerance plus the argmax agreement rate.

It mirrors the device path's numerics contract (paper_2402_15678_b200/csrc/
model.cu, gemm.cu): bf16 weights and bf16 activations between kernels, every
reduction in fp32, each op rounding its result to bf16 once; only the fp32
summation order differs.  `OracleModel` also implements the reference's
`ModelOracle` protocol (greedy point-mass next_dist) so the reference engine
can drive it for the CPU baseline.
"""
from __future__ import annotations

import math

import numpy as np
import torch

BF16 = torch.bfloat16


def _bf(x: torch.Tensor) -> torch.Tensor:
    """Round fp32 -> bf16 -> fp32 (one rounding point of the contract)."""
    return x.to(BF16).to(torch.float32)


def _id(x: torch.Tensor) -> torch.Tensor:
    return x


def layernorm(x, g, b, eps, rnd=_bf):
    mean = x.mean(-1, keepdim=True)
    var = ((x - mean) ** 2).mean(-1, keepdim=True)
    return rnd((x - mean) * torch.rsqrt(var + eps) * g + b)


def forward(w: dict, cfg, tokens, start: int = 0, last_only: bool = False, exact: bool = False) -> torch.Tensor:
    """Full causal forward of one sequence (positions start..start+T-1 with no
    cache: start must be 0).  tokens: [T] ints -> logits [T, V] fp32 (or [1, V]
    for the last position only).

    exact=True: the fp32 verification-mode contract (paper_2402_15678_b200/
    fp32.py) — no bf16 rounding point anywhere, every op in fp32."""
    assert start == 0
    rnd = _id if exact else _bf
    f32 = {k: v.float() for k, v in w.items()}
    tok = torch.as_tensor(list(tokens), dtype=torch.long)
    T = tok.numel()
    pos = torch.arange(T) + cfg.pos_offset
    x = rnd(f32["tok_emb"][tok] + f32["pos_emb"][pos])
    H, D = cfg.n_heads, cfg.head_dim
    scale = 1.0 / math.sqrt(D)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool), 1)
    for i in range(cfg.n_layers):
        p = f"l{i}."
        h = layernorm(x, f32[p + "ln1_g"], f32[p + "ln1_b"], cfg.eps, rnd)
        qkv = rnd(h @ f32[p + "w_qkv"].T + f32[p + "b_qkv"])
        q, k, v = qkv.split(cfg.d, dim=-1)
        q = q.view(T, H, D).transpose(0, 1) * scale
        k = k.view(T, H, D).transpose(0, 1)
        v = v.view(T, H, D).transpose(0, 1)
        s = q @ k.transpose(1, 2)
        s = s.masked_fill(mask, float("-inf"))
        a = torch.softmax(s, dim=-1) @ v
        a = rnd(a.transpose(0, 1).reshape(T, cfg.d))
        x = rnd(a @ f32[p + "w_o"].T + f32[p + "b_o"] + x)
        h = layernorm(x, f32[p + "ln2_g"], f32[p + "ln2_b"], cfg.eps, rnd)
        ff = rnd(torch.relu(h @ f32[p + "w_fc1"].T + f32[p + "b_fc1"]))
        x = rnd(ff @ f32[p + "w_fc2"].T + f32[p + "b_fc2"] + x)
    if last_only:
        x = x[-1:]
    h = layernorm(x, f32["lnf_g"], f32["lnf_b"], cfg.eps, rnd)
    return h @ f32["tok_emb"].T


def greedy_generate(w, cfg, prompt, n_new: int, exact: bool = False) -> list[int]:
    """Plain greedy decoding (first-index argmax), no speculation."""
    ctx = list(prompt)
    for _ in range(n_new):
        logits = forward(w, cfg, ctx, last_only=True, exact=exact)[-1]
        ctx.append(int(torch.argmax(logits)))
    return ctx[len(prompt):]


class OracleModel:
    """The reference's ModelOracle protocol (vocab_size, context_cap,
    next_dist) over `forward`, greedy: next_dist is the point mass on the
    first-index argmax (the greedy contract of SURVEY §0 fact 1)."""

    def __init__(self, w: dict, cfg, context_cap: int = 4096):
        self.w, self.cfg = w, cfg
        self.vocab_size = cfg.vocab
        self.context_cap = context_cap
        self._f32 = None

    def argmax_next(self, context) -> int:
        return int(torch.argmax(forward(self.w, self.cfg, context, last_only=True)[-1]))

    def next_dist(self, context):
        import sys
        from importlib import import_module
        core = sys.modules.get("aggspec.core") or import_module("paper_2402_15678_b200.core")
        p = np.zeros(self.vocab_size)
        p[self.argmax_next(context)] = 1.0
        return core.ProbDist(p)
