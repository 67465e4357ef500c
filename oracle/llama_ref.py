"""fp32 PyTorch-CPU reference of the Llama-2-style decoder — TEST INFRASTRUCTURE ONLY.

The reference package has no model (ModelOracle, aggspec/oracles.py:19-26, is
the plug-in point): model numerics are "parity unpinned by the reference"
 and checked against this restatement with a stated tolerance plus
the argmax agreement rate.

Numerics contract of the device path (paper_2402_15678_b200/llama.py,
csrc/model.cu, attention.cu, gemm.cu): bf16 weights/activations between
kernels, fp32 reductions, one bf16 rounding per op — RMSNorm, the QKV GEMM,
RoPE of q and k (fp32 table of (cos, sin) computed in fp64, rotate-half
pairing), attention, O-proj + residual, gated SiLU silu(g)*u in fp32 from the
fp32 gate/up GEMM accumulators (rounded once), down-proj + residual; LM-head
logits fp32.  Only the fp32 summation order differs.
"""
from __future__ import annotations

import math

import numpy as np
import torch

BF16 = torch.bfloat16


def _bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(BF16).to(torch.float32)


def _id(x: torch.Tensor) -> torch.Tensor:
    return x


def rmsnorm(x, g, eps, rnd=_bf):
    return rnd(x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * g)


def rope_table(max_pos: int, D: int, theta: float) -> torch.Tensor:
    inv = theta ** (-np.arange(0, D, 2, dtype=np.float64) / D)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.stack([np.cos(ang), np.sin(ang)], -1).astype(np.float32))


def rope(x: torch.Tensor, pos: torch.Tensor, table: torch.Tensor, rnd=_bf) -> torch.Tensor:
    """x [T, H, D] fp32 (bf16 values), rotate-half pairing, one bf16 rounding."""
    D = x.shape[-1]
    cs = table[pos]  # [T, D/2, 2]
    c, s = cs[..., 0][:, None, :], cs[..., 1][:, None, :]
    a, b = x[..., : D // 2], x[..., D // 2:]
    return rnd(torch.cat([a * c - b * s, b * c + a * s], dim=-1))


def split_gate_up(w_gu: torch.Tensor, ffn: int):
    j = torch.arange(ffn)
    gate = (j // 64) * 128 + j % 64
    return w_gu[gate], w_gu[gate + 64]


def fold(w: dict, cfg) -> dict:
    """LlamaWeights.fold_norms restated: gains folded into the consuming
    projection with one bf16 rounding, gains := 1."""
    out = dict(w)
    pairs = [(f"l{i}.attn_norm", f"l{i}.w_qkv") for i in range(cfg.n_layers)]
    pairs += [(f"l{i}.mlp_norm", f"l{i}.w_gu") for i in range(cfg.n_layers)] + [("norm_f", "lm_head")]
    for g, name in pairs:
        out[name] = (w[name].float() * w[g].float()[None, :]).to(BF16)
        out[g] = torch.ones_like(w[g])
    return out


def rstd(x, eps):
    return torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)


def forward(w: dict, cfg, tokens, last_only: bool = False, fused_norm: bool = False,
            exact: bool = False) -> torch.Tensor:
    """Full causal forward of one sequence from position 0 (no cache).
    tokens [T] -> logits [T, V] fp32 (or [1, V]).

    fused_norm: the verifier's contract (LlamaModel fuse_norm): gains folded
    into the next projection; for every layer but the first the projection
    runs on the raw residual stream and its fp32 result is scaled by
    rstd(x) = rsqrt(mean(x^2) + eps), rounded once — no bf16 normalised
    activation in between.

    exact=True: the fp32 verification-mode contract (paper_2402_15678_b200/
    fp32.py) — no bf16 rounding point anywhere (explicit norms only)."""
    if exact and fused_norm:
        raise ValueError("the fp32 mode has explicit norms (fused_norm=False)")
    rnd = _id if exact else _bf
    if fused_norm:
        w = fold(w, cfg)
    f32 = {k: v.float() for k, v in w.items()}
    tok = torch.as_tensor(list(tokens), dtype=torch.long)
    T = tok.numel()
    H, Hkv, D = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    G = H // Hkv
    table = rope_table(max(T, 1), D, cfg.rope_theta)
    pos = torch.arange(T)
    x = f32["tok_emb"][tok]
    scale = 1.0 / math.sqrt(D)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool), 1)
    for i in range(cfg.n_layers):
        p = f"l{i}."
        if fused_norm and i > 0:
            qkv = rnd((x @ f32[p + "w_qkv"].T) * rstd(x, cfg.eps))
        else:
            h = rmsnorm(x, f32[p + "attn_norm"], cfg.eps, rnd)
            qkv = rnd(h @ f32[p + "w_qkv"].T)
        q = rope(qkv[:, : H * D].view(T, H, D), pos, table, rnd)
        k = rope(qkv[:, H * D: (H + Hkv) * D].view(T, Hkv, D), pos, table, rnd)
        v = qkv[:, (H + Hkv) * D:].view(T, Hkv, D)
        k = k.repeat_interleave(G, dim=1)  # query head h reads KV head h // G
        v = v.repeat_interleave(G, dim=1)
        sc = (q.transpose(0, 1) @ k.transpose(0, 1).transpose(1, 2)) * scale
        sc = sc.masked_fill(mask, float("-inf"))
        a = rnd((torch.softmax(sc, dim=-1) @ v.transpose(0, 1)).transpose(0, 1).reshape(T, H * D))
        x = rnd(a @ f32[p + "w_o"].T + x)
        wg, wu = split_gate_up(f32[p + "w_gu"], cfg.ffn)
        if fused_norm:
            r = rstd(x, cfg.eps)
            gt, up = (x @ wg.T) * r, (x @ wu.T) * r
        else:
            h = rmsnorm(x, f32[p + "mlp_norm"], cfg.eps, rnd)
            gt, up = h @ wg.T, h @ wu.T
        ff = rnd(gt / (1.0 + torch.exp(-gt)) * up)
        x = rnd(ff @ f32[p + "w_down"].T + x)
    if last_only:
        x = x[-1:]
    if fused_norm:
        return (x @ f32["lm_head"].T) * rstd(x, cfg.eps)
    return rmsnorm(x, f32["norm_f"], cfg.eps, rnd) @ f32["lm_head"].T


def greedy_generate(w, cfg, prompt, n_new: int, fused_norm: bool = False, exact: bool = False) -> list[int]:
    ctx = list(prompt)
    for _ in range(n_new):
        ctx.append(int(torch.argmax(forward(w, cfg, ctx, last_only=True, fused_norm=fused_norm, exact=exact)[-1])))
    return ctx[len(prompt):]
