"""fp32 verification mode: the OPT and Llama-2 forwards with fp32 activations,
fp32 KV cache and fp32 accumulation (csrc/fp32.cu), behind the same
forward(tokens, start, slot, cache, logits, head_rows) interface as
opt.OPTModel / llama.LlamaModel, so SpecEngine(precision="fp32") runs the
speculate-vote-verify rounds unchanged on top of it.

Why: north_star asks for accepted token sequences and vote results bit-exact
against the reference in an fp32 verification mode.  The reference engine
(aggspec/engine.py:252-330) is driven, in the golden generator, by fp32 CPU
ModelOracles (aggspec/oracles.py:19-26 protocol; oracle/opt_ref.py and
oracle/llama_ref.py with exact=True: no bf16 rounding anywhere).  This module
is the device side of that contract: nothing is rounded below fp32, so the
device and the CPU oracle differ only by fp32 summation order.  The weights
are the same bf16 tensors as the bf16 path (bf16 values are exact in fp32).
"""
from __future__ import annotations

import math

import torch

from . import _dev
from . import _native
from .kernels import rope_table

F32 = torch.float32
BF16 = torch.bfloat16


def embed(tok, start, Q, tok_emb, pos_emb, pos_offset, out, stream=None):
    R, d = tok.numel(), tok_emb.shape[1]
    _native.call("ms_embed_f32", _dev.ptr(tok, torch.int32, "tok"), _dev.ptr(start, torch.int32, "start"), Q,
                 _dev.ptr(tok_emb, BF16), _dev.ptr(pos_emb, BF16), pos_offset, R, d, _dev.ptr(out, F32),
                 _dev.stream_ptr(stream))
    return out


def norm(x, gamma, beta, eps, out, rows=None, rms=False, stream=None):
    """LayerNorm (beta given) or RMSNorm (rms=True) of x rows, fp32."""
    d = x.shape[1]
    R = x.shape[0] if rows is None else rows.numel()
    _native.call("ms_norm_f32", _dev.ptr(x, F32), x.stride(0), _dev.ptr(rows, torch.int32, "rows"),
                 _dev.ptr(gamma, BF16), _dev.ptr(beta, BF16), eps, int(rms), R, d, _dev.ptr(out, F32),
                 out.stride(0), _dev.stream_ptr(stream))
    return out


def linear(x, w, out, bias=None, residual=None, act=0, stream=None):
    """out = act(x @ w.T + bias) (+ residual); x/out/residual fp32, w bf16;
    act=2: gated SiLU of the 64-row interleaved gate/up weight."""
    M, K = x.shape
    N = w.shape[0]
    if w.dtype != BF16 or not w.is_contiguous() or w.shape[1] != K or x.stride(1) != 1:
        raise ValueError("x [M, K] fp32 and w [N, K] contiguous bf16")
    _native.call("ms_linear_f32", _dev.ptr(x, F32), x.stride(0), w.data_ptr(),
                 None if bias is None else _dev.ptr(bias, BF16, "bias"),
                 None if residual is None else _dev.ptr(residual, F32),
                 0 if residual is None else residual.stride(0), _dev.ptr(out, F32), out.stride(0), M, N, K, act,
                 _dev.stream_ptr(stream))
    return out


def attention(qkv, B, Q, H, Hkv, D, slot, start, k_cache, v_cache, scale, out, rope=None, scale_q=False,
              stream=None):
    T = k_cache.shape[2]
    if k_cache.dtype != F32 or v_cache.dtype != F32:
        raise ValueError("fp32 mode needs an fp32 KV cache")
    _native.call("ms_attention_f32", _dev.ptr(qkv, F32), qkv.stride(0), B, Q, H, Hkv, D,
                 _dev.ptr(slot, torch.int32), _dev.ptr(start, torch.int32), T, k_cache.data_ptr(),
                 v_cache.data_ptr(), None if rope is None else _dev.ptr(rope, F32), scale, int(scale_q),
                 _dev.ptr(out, F32), out.stride(0), _dev.stream_ptr(stream))
    return out


class _F32Model:
    precision = "fp32"

    def __init__(self, w, max_rows: int, device="cuda"):
        self.w, self.cfg = w, w.cfg
        c = self.cfg
        self.device = torch.device(device)
        self.max_rows = max_rows
        H, Hkv, D = c.n_heads, c.n_kv_heads, c.head_dim
        self.x = torch.empty((max_rows, c.d), dtype=F32, device=device)
        self.h = torch.empty((max_rows, c.d), dtype=F32, device=device)
        self.qkv = torch.empty((max_rows, (H + 2 * Hkv) * D), dtype=F32, device=device)
        self.attn = torch.empty((max_rows, H * D), dtype=F32, device=device)
        self.ff = torch.empty((max_rows, c.ffn), dtype=F32, device=device)
        self.scale = 1.0 / math.sqrt(D)

    def _check(self, tokens, cache):
        if tokens.numel() > self.max_rows:
            raise ValueError(f"{tokens.numel()} rows exceed max_rows={self.max_rows}")
        if cache.k[0].dtype != F32:
            raise ValueError("fp32 mode needs KVCache(..., dtype=torch.float32)")


class OPTModelF32(_F32Model):
    """OPT-style decoder in fp32 (contract: oracle/opt_ref.forward(exact=True))."""

    def forward(self, tokens, start, slot, cache, logits, head_rows=None, stream=None, prefill: bool = False):
        self._check(tokens, cache)
        c, w = self.cfg, self.w
        B, Q = tokens.shape
        R = B * Q
        x, h, qkv, at, ff = self.x[:R], self.h[:R], self.qkv[:R], self.attn[:R], self.ff[:R]
        embed(tokens, start, Q, w["tok_emb"], w["pos_emb"], c.pos_offset, out=x, stream=stream)
        for i in range(c.n_layers):
            p = f"l{i}."
            norm(x, w[p + "ln1_g"], w[p + "ln1_b"], c.eps, out=h, stream=stream)
            linear(h, w[p + "w_qkv"], qkv, bias=w[p + "b_qkv"], stream=stream)
            attention(qkv, B, Q, c.n_heads, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i],
                      self.scale, at, scale_q=True, stream=stream)
            linear(at, w[p + "w_o"], x, bias=w[p + "b_o"], residual=x, stream=stream)
            norm(x, w[p + "ln2_g"], w[p + "ln2_b"], c.eps, out=h, stream=stream)
            linear(h, w[p + "w_fc1"], ff, bias=w[p + "b_fc1"], act=1, stream=stream)
            linear(ff, w[p + "w_fc2"], x, bias=w[p + "b_fc2"], residual=x, stream=stream)
        Rh = R if head_rows is None else head_rows.numel()
        if Rh == 0:
            return logits
        hf = self.h[:Rh]
        norm(x, w["lnf_g"], w["lnf_b"], c.eps, out=hf, rows=head_rows, stream=stream)
        linear(hf, w["tok_emb"], logits, stream=stream)
        return logits


class LlamaModelF32(_F32Model):
    """Llama-2-style decoder in fp32 (contract: oracle/llama_ref.forward(exact=True),
    explicit RMSNorms — no norm folding)."""

    def __init__(self, w, max_rows: int, device="cuda"):
        super().__init__(w, max_rows, device)
        c = self.cfg
        self.rope = rope_table(c.max_pos, c.head_dim, c.rope_theta, device=device)

    def forward(self, tokens, start, slot, cache, logits, head_rows=None, stream=None, prefill: bool = False):
        self._check(tokens, cache)
        c, w = self.cfg, self.w
        if cache.max_len > c.max_pos:
            raise ValueError("KV cache longer than the RoPE table")
        B, Q = tokens.shape
        R = B * Q
        x, h, qkv, at, ff = self.x[:R], self.h[:R], self.qkv[:R], self.attn[:R], self.ff[:R]
        embed(tokens, start, Q, w["tok_emb"], None, 0, out=x, stream=stream)
        for i in range(c.n_layers):
            p = f"l{i}."
            norm(x, w[p + "attn_norm"], None, c.eps, out=h, rms=True, stream=stream)
            linear(h, w[p + "w_qkv"], qkv, stream=stream)
            attention(qkv, B, Q, c.n_heads, c.n_kv_heads, c.head_dim, slot, start, cache.k[i], cache.v[i],
                      self.scale, at, rope=self.rope, stream=stream)
            linear(at, w[p + "w_o"], x, residual=x, stream=stream)
            norm(x, w[p + "mlp_norm"], None, c.eps, out=h, rms=True, stream=stream)
            linear(h, w[p + "w_gu"], ff, act=2, stream=stream)
            linear(ff, w[p + "w_down"], x, residual=x, stream=stream)
        Rh = R if head_rows is None else head_rows.numel()
        if Rh == 0:
            return logits
        hf = self.h[:Rh]
        norm(x, w["norm_f"], None, c.eps, out=hf, rows=head_rows, rms=True, stream=stream)
        linear(hf, w["lm_head"], logits, stream=stream)
        return logits
