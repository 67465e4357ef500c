"""OPT-style decoder (pre-LN, learned positions, ReLU FFN, tied LM head) on the
libminions kernels: the SSM drafters and the LLM verifier of the speculation
path.

The reference has no model: `ModelOracle.next_dist(context)`
(aggspec/oracles.py:19-26) stands in for one forward position, called s times
per drafter by draft_sequence (aggspec/oracles.py:135-153) and s+1 times per
request by the verify loop (aggspec/engine.py:294-296).  Here one `forward`
call runs Q consecutive positions for B requests at once against a KV cache:
Q = s+1 for the verifier, Q = 1 per SSM decode step.

Memory layout (HBM):
  weights    bf16, nn.Linear [out, in]; q/k/v fused as w_qkv [3d, d]
  KV cache   per layer K and V [slots, H, T, D] bf16 — a (slot, head) pair is
             one contiguous [T, D] stream for the attention kernel
  activations x [B*Q, d] bf16 residual stream, updated in place by the
             O-proj / FC2 epilogues (residual add fused)
"""
from __future__ import annotations

import math

import torch

from . import kernels as K

from .weights import KVCache, OPTConfig, OPTWeights  # noqa: F401
from .weights import OPT_CONFIGS as CONFIGS  # noqa: F401

BF16 = torch.bfloat16


class OPTModel:
    """Batched forward over the kernels with static activation buffers (so a
    forward of a given (B, Q) can be captured in a CUDA graph)."""


    def __init__(self, w: OPTWeights, max_rows: int, device="cuda", small_gemm: bool = False,
                 split_kv: bool = False):
        """small_gemm: layer GEMMs of <= 64 token rows use the low-latency
        ms_gemv (drafters' decode steps); the verifier keeps the tcgen05 path
        everywhere, so its numerics never depend on the row count.
        split_kv: attention split over the cache length (fixed chunks, merged
        in chunk order; measured slower on the benchmark's shapes)."""
        self.split_kv = bool(split_kv)
        self.w, self.cfg = w, w.cfg
        self.small_gemm = small_gemm
        c = self.cfg
        self.device = torch.device(device)
        self.max_rows = max_rows
        self.x = torch.empty((max_rows, c.d), dtype=BF16, device=device)
        self.h = torch.empty((max_rows, c.d), dtype=BF16, device=device)
        self.qkv = torch.empty((max_rows, 3 * c.d), dtype=BF16, device=device)
        self.attn = torch.empty((max_rows, c.d), dtype=BF16, device=device)
        self.ff = torch.empty((max_rows, c.ffn), dtype=BF16, device=device)
        self.scale = 1.0 / math.sqrt(c.head_dim)
        self._aws: dict = {}

    def _attn_ws(self, B: int, Q: int, T: int):
        """Split-KV attention scratch, one per (B, Q, T) shape (allocated on the
        first, eager call — never inside a graph capture)."""
        key = (B, Q, T)
        if key not in self._aws:
            c = self.cfg
            self._aws[key] = K.AttnWorkspace(B, Q, c.n_heads, c.head_dim, T, self.device)
        return self._aws[key]

    def forward(self, tokens: torch.Tensor, start: torch.Tensor, slot: torch.Tensor, cache: KVCache,
                logits: torch.Tensor, head_rows: torch.Tensor | None = None, stream=None,
                prefill: bool = False) -> torch.Tensor:
        """Run Q positions for B requests.

        tokens [B, Q] int32: row b holds the tokens at positions start[b] .. start[b]+Q-1
        slot [B] int32: KV-cache slot of each request
        head_rows [R'] int32 or None: rows (of the B*Q) whose logits are computed
        logits [R', V] fp32 (out)
        """
        c, w = self.cfg, self.w
        B, Q = tokens.shape
        R = B * Q
        if R > self.max_rows:
            raise ValueError(f"{R} rows exceed max_rows={self.max_rows}")
        x, h, qkv, at, ff = self.x[:R], self.h[:R], self.qkv[:R], self.attn[:R], self.ff[:R]
        K.embed(tokens, start, Q, w["tok_emb"], w["pos_emb"], c.pos_offset, out=x, stream=stream)
        # split-KV attention is opt-in: measured slower at these context lengths
        aws = self._attn_ws(B, Q, cache.max_len) if self.split_kv else None
        small = self.small_gemm and R <= 64
        # prompt prefill (caller-chosen, never by row count): tcgen05 CTA-pair GEMMs
        wide = prefill

        def lin(xx, wname, bname, **kw):
            if wide:
                return K.linear_wide(xx, w[wname], w[bname], stream=stream, **kw)
            # ms_gemv only where it measured faster (tools/probe_gemm_graph.py):
            # short K; long-K projections (FC2) keep the cluster split-K path
            if small and xx.shape[1] <= K.GEMV_MAX_K:
                return K.gemv(xx, w[wname], w[bname], stream=stream, **kw)
            return K.linear(xx, w[wname], w[bname], stream=stream, **kw)

        for i in range(c.n_layers):
            p = f"l{i}."
            K.layernorm(x, w[p + "ln1_g"], w[p + "ln1_b"], c.eps, out=h, stream=stream)
            lin(h, p + "w_qkv", p + "b_qkv", out=qkv)
            K.attention(qkv, B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i],
                        self.scale, out=at, ws=aws, stream=stream, page=getattr(cache, "page", None),
                        prefill=prefill)
            lin(at, p + "w_o", p + "b_o", residual=x, out=x)
            K.layernorm(x, w[p + "ln2_g"], w[p + "ln2_b"], c.eps, out=h, stream=stream)
            lin(h, p + "w_fc1", p + "b_fc1", act=1, out=ff)
            lin(ff, p + "w_fc2", p + "b_fc2", residual=x, out=x)
        Rh = R if head_rows is None else head_rows.numel()
        hf = self.h[:Rh]
        K.layernorm(x, w["lnf_g"], w["lnf_b"], c.eps, out=hf, rows=head_rows, stream=stream)
        K.linear(hf, w["tok_emb"], out=logits, out_f32=True, stream=stream)
        return logits
