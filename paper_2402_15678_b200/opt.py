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
import os
from dataclasses import dataclass

import torch

from . import kernels as K

BF16 = torch.bfloat16


@dataclass(frozen=True)
class OPTConfig:
    name: str
    n_layers: int
    d: int
    n_heads: int
    ffn: int
    vocab: int = 50272
    max_pos: int = 2048
    eps: float = 1e-5
    pos_offset: int = 2  # OPT's learned-position offset

    family = "opt"

    @property
    def head_dim(self) -> int:
        return self.d // self.n_heads

    @property
    def n_kv_heads(self) -> int:
        return self.n_heads

    def matmul_params(self) -> int:
        """Parameters streamed per forward (layers + tied LM head)."""
        per_layer = 3 * self.d * self.d + self.d * self.d + 2 * self.d * self.ffn
        return self.n_layers * per_layer + self.vocab * self.d

    def kv_bytes_per_token(self) -> int:
        return self.n_layers * 2 * self.d * 2


CONFIGS = {
    "opt-13b": OPTConfig("opt-13b", 40, 5120, 40, 20480),
    "opt-125m": OPTConfig("opt-125m", 12, 768, 12, 3072),
    # cfg1 of BASELINE.json: tiny OPT-style target and 1-layer drafters
    "tiny-target": OPTConfig("tiny-target", 4, 256, 4, 1024),
    "tiny-ssm": OPTConfig("tiny-ssm", 1, 256, 4, 1024),
}


class OPTWeights:
    """Random-init weights (normal(0, 0.02) for Linear/Embedding, zero bias,
    unit LayerNorm), generated with a seeded torch.Generator on `device`."""

    def __init__(self, cfg: OPTConfig, tensors: dict[str, torch.Tensor]):
        self.cfg = cfg
        self.t = tensors

    @classmethod
    def random(cls, cfg: OPTConfig, seed: int, device="cuda", std: float = 0.02,
               bias_std: float = 0.0) -> "OPTWeights":
        g = torch.Generator(device=device).manual_seed(seed)
        dev = torch.device(device)

        def normal(*shape, s=std):
            return (torch.randn(*shape, generator=g, device=dev, dtype=torch.float32) * s).to(BF16)

        def bias(n):
            return normal(n, s=bias_std) if bias_std > 0 else torch.zeros(n, dtype=BF16, device=dev)

        d, f = cfg.d, cfg.ffn
        t = {"tok_emb": normal(cfg.vocab, d), "pos_emb": normal(cfg.max_pos + cfg.pos_offset, d),
             "lnf_g": torch.ones(d, dtype=BF16, device=dev), "lnf_b": torch.zeros(d, dtype=BF16, device=dev)}
        for i in range(cfg.n_layers):
            p = f"l{i}."
            t[p + "ln1_g"] = torch.ones(d, dtype=BF16, device=dev)
            t[p + "ln1_b"] = torch.zeros(d, dtype=BF16, device=dev)
            t[p + "w_qkv"] = normal(3 * d, d)
            t[p + "b_qkv"] = bias(3 * d)
            t[p + "w_o"] = normal(d, d)
            t[p + "b_o"] = bias(d)
            t[p + "ln2_g"] = torch.ones(d, dtype=BF16, device=dev)
            t[p + "ln2_b"] = torch.zeros(d, dtype=BF16, device=dev)
            t[p + "w_fc1"] = normal(f, d)
            t[p + "b_fc1"] = bias(f)
            t[p + "w_fc2"] = normal(d, f)
            t[p + "b_fc2"] = bias(d)
        return cls(cfg, t)

    def to(self, device) -> "OPTWeights":
        return OPTWeights(self.cfg, {k: v.to(device) for k, v in self.t.items()})

    def __getitem__(self, k: str) -> torch.Tensor:
        return self.t[k]


class KVCache:
    """Per-layer K/V caches [slots, Hkv, T, D] bf16 (Hkv = KV heads: the query
    heads for OPT, the grouped KV heads for Llama-2-70B)."""

    def __init__(self, cfg, slots: int, max_len: int, device="cuda"):
        shape = (slots, cfg.n_kv_heads, max_len, cfg.head_dim)
        self.k = [torch.zeros(shape, dtype=BF16, device=device) for _ in range(cfg.n_layers)]
        self.v = [torch.zeros(shape, dtype=BF16, device=device) for _ in range(cfg.n_layers)]
        self.slots, self.max_len = slots, max_len

    def nbytes(self) -> int:
        return sum(t.numel() * 2 for t in self.k + self.v)


class OPTModel:
    """Batched forward over the kernels with static activation buffers (so a
    forward of a given (B, Q) can be captured in a CUDA graph)."""

    # fuse LayerNorm into the QKV / FC1 GEMMs when rows x d is at most this
    # (every GEMM CTA re-reads the rows for their statistics).  Off by default:
    # measured slower on the OPT-125M decode chain (2.51 vs 2.17 ms per draft
    # round) — the statistics pass sits on the GEMM's critical path, so the
    # saved launch is paid back; MS_FUSE_LN=1 enables it.
    FUSE_LN_ELEMS = 131072 if os.environ.get("MS_FUSE_LN", "0") == "1" else 0
    SPLIT_KV = os.environ.get("MS_SPLITKV", "0") == "1"

    def __init__(self, w: OPTWeights, max_rows: int, device="cuda", small_gemm: bool = False):
        """small_gemm: layer GEMMs of <= 64 token rows use the low-latency
        ms_gemv (drafters' decode steps); the verifier keeps the tcgen05 path
        everywhere, so its numerics never depend on the row count."""
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
        # GEMM schedule: cluster split-K (measured faster than the persistent
        # stream-K path, whose tile fix-up is a serial tail — tools/probe_gemm_graph.py);
        # MS_STREAM_K=1 selects stream-K (scratch is per model = per stream)
        self.ws = None
        if os.environ.get("MS_STREAM_K", "0") == "1":
            self.ws = K.Workspace(self.device)
            for n, k in ((3 * c.d, c.d), (c.d, c.d), (c.ffn, c.d), (c.d, c.ffn), (c.vocab, c.d)):
                self.ws.fit(min(max_rows, 256), n, k)

    def _attn_ws(self, B: int, Q: int, T: int):
        """Split-KV attention scratch, one per (B, Q, T) shape (allocated on the
        first, eager call — never inside a graph capture)."""
        key = (B, Q, T)
        if key not in self._aws:
            c = self.cfg
            self._aws[key] = K.AttnWorkspace(B, Q, c.n_heads, c.head_dim, T, self.device)
        return self._aws[key]

    def forward(self, tokens: torch.Tensor, start: torch.Tensor, slot: torch.Tensor, cache: KVCache,
                logits: torch.Tensor, head_rows: torch.Tensor | None = None, stream=None) -> torch.Tensor:
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
        ws = self.ws
        K.embed(tokens, start, Q, w["tok_emb"], w["pos_emb"], c.pos_offset, out=x, stream=stream)
        # split-KV attention is opt-in: measured slower at these context lengths
        aws = self._attn_ws(B, Q, cache.max_len) if self.SPLIT_KV else None
        # small (decode-sized) activations: LayerNorm fused into the next GEMM
        fuse_ln = R * c.d <= self.FUSE_LN_ELEMS
        small = self.small_gemm and R <= 64

        def lin(xx, wname, bname, **kw):
            # ms_gemv only where it measured faster (tools/probe_gemm_graph.py):
            # short K; long-K projections (FC2) keep the cluster split-K path
            if small and xx.shape[1] <= 1024:
                return K.gemv(xx, w[wname], w[bname], stream=stream, **kw)
            return K.linear(xx, w[wname], w[bname], ws=ws, stream=stream, **kw)

        for i in range(c.n_layers):
            p = f"l{i}."
            if fuse_ln and not small:
                K.linear_ln(x, w[p + "ln1_g"], w[p + "ln1_b"], w[p + "w_qkv"], w[p + "b_qkv"], c.eps,
                            out=qkv, stream=stream)
            else:
                K.layernorm(x, w[p + "ln1_g"], w[p + "ln1_b"], c.eps, out=h, stream=stream)
                lin(h, p + "w_qkv", p + "b_qkv", out=qkv)
            K.attention(qkv, B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i],
                        self.scale, out=at, ws=aws, stream=stream, page=getattr(cache, "page", None))
            lin(at, p + "w_o", p + "b_o", residual=x, out=x)
            if fuse_ln and not small:
                K.linear_ln(x, w[p + "ln2_g"], w[p + "ln2_b"], w[p + "w_fc1"], w[p + "b_fc1"], c.eps,
                            act=1, out=ff, stream=stream)
            else:
                K.layernorm(x, w[p + "ln2_g"], w[p + "ln2_b"], c.eps, out=h, stream=stream)
                lin(h, p + "w_fc1", p + "b_fc1", act=1, out=ff)
            lin(ff, p + "w_fc2", p + "b_fc2", residual=x, out=x)
        Rh = R if head_rows is None else head_rows.numel()
        hf = self.h[:Rh]
        K.layernorm(x, w["lnf_g"], w["lnf_b"], c.eps, out=hf, rows=head_rows, stream=stream)
        K.linear(hf, w["tok_emb"], out=logits, out_f32=True, ws=ws, stream=stream)
        return logits
