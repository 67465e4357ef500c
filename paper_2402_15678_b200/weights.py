"""Model definitions without the kernels: the OPT and Llama-2 configurations,
seeded random-init weights and the KV-cache layout.  Torch-only (no
libminions import), so the CPU reference arm of bench.py and the golden
generators can build the exact same weights without loading the sm_100a
library.  opt.py / llama.py re-export these names.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

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


OPT_CONFIGS = {
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
    """Per-layer K/V caches [slots, Hkv, T, D] (Hkv = KV heads: the query
    heads for OPT, the grouped KV heads for Llama-2-70B); bf16, or fp32 for
    the fp32 verification mode."""

    def __init__(self, cfg, slots: int, max_len: int, device="cuda", dtype=BF16):
        shape = (slots, cfg.n_kv_heads, max_len, cfg.head_dim)
        self.k = [torch.zeros(shape, dtype=dtype, device=device) for _ in range(cfg.n_layers)]
        self.v = [torch.zeros(shape, dtype=dtype, device=device) for _ in range(cfg.n_layers)]
        self.slots, self.max_len, self.dtype = slots, max_len, dtype

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.k + self.v)


@dataclass(frozen=True)
class LlamaConfig:
    name: str
    n_layers: int
    d: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int = 32000
    max_pos: int = 8192  # RoPE table length (cfg5: 4K prompts + generation exceed Llama-2's 4096)
    eps: float = 1e-5
    rope_theta: float = 10000.0
    hd: int = 0  # head dim when it is not d / n_heads (a tensor-parallel shard)

    family = "llama"

    @property
    def head_dim(self) -> int:
        return self.hd or self.d // self.n_heads

    @property
    def qkv_out(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def matmul_params(self) -> int:
        """Parameters streamed per forward (layers + LM head)."""
        per_layer = self.d * self.qkv_out + self.d * self.n_heads * self.head_dim + 3 * self.d * self.ffn
        return self.n_layers * per_layer + self.vocab * self.d

    def kv_bytes_per_token(self) -> int:
        return self.n_layers * 2 * self.n_kv_heads * self.head_dim * 2


LLAMA_CONFIGS = {
    "llama-2-70b": LlamaConfig("llama-2-70b", 80, 8192, 64, 8, 28672),
    "llama-2-13b": LlamaConfig("llama-2-13b", 40, 5120, 40, 40, 13824),
    # max_pos = RoPE table length: 8192 so the drafters cover cfg5's 4K prompts
    # (the released Llama-160M was trained at 2048; rotary positions extend)
    "llama-160m": LlamaConfig("llama-160m", 12, 768, 12, 12, 3072, max_pos=8192, eps=1e-6),
    # test-sized Llama shapes (GQA 2:1, D = 64)
    "tiny-llama": LlamaConfig("tiny-llama", 4, 256, 4, 2, 512, max_pos=1024),
    "tiny-llama-ssm": LlamaConfig("tiny-llama-ssm", 1, 256, 4, 4, 512, max_pos=1024),
    # tensor-parallel test shape: splits over 2, 4 and 8 ranks (GQA 2:1, D = 64)
    "tiny-llama-tp": LlamaConfig("tiny-llama-tp", 2, 1024, 16, 8, 4096, max_pos=1024),
}


def gate_up_rows(ffn: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Row indices of the gate and up projections inside the interleaved w_gu."""
    j = torch.arange(ffn)
    gate = (j // 64) * 128 + j % 64
    return gate, gate + 64


class LlamaWeights:
    """Random-init weights (normal(0, 0.02) for Linear/Embedding — the HF
    initializer_range —, unit RMSNorm gains), seeded torch.Generator on `device`."""

    def __init__(self, cfg: LlamaConfig, tensors: dict[str, torch.Tensor]):
        self.cfg = cfg
        self.t = tensors

    @classmethod
    def random(cls, cfg: LlamaConfig, seed: int, device="cuda", std: float = 0.02,
               norm_std: float = 0.0) -> "LlamaWeights":
        if cfg.ffn % 64:
            raise ValueError("ffn must be a multiple of 64 (interleaved gate/up blocks)")
        g = torch.Generator(device=device).manual_seed(seed)
        dev = torch.device(device)

        def normal(*shape, s=std):
            out = torch.empty(*shape, dtype=BF16, device=dev)
            rows = max(1, (1 << 27) // max(1, shape[-1]))  # <= 512 MB fp32 temporaries
            flat = out.view(-1, shape[-1])
            for r0 in range(0, flat.shape[0], rows):
                n = min(rows, flat.shape[0] - r0)
                flat[r0: r0 + n] = (torch.randn(n, shape[-1], generator=g, device=dev) * s).to(BF16)
            return out

        def gain(n):
            if norm_std > 0:
                return (1.0 + torch.randn(n, generator=g, device=dev) * norm_std).to(BF16)
            return torch.ones(n, dtype=BF16, device=dev)

        d, f = cfg.d, cfg.ffn
        t = {"tok_emb": normal(cfg.vocab, d), "norm_f": gain(d), "lm_head": normal(cfg.vocab, d)}
        for i in range(cfg.n_layers):
            p = f"l{i}."
            t[p + "attn_norm"] = gain(d)
            t[p + "w_qkv"] = normal(cfg.qkv_out, d)
            t[p + "w_o"] = normal(d, cfg.n_heads * cfg.head_dim)
            t[p + "mlp_norm"] = gain(d)
            t[p + "w_gu"] = normal(2 * f, d)
            t[p + "w_down"] = normal(d, f)
        return cls(cfg, t)

    def to(self, device) -> "LlamaWeights":
        return LlamaWeights(self.cfg, {k: v.to(device) for k, v in self.t.items()})

    def fold_norms(self) -> "LlamaWeights":
        """Fold every RMSNorm gain into the projection that consumes it, in
        place: w_qkv[:, k] *= attn_norm[k], w_gu[:, k] *= mlp_norm[k],
        lm_head[:, k] *= norm_f[k] (one bf16 rounding), gains := 1.  Exact
        no-op on values for unit gains (random init)."""
        if getattr(self, "folded", False):
            return self
        c, t = self.cfg, self.t
        pairs = [(f"l{i}.attn_norm", f"l{i}.w_qkv") for i in range(c.n_layers)]
        pairs += [(f"l{i}.mlp_norm", f"l{i}.w_gu") for i in range(c.n_layers)] + [("norm_f", "lm_head")]
        for g, w in pairs:
            if not bool(torch.all(t[g] == 1)):
                t[w].mul_(t[g].to(t[w].dtype)[None, :])
            t[g] = torch.ones_like(t[g])  # a new tensor: shared gains elsewhere are untouched
        self.folded = True
        return self

    def __getitem__(self, k: str) -> torch.Tensor:
        return self.t[k]


CONFIGS = {**OPT_CONFIGS, **LLAMA_CONFIGS}
