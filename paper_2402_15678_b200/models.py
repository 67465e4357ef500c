"""Model registry: the OPT (cfg1/cfg2) and Llama-2 (cfg3/cfg5, the headline
metric's Llama-2-70B + Llama-160M) families behind one forward interface, so
the speculation engine is model-family agnostic."""
from __future__ import annotations

from . import llama, opt

CONFIGS = {**opt.CONFIGS, **llama.CONFIGS}


def config(name: str):
    if name not in CONFIGS:
        raise KeyError(f"unknown model {name!r}; known: {sorted(CONFIGS)}")
    return CONFIGS[name]


def random_weights(cfg, seed: int, device="cuda", **kw):
    if cfg.family == "llama":
        return llama.LlamaWeights.random(cfg, seed, device=device, **kw)
    return opt.OPTWeights.random(cfg, seed, device=device, **kw)


def make_model(w, max_rows: int, device="cuda", small_gemm: bool = False, precision: str = "bf16"):
    """precision "bf16" (the product path) or "fp32" (the fp32 verification
    mode, fp32.py: fp32 activations / KV cache, parity with the fp32 oracles)."""
    if precision == "fp32":
        from .fp32 import LlamaModelF32, OPTModelF32
        return (LlamaModelF32 if w.cfg.family == "llama" else OPTModelF32)(w, max_rows=max_rows, device=device)
    if precision != "bf16":
        raise ValueError(f"precision must be 'bf16' or 'fp32', got {precision!r}")
    if w.cfg.family == "llama":
        return llama.LlamaModel(w, max_rows=max_rows, device=device, small_gemm=small_gemm)
    return opt.OPTModel(w, max_rows=max_rows, device=device, small_gemm=small_gemm)
