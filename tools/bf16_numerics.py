"""bf16 numerics report (north_star: "logits within 1e-3 relative in bf16 with
the token-agreement rate stated"; VERDICT r1 "next round" #1).

For each model shape, random init (normal(0, 0.02), the bench's init), a
prompt of P tokens is prefilled and then a verify-shaped call of Q = 5 rows
runs at context P (the speculate-vote-verify path's forward).  The device's
logits of every row are compared with three fp32 CPU references over the same
bf16 weights:

  exact     oracle/*_ref.forward(exact=True): fp32 everywhere, no rounding —
            the precision loss of the bf16 product path;
  contract  the bf16 contract (one bf16 rounding per op, as the device) —
            the implementation error alone (summation order);
  fp32dev   the device's fp32 verification mode vs `exact`.

Reported per model: max relative logit error = max|l_dev - l_ref| / max|l_ref|
over all rows, the median per-row relative error, and the argmax agreement
rate (device argmax == reference argmax) over all rows.  Output: one JSON
object per line (default profiles/r2_bf16_numerics.jsonl).

    python tools/bf16_numerics.py [--out profiles/r2_bf16_numerics.jsonl] [--big]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import llama_ref, opt_ref  # noqa: E402
from paper_2402_15678_b200.models import make_model  # noqa: E402
from paper_2402_15678_b200.weights import CONFIGS, KVCache, LlamaConfig, LlamaWeights, OPTWeights  # noqa: E402

SHAPES = {
    "tiny-target": CONFIGS["tiny-target"],            # cfg1 target (OPT)
    "opt-125m": CONFIGS["opt-125m"],                  # cfg2 drafter
    "tiny-llama": CONFIGS["tiny-llama"],
    "llama-160m": CONFIGS["llama-160m"],              # cfg3 drafter
}
BIG = {
    # two-layer slices of the verifiers (full width, heads, FFN, vocabulary)
    "llama-2-70b[2L]": LlamaConfig("llama-2-70b-2l", 2, 8192, 64, 8, 28672),
    "llama-2-13b[2L]": LlamaConfig("llama-2-13b-2l", 2, 5120, 40, 40, 13824),
}


def weights(cfg, seed=0):
    if cfg.family == "llama":
        return LlamaWeights.random(cfg, seed, device="cpu")
    return OPTWeights.random(cfg, seed, device="cpu")


def ref_logits(w, cfg, toks, exact, fused_norm=False):
    if cfg.family == "llama":
        return llama_ref.forward(w, cfg, toks, fused_norm=fused_norm, exact=exact)
    return opt_ref.forward(w, cfg, toks, exact=exact)


def device_logits(wd, cfg, toks, P, Q, precision, small_gemm=False):
    """Prefill positions 0..P-1, then one verify-shaped call of Q rows at P."""
    model = make_model(wd, max_rows=max(P, Q) + 8, precision=precision, small_gemm=small_gemm)
    cache = KVCache(cfg, 1, P + Q + 8, "cuda", dtype=torch.float32 if precision == "fp32" else torch.bfloat16)
    slot = torch.zeros(1, dtype=torch.int32, device="cuda")
    t = torch.tensor([toks], dtype=torch.int32, device="cuda")
    lp = torch.empty(P, cfg.vocab, device="cuda")
    model.forward(t[:, :P].contiguous(), torch.zeros(1, dtype=torch.int32, device="cuda"), slot, cache, lp)
    lq = torch.empty(Q, cfg.vocab, device="cuda")
    model.forward(t[:, P:P + Q].contiguous(), torch.full((1,), P, dtype=torch.int32, device="cuda"), slot, cache, lq)
    torch.cuda.synchronize()
    return torch.cat([lp, lq]).cpu(), model


def compare(got, ref):
    scale = ref.abs().max().item()
    d = (got - ref).abs()
    row = (d.max(-1).values / ref.abs().max(-1).values).numpy()
    return dict(max_rel=round(d.max().item() / scale, 7), median_row_rel=round(float(np.median(row)), 7),
                argmax_agree=round(float((got.argmax(-1) == ref.argmax(-1)).float().mean()), 5),
                rows=int(ref.shape[0]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_bf16_numerics.jsonl"))
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--big", action="store_true", help="also the 70B / 13B two-layer slices")
    a = ap.parse_args()
    torch.set_num_threads(os.cpu_count() or 1)
    shapes = dict(SHAPES, **(BIG if a.big else {}))
    P, Q = a.prompt, 5
    lines = []
    for name, cfg in shapes.items():
        t0 = time.time()
        w = weights(cfg)
        toks = [int(x) for x in np.random.default_rng(1).integers(0, cfg.vocab, size=P + Q)]
        wd = w.to("cuda")
        rec = dict(model=name, family=cfg.family, layers=cfg.n_layers, d=cfg.d, vocab=cfg.vocab, prompt=P, verify_q=Q)
        bf, model = device_logits(wd, cfg, toks, P, Q, "bf16")
        fused = bool(getattr(model, "fuse_norm", False))
        rec["fused_norm"] = fused
        exact = ref_logits(w.t, cfg, toks, exact=True)
        contract = ref_logits(w.t, cfg, toks, exact=False, fused_norm=fused)
        rec["bf16_vs_exact"] = compare(bf, exact)
        rec["bf16_vs_contract"] = compare(bf, contract)
        rec["verify_rows_bf16_vs_exact"] = compare(bf[P:], exact[P:])
        f32, _ = device_logits(wd, cfg, toks, P, Q, "fp32")
        rec["fp32dev_vs_exact"] = compare(f32, exact)
        rec["secs"] = round(time.time() - t0, 1)
        print(json.dumps(rec), flush=True)
        lines.append(rec)
        del wd, model
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        for r in lines:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
