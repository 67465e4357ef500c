"""Model-forward numerics with the tolerances written down (north_star: logits
within 1e-3 relative, token-agreement rate stated).

The measured numbers for every model shape (cfg1 / cfg2 / cfg3 drafters and
two-layer slices of the 70B / 13B verifiers) are in
profiles/r2_bf16_numerics.jsonl (tools/bf16_numerics.py).  bf16 cannot meet
1e-3: its unit roundoff is 2^-9 = 1.95e-3, and the bf16 contract rounds the
activations ~7 times per layer; measured 0.5-1.8 % of the max logit with
97-98.5 % argmax agreement on random-init weights (whose top-2 logit gaps are
tiny).  The fp32 verification mode meets it with >= 80x margin (<= 1.3e-5).
"""
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.mark.parametrize("name", ["tiny-target", "tiny-llama", "llama-160m"])
def test_logit_error_bounds(name):
    import bf16_numerics as N
    cfg = N.SHAPES[name]
    w = N.weights(cfg)
    P, Q = 64, 5
    toks = [int(x) for x in np.random.default_rng(1).integers(0, cfg.vocab, size=P + Q)]
    wd = w.to("cuda")
    exact = N.ref_logits(w.t, cfg, toks, exact=True)
    bf, _ = N.device_logits(wd, cfg, toks, P, Q, "bf16")
    r = N.compare(bf, exact)
    assert r["max_rel"] < 1.5e-2 and r["argmax_agree"] >= 0.95, r
    f32, _ = N.device_logits(wd, cfg, toks, P, Q, "fp32")
    r = N.compare(f32, exact)
    assert r["max_rel"] < 1e-4 and r["argmax_agree"] == 1.0, r  # the 1e-3 target, with margin
