"""The ModelOracle plug-in boundary on the GPU model (oracles.OPTOracle)."""
import numpy as np
import pytest

from oracle import opt_ref

pytestmark = pytest.mark.gpu


def _oracle(seed=0):
    from paper_2402_15678_b200.opt import CONFIGS, OPTWeights
    from paper_2402_15678_b200.oracles import OPTOracle
    cfg = CONFIGS["tiny-target"]
    w = OPTWeights.random(cfg, seed, device="cpu", std=0.05, bias_std=0.02)
    return OPTOracle(w.to("cuda"), context_cap=256), w, cfg


def test_protocol_and_prefix_cache_consistency():
    from paper_2402_15678_b200.oracles import ModelOracle
    o, w, cfg = _oracle()
    assert isinstance(o, ModelOracle)
    rng = np.random.default_rng(0)
    base = [int(t) for t in rng.integers(0, cfg.vocab, size=20)]
    fresh = _oracle()[0]
    # extend, branch, shrink: the cached path must equal a fresh computation
    for ctx in (base, base + [5], base + [5, 9], base[:10], base[:10] + [7, 7, 7], base):
        a = o.argmax_next(ctx)
        f2 = _oracle()[0]
        assert a == f2.argmax_next(ctx)
    d = o.next_dist(base)
    assert d.point_mass_token() == fresh.argmax_next(base)


def test_draft_sequence_is_greedy_and_consumes_one_uniform_per_step():
    from paper_2402_15678_b200.core import seeded_rng
    from paper_2402_15678_b200.oracles import draft_sequence
    o, w, cfg = _oracle(1)
    ctx = list(range(3, 15))
    rng = seeded_rng(0, "draft/req-000/0")
    toks, dists = draft_sequence(o, ctx, 5, rng)
    ref = seeded_rng(0, "draft/req-000/0")
    ref.random(5)
    assert rng.random() == ref.random()
    assert [d.point_mass_token() for d in dists] == toks
    want = opt_ref.greedy_generate(w.t, cfg, ctx, 5)
    agree = sum(int(a == b) for a, b in zip(toks, want))
    assert agree >= 4


def test_context_errors():
    from paper_2402_15678_b200.core import ContextTooLong
    o, *_ = _oracle()
    with pytest.raises(ValueError):
        o.next_dist([])
    with pytest.raises(ContextTooLong):
        o.next_dist(list(range(300)))


def test_llama_oracle_greedy_matches_reference():
    """GPUOracle over Llama-2-family weights (the headline model family) drives
    the reference's per-position protocol; greedy drafts agree with the fp32
    CPU Llama reference."""
    from oracle import llama_ref
    from paper_2402_15678_b200.core import seeded_rng
    from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights
    from paper_2402_15678_b200.oracles import GPUOracle, ModelOracle, draft_sequence
    cfg = CONFIGS["tiny-llama"]
    w = LlamaWeights.random(cfg, 2, device="cpu", std=0.05, norm_std=0.1)
    o = GPUOracle(w.to("cuda"), context_cap=256)
    assert isinstance(o, ModelOracle)
    ctx = list(range(7, 20))
    toks, _ = draft_sequence(o, ctx, 6, seeded_rng(0, "draft/req-000/0"))
    want = llama_ref.greedy_generate(w.t, cfg, ctx, 6)
    assert sum(int(a == b) for a, b in zip(toks, want)) >= 5
