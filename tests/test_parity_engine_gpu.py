"""Engine-level parity with the REFERENCE engine (VERDICT r1 "next round" #1, #2).

tests/golden/engine_streams.json holds what the unmodified reference engine
(aggspec run_sequential / run_pipelined, aggspec/engine.py:619-671) produced
on cfg1 when driven by fp32 CPU transformer oracles over the same weights
(tests/golden/make_engine_golden.py), greedy (point-mass oracles) and
stochastic (softmax oracles: sampled drafts, speculative-sampling verify with
the reference's per-request PCG64 streams — SpecEngine(sampling=True)).  SpecEngine(precision="fp32") — the
fp32 verification mode (csrc/fp32.cu) — must reproduce it exactly:

  * every request's generated token stream,
  * every drafter's s draft tokens in every round (the reference recomputes
    each draft from the full context, aggspec/oracles.py:135-153; the device
    keeps per-drafter KV caches rolled back to lcp(draft, emitted) and
    caught up, engine.py _finish_verify / _upload — so this pins the rollback),
  * every verify round's request batch, s, accepted counts, emitted counts,
    voted drafter, selector decision, next s and the fp64 drafter weights.

The selector is fed the reference CostModel's t_llm (sim_cost), as the
reference's simulated clock does, so the s trajectory is reproducible.

The bf16 product path is pinned separately: with no fidelity injection each
drafter's per-round draft must equal that drafter's own greedy continuation
of the current context recomputed from scratch on the device (fresh cache,
same kernels), over >= 20 adaptive rounds.
"""
import json
import os
import re

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "engine_streams.json")


class _Cost:
    """t_llm of the reference CostModel (aggspec/oracles.py:157-183)."""

    def __init__(self, d0, d1, d2, **_):
        self.d0, self.d1, self.d2 = d0, d1, d2

    def t_llm(self, b, s):
        return self.d0 + self.d1 * b + self.d2 * b * s


def _models(kind):
    from paper_2402_15678_b200.weights import CONFIGS, OPTWeights
    tc, sc = CONFIGS["tiny-target"], CONFIGS["tiny-ssm"]
    target = OPTWeights.random(tc, 0, device="cpu")
    if kind == "random":
        drafters = [OPTWeights.random(sc, k + 1, device="cpu") for k in range(3)]
    else:  # layerskip: drafter k = target embeddings + target layer k
        drafters = []
        for k in range(3):
            t = {n: v.clone() for n, v in target.t.items() if not re.match(r"l\d+\.", n)}
            for n, v in target.t.items():
                if n.startswith(f"l{k}."):
                    t["l0." + n.split(".", 1)[1]] = v.clone()
            drafters.append(OPTWeights(sc, t))
    return target.to("cuda"), [d.to("cuda") for d in drafters]


def _scenarios():
    with open(GOLDEN) as f:
        return json.load(f)["scenarios"]


_IDS = ["random-seq", "random-pipe", "layerskip-seq", "layerskip-pipe"]


@pytest.mark.parametrize("idx", range(8), ids=[f"{m}-{i}" for m in ("greedy", "sample") for i in _IDS])
def test_fp32_engine_reproduces_reference_engine(idx):
    from paper_2402_15678_b200.core import EngineConfig, Request
    from paper_2402_15678_b200.engine import SpecEngine
    sc = _scenarios()[idx]
    target, drafters = _models(sc["kind"])
    c = sc["cfg"]
    cfg = EngineConfig(vocab_size=target.cfg.vocab, b_llm=c["b_llm"], b_ssm=c["b_ssm"], s_init=c["s_init"],
                       s_min=c["s_min"], s_max=c["s_max"], initial_weights=(1.0, 1.0, 1.0), seed=c["seed"])
    pipelined = sc["schedule"] == "pipelined"
    eng = SpecEngine(target, drafters, cfg, slots=4, max_len=96, precision="fp32", pipelined=pipelined,
                     record=True, adaptive=sc["adaptive"], sim_cost=_Cost(**sc["cost"]),
                     sampling=sc["mode"] == "sample")
    reqs = [Request(rid, list(p), 64) for rid, p in sc["prompts"].items()]
    res = eng.run(reqs)
    assert res.outputs == sc["outputs"]
    assert len(res.rounds) == len(sc["verify"])
    seen = {r.id: 0 for r in reqs}
    for rd, want in zip(res.rounds, sc["verify"]):
        got = dict(request_ids=list(rd.request_ids), s=rd.s, accepted=rd.accepted, emitted=rd.emitted,
                   voted=rd.voted, decision=rd.decision, s_next=rd.s_next,
                   weights={str(k): v for k, v in rd.weights.items()})
        exp = {k: want[k] for k in got}
        assert got == exp, f"round {want['round_index']}"
        t = rd.trace
        for j, b in enumerate(t["active"]):
            rid = rd.request_ids[j]
            gold = sc["drafts"][rid][seen[rid]]
            seen[rid] += 1
            assert t["drafts"][b].tolist() == gold, f"drafts of {rid} in round {want['round_index']}"
    assert all(seen[rid] == len(sc["drafts"][rid]) for rid in seen)


def _greedy_from_scratch(model, cfg, ctx, s, chunk=16):
    """Drafter's greedy continuation recomputed from nothing: a fresh KV cache,
    the context fed from position 0 in <= chunk-row forwards, then s one-row
    decode steps (every kernel's per-row result is independent of the row
    count on this path, so this equals what the engine computes for a row)."""
    from paper_2402_15678_b200 import _dev, _native
    from paper_2402_15678_b200.weights import KVCache
    cache = KVCache(cfg, 1, 128, "cuda")
    slot = torch.zeros(1, dtype=torch.int32, device="cuda")
    logits = torch.empty(1, cfg.vocab, device="cuda")
    am = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.zeros(1, dtype=torch.int64, device="cuda")
    seq = list(ctx)
    out = []
    p0 = 0
    while p0 < len(seq):
        n = min(chunk, len(seq) - p0)
        tok = torch.tensor([seq[p0: p0 + n]], dtype=torch.int32, device="cuda")
        st = torch.tensor([p0], dtype=torch.int32, device="cuda")
        model.forward(tok, st, slot, cache, logits, head_rows=torch.tensor([n - 1], dtype=torch.int32, device="cuda"))
        p0 += n
    for j in range(s):
        _native.call("ms_argmax_rows", logits.data_ptr(), 0, 1, cfg.vocab, cfg.vocab, am.data_ptr(), ws.data_ptr(),
                     _dev.stream_ptr())
        t = int(am.item())
        out.append(t)
        if j + 1 < s:
            tok = torch.tensor([[t]], dtype=torch.int32, device="cuda")
            st = torch.tensor([len(seq)], dtype=torch.int32, device="cuda")
            model.forward(tok, st, slot, cache, logits)
            seq.append(t)
    return out


@pytest.mark.parametrize("pipelined", [False, True])
def test_bf16_drafts_equal_own_greedy_continuation(pipelined):
    """bf16 product path, fidelity=None, adaptive s: each drafter's draft in
    every round == its greedy continuation of the round's context recomputed
    from scratch (VERDICT r1 weak #1 / ADVICE medium: KV rollback + catch-up)."""
    from paper_2402_15678_b200.core import EngineConfig, Request
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.models import make_model
    target, drafters = _models("layerskip")
    cfg = EngineConfig(vocab_size=target.cfg.vocab, b_llm=4, b_ssm=4, s_init=4, s_min=1, s_max=8,
                       initial_weights=(1.0, 1.0, 1.0), decision_threshold=3)
    eng = SpecEngine(target, drafters, cfg, slots=4, max_len=128, pipelined=pipelined, record=True,
                     sim_cost=_Cost(56.5, 0.75, 2.5))
    rng = np.random.default_rng(3)
    reqs = [Request(f"r{i}", [int(t) for t in rng.integers(0, target.cfg.vocab, size=int(rng.integers(4, 9)))], 48)
            for i in range(4)]
    ctx = {r.id: list(r.prompt) for r in reqs}
    res = eng.run(reqs)
    assert len(res.rounds) >= 20
    assert len({rd.s for rd in res.rounds}) >= 2, "the selector never moved s"
    fresh = [make_model(w, max_rows=64, small_gemm=True) for w in drafters]
    checked = lcp_pos = 0
    for rd in res.rounds:
        t = rd.trace
        for j, b in enumerate(t["active"]):
            rid = rd.request_ids[j]
            for k in range(3):
                want = _greedy_from_scratch(fresh[k], drafters[k].cfg, ctx[rid], rd.s)
                assert t["drafts"][b, k].tolist() == want, (rid, k, rd.round_index)
                checked += 1
            emitted = [int(x) for x in t["emitted"][b, : t["n_emit"][b]]]
            lcp_pos += int(any(t["drafts"][b, k, 0] == emitted[0] for k in range(3)))
            ctx[rid].extend(emitted)
    assert checked >= 3 * 20
    assert lcp_pos > 0, "no drafter ever matched: the rollback-to-lcp path was not exercised"
