"""End-to-end speculation rounds on the GPU (cfg1 shape: tiny OPT-style target
4L d=256 + 3 x 1L drafters, B=4, s=4, greedy, 64 new tokens).

* lossless: the speculative output equals plain greedy decoding of the target
  (exactly — the forward is batch-invariant) and agrees with the fp32 CPU
  reference model's greedy decode;
* every round's integer decisions (vote path / voted drafter, accepted count,
  emitted tokens, weight updates, selector moves) replayed through the CPU
  oracle restatement of the reference (oracle/aggspec_oracle.py) match.
"""
import numpy as np
import pytest
import torch

from oracle import aggspec_oracle as O
from oracle import opt_ref

pytestmark = pytest.mark.gpu


def _setup(fidelity=None, s_init=4, adaptive=True, n_new=64, B=4, seed=0, stop=None, graphs=True,
           decision_threshold=8):
    from paper_2402_15678_b200.core import EngineConfig, Request
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.opt import CONFIGS, OPTWeights
    tcfg, scfg = CONFIGS["tiny-target"], CONFIGS["tiny-ssm"]
    target = OPTWeights.random(tcfg, 0, device="cpu", std=0.05, bias_std=0.02)
    drafters = [OPTWeights.random(scfg, k + 1, device="cpu", std=0.05, bias_std=0.02) for k in range(3)]
    cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=B, b_ssm=B, s_init=s_init,
                       initial_weights=(1.0, 1.0, 1.0), stop_token=stop,
                       decision_threshold=decision_threshold)
    eng = SpecEngine(target.to("cuda"), [d.to("cuda") for d in drafters], cfg, slots=B, max_len=160,
                     fidelity=fidelity, adaptive=adaptive, record=True, use_graphs=graphs)
    rng = np.random.default_rng(seed)
    reqs = [Request(f"req-{i:03d}", [int(t) for t in rng.integers(0, tcfg.vocab, size=int(rng.integers(4, 9)))],
                    n_new) for i in range(B)]
    return eng, reqs, target, tcfg


def _fresh(reqs):
    from paper_2402_15678_b200.core import Request
    return [Request(r.id, list(r.prompt), r.max_new_tokens) for r in reqs]


@pytest.mark.parametrize("graphs", [False, True])
def test_speculative_equals_greedy(graphs):
    eng, reqs, target, tcfg = _setup(graphs=graphs)
    teacher = eng.greedy_teacher(_fresh(reqs), 64)
    res = eng.run(reqs)
    assert res.outputs == teacher
    # agreement with the fp32 CPU reference's greedy decode
    agree = tot = 0
    for r in reqs[:2]:
        ref = opt_ref.greedy_generate(target.t, tcfg, r.prompt, 24)
        got = res.outputs[r.id][:24]
        n = next((i for i in range(24) if ref[i] != got[i]), 24)
        agree += n
        tot += 24
    assert agree / tot >= 0.5, (agree, tot)


def test_full_fidelity_accepts_everything():
    eng, reqs, *_ = _setup(fidelity=[1.0, 1.0, 1.0], adaptive=False)
    teacher = eng.greedy_teacher(_fresh(reqs), 64)
    eng.prefill(reqs)
    eng.set_teacher(teacher)
    res = eng.decode()
    assert res.outputs == teacher
    full = [a for r in res.rounds for a in r.accepted]
    assert np.mean(full) > 3.5  # s = 4, truncation only in the last round
    assert sum(len(v) for v in res.outputs.values()) == 4 * 64


def test_partial_fidelity_lossless_and_rounds_match_oracle():
    eng, reqs, *_ = _setup(fidelity=[0.9, 0.7, 0.5], decision_threshold=3)
    teacher = eng.greedy_teacher(_fresh(reqs), 64)
    eng.prefill(reqs)
    eng.set_teacher(teacher)
    res = eng.decode()
    assert res.outputs == teacher
    w = {0: 1.0, 1: 1.0, 2: 1.0}
    sel = O.SelectorOracle(s_init=4, decision_threshold=3)
    for st in res.rounds:
        tr = st.trace
        s = st.s
        assert s == sel.s
        log = {0: [], 1: [], 2: []}
        vl_counts = []
        assert tr["weights_used"].tolist() == [w[k] for k in range(3)]
        for b in tr["active"]:
            path, voted = O.vote_one(tr["drafts"][b], tr["weights_used"])
            assert path == tr["path"][b].tolist() and voted == tr["voted"][b]
            acc, em, _ = O.verify_greedy_one(path, tr["tgt"][b])
            use, _ = O.commit_one(em, int(tr["remaining"][b]), None)
            assert acc == tr["n_acc"][b] and use == tr["emitted"][b, : tr["n_emit"][b]].tolist()
            log[voted].append(acc / s)
            vl_counts.append(len(use))
        w = O.update_weights(w, log)
        assert [w[k] for k in range(3)] == [st.weights[k] for k in range(3)]
        sel.observe(st.t_verify_ms, float(np.mean(vl_counts)), s)
        assert sel.maybe_adjust() == st.decision
        assert sel.s == st.s_next
    assert len({st.s for st in res.rounds}) >= 1


def test_stop_token_and_budget():
    eng, reqs, *_ = _setup(n_new=20)
    teacher = eng.greedy_teacher(_fresh(reqs), 20)
    stop = teacher[reqs[0].id][7]
    eng2, reqs2, *_ = _setup(n_new=20, stop=stop)
    res = eng2.run(reqs2)
    for r in reqs2:
        t = teacher[r.id]
        want = t[: t.index(stop) + 1] if stop in t else t
        assert res.outputs[r.id] == want


@pytest.mark.parametrize("fidelity", [None, [0.9, 0.8, 0.6]])
def test_pipelined_schedule_is_lossless_and_alternates(fidelity):
    """Pipelined mode (two request groups: the verifier works on one while the
    drafters draft the other, aggspec/engine.py:494-576) produces the same
    token streams as plain greedy decoding — the reference's sequential ==
    pipelined token-stream equivalence (tests/test_engine.py:106-133)."""
    from paper_2402_15678_b200.core import EngineConfig, Request
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.opt import CONFIGS, OPTWeights
    tcfg, scfg = CONFIGS["tiny-target"], CONFIGS["tiny-ssm"]
    target = OPTWeights.random(tcfg, 0, device="cuda", std=0.05, bias_std=0.02)
    drafters = [OPTWeights.random(scfg, k + 1, device="cuda", std=0.05, bias_std=0.02) for k in range(3)]
    cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=4, b_ssm=4, initial_weights=(1.0, 1.0, 1.0),
                       decision_threshold=3)
    eng = SpecEngine(target, drafters, cfg, slots=8, max_len=120, pipelined=True, fidelity=fidelity)
    rng = np.random.default_rng(5)
    reqs = [Request(f"req-{i:03d}", [int(t) for t in rng.integers(0, tcfg.vocab, size=int(rng.integers(4, 9)))],
                    int(rng.integers(20, 48))) for i in range(7)]
    teacher = eng.greedy_teacher([Request(r.id, list(r.prompt), r.max_new_tokens) for r in reqs], 48)
    eng.prefill(reqs)
    if fidelity:
        eng.set_teacher(teacher)
    res = eng.decode()
    for r in reqs:
        assert res.outputs[r.id] == teacher[r.id][: r.max_new_tokens]
    groups = [rd.group for rd in res.rounds]
    assert groups[:6] == [0, 1, 0, 1, 0, 1]
    if fidelity:
        assert res.mean_accepted > 1.0
