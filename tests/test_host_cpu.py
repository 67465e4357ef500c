"""Host-side logic of the product package against the reference-generated
golden traces (CPU only)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2402_15678_b200 import core, selector, voting


def test_selector_matches_reference_trace():
    with open(os.path.join(GOLDEN, "selector_trace.json")) as fh:
        traces = json.load(fh)
    for t in traces:
        cfg = core.EngineConfig(vocab_size=8, s_init=t["s_init"],
                                decision_threshold=t["decision_threshold"])
        st = selector.SelectorState.from_config(cfg)
        for r, (t_llm, vl, s_used, dec, s_next) in enumerate(t["events"]):
            selector.observe(st, selector.MonitorSample(r, t_llm, vl, s_used))
            _, d = selector.maybe_adjust(st)
            assert d.value == dec and st.current_s == s_next


def test_weights_match_reference_trace():
    with open(os.path.join(GOLDEN, "weights_trace.json")) as fh:
        traces = json.load(fh)
    for t in traces:
        K = t["K"]
        cfg = core.EngineConfig(vocab_size=8, initial_weights=tuple([1.0] * K))
        tab = voting.WeightTable.from_config(list(range(K)), cfg)
        for st in t["steps"]:
            for sid, rate in st["calls"]:
                voting.record_acr(tab, sid, rate)
            voting.update_weights(tab, cfg)
            assert [tab.weights[k] for k in range(K)] == st["weights"]


def test_merge_errors_and_packing():
    w = {0: 1.0, 1: 2.0}
    with pytest.raises(ValueError):
        voting.merge([], w)
    with pytest.raises(voting.LengthMismatch):
        voting.merge([(0, [])], w)
    with pytest.raises(voting.LengthMismatch):
        voting.merge([(0, [1, 2]), (1, [1])], w)
    with pytest.raises(voting.UnknownSSM):
        voting.merge([(7, [1])], w)
    tr = voting.merge([(1, [3, 4]), (0, [3, 5])], w)
    assert tr.tokens.tolist() == [[3, 4], [3, 5]] and tr.weights.tolist() == [2.0, 1.0]
    assert voting.drafter_ranks(tr.ids).tolist() == [1, 0]


def test_drafter_ranks_sorted_ids():
    ids = [42, 7, 99, 0]
    assert voting.drafter_ranks(ids).tolist() == [2, 1, 3, 0]


def test_validate_config_lists_all_violations():
    with pytest.raises(core.ConfigInvalid) as ei:
        core.validate_config(core.EngineConfig(vocab_size=0, b_llm=0, s_init=0))
    assert len(ei.value.violations) >= 3


def test_seeded_rng_matches_reference_stream():
    """verify_stoch.npz holds the uniforms the reference drew from
    seeded_rng(i, "verify/req-%03d"); our seeded_rng must reproduce them."""
    with np.load(os.path.join(GOLDEN, "verify_stoch.npz")) as z:
        us = z["V5_uniforms"]
    for i in range(50):
        want = [u for u in us[i] if u >= 0]
        rng = core.seeded_rng(i, f"verify/req-{i:03d}")
        assert [rng.random() for _ in want] == list(want)


def test_probdist_guards():
    with pytest.raises(ValueError):
        core.ProbDist([0.5, 0.6])
    d = core.ProbDist([0.0, 1.0])
    assert d.point_mass_token() == 1
    assert core.ProbDist([0.5, 0.5]).point_mass_token() is None


def test_llama_rope_table_and_gate_up_layout_match_reference():
    """Host-side Llama plumbing (no kernels): the RoPE table and the interleaved
    gate/up row map the device path uses equal the fp32 reference's."""
    import torch
    from oracle import llama_ref
    from paper_2402_15678_b200 import kernels as Kn
    from paper_2402_15678_b200.llama import CONFIGS, gate_up_rows
    assert torch.equal(Kn.rope_table(64, 128, 10000.0, device="cpu"), llama_ref.rope_table(64, 128, 10000.0))
    g, u = gate_up_rows(192)
    w = torch.arange(384).float()[:, None]
    wg, wu = llama_ref.split_gate_up(w, 192)
    assert torch.equal(wg[:, 0].long(), g) and torch.equal(wu[:, 0].long(), u)
    assert sorted(torch.cat([g, u]).tolist()) == list(range(384))
    c = CONFIGS["llama-2-70b"]
    assert c.matmul_params() == 68_713_185_280  # 68.71 G incl. LM head
    assert c.kv_bytes_per_token() == 327_680
    assert CONFIGS["llama-2-13b"].kv_bytes_per_token() == 819_200


def test_llama_reference_gqa_equals_mha_with_repeated_kv():
    """oracle/llama_ref: a GQA model equals the MHA model whose K/V projection
    rows are repeated per group (checks the reference's head mapping)."""
    import torch
    from oracle import llama_ref
    from paper_2402_15678_b200.llama import LlamaConfig, LlamaWeights
    gq = LlamaConfig("g", 1, 64, 4, 2, 128, vocab=50, max_pos=64)
    mh = LlamaConfig("m", 1, 64, 4, 4, 128, vocab=50, max_pos=64)
    w = LlamaWeights.random(gq, 0, device="cpu", std=0.1).t
    D = 16
    wq, wk, wv = w["l0.w_qkv"][:64], w["l0.w_qkv"][64:96], w["l0.w_qkv"][96:]
    rep = lambda m: m.view(2, D, 64).repeat_interleave(2, dim=0).reshape(64, 64)  # noqa: E731
    w2 = dict(w)
    w2["l0.w_qkv"] = torch.cat([wq, rep(wk), rep(wv)])
    toks = [3, 7, 1, 40, 2, 9]
    torch.testing.assert_close(llama_ref.forward(w, gq, toks), llama_ref.forward(w2, mh, toks))


def test_tp_shard_math_reproduces_full_layer():
    """The Megatron split of tp.shard_llama (column-parallel QKV / gate-up,
    row-parallel O / down, vocab-parallel head): summing the ranks' fp32
    partials reproduces the unsharded computation (CPU, fp32, no kernels)."""
    import math
    import torch
    from oracle import llama_ref
    from paper_2402_15678_b200.llama import LlamaConfig, LlamaWeights
    from paper_2402_15678_b200.tp import shard_llama
    c = LlamaConfig("t", 1, 64, 8, 4, 256, vocab=64, max_pos=32)
    w = LlamaWeights.random(c, 0, device="cpu", std=0.1)
    f = {k: v.float() for k, v in w.t.items()}
    T = 5
    x = torch.randn(T, c.d)
    table = llama_ref.rope_table(T, c.head_dim, c.rope_theta)
    pos = torch.arange(T)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool), 1)

    def attn(wqkv, H, Hkv):
        D = c.head_dim
        qkv = x @ wqkv.T
        q = llama_ref.rope(qkv[:, :H * D].view(T, H, D), pos, table)
        k = llama_ref.rope(qkv[:, H * D:(H + Hkv) * D].view(T, Hkv, D), pos, table).repeat_interleave(H // Hkv, 1)
        v = qkv[:, (H + Hkv) * D:].view(T, Hkv, D).repeat_interleave(H // Hkv, 1)
        s = (q.transpose(0, 1) @ k.transpose(0, 1).transpose(1, 2)) / math.sqrt(D)
        return (torch.softmax(s.masked_fill(mask, float("-inf")), -1) @ v.transpose(0, 1)).transpose(0, 1).reshape(T, -1)

    def mlp(wgu, wd, F):
        g, u = llama_ref.split_gate_up(wgu, F)
        a, b = x @ g.T, x @ u.T
        return (a / (1 + torch.exp(-a)) * b) @ wd.T

    want_o = attn(f["l0.w_qkv"], c.n_heads, c.n_kv_heads) @ f["l0.w_o"].T
    want_m = mlp(f["l0.w_gu"], f["l0.w_down"], c.ffn)
    for t in (2, 4):
        got_o = torch.zeros_like(want_o)
        got_m = torch.zeros_like(want_m)
        heads = []
        for r in range(t):
            s = {k: v.float() for k, v in shard_llama(w, r, t).t.items()}
            sc = shard_llama(w, r, t).cfg
            got_o += attn(s["l0.w_qkv"], sc.n_heads, sc.n_kv_heads) @ s["l0.w_o"].T
            got_m += mlp(s["l0.w_gu"], s["l0.w_down"], sc.ffn)
            heads.append(x @ s["lm_head"].T)
        torch.testing.assert_close(got_o, want_o, rtol=1e-4, atol=1e-5)
        torch.testing.assert_close(got_m, want_m, rtol=1e-4, atol=1e-5)
        torch.testing.assert_close(torch.cat(heads, 1), x @ f["lm_head"].T)


def test_trace_and_metrics_match_reference_golden(golden_dir):
    """trace.TraceEvent.to_json and collect_metrics reproduce the reference's
    (aggspec/engine.py:49-168) on a golden trace generated by running it."""
    import json
    import os
    from paper_2402_15678_b200.core import Request
    from paper_2402_15678_b200.trace import TraceEvent, collect_metrics
    g = json.load(open(os.path.join(golden_dir, "metrics_golden.json")))
    evs = []
    for e in g["events"]:
        ev = TraceEvent(e["seq"], e["kind"], e["start"], e["end"], e["s"], e["request_ids"], e["pool_depth"])
        if e["kind"] == "verify":
            ev.round_index, ev.accepted, ev.emitted, ev.voted = e["round"], e["accepted"], e["emitted"], e["voted"]
            ev.vl, ev.decision, ev.s_next = e["vl"], e["decision"], e["s_next"]
            ev.weights = {int(k): v for k, v in e["weights"].items()}
        assert json.loads(ev.to_json()) == e
        evs.append(ev)
    reqs = []
    for r in g["requests"]:
        q = Request(r["id"], [1], 20)
        q.generated = r["generated"]
        q.finish_time = r["finish_time"]
        reqs.append(q)
    m = collect_metrics(evs, reqs)
    for k, v in g["metrics"].items():
        assert getattr(m, k) == v, k
    assert {str(k): v for k, v in m.per_ssm_acceptance.items()} == g["per_ssm_acceptance"]
    assert [list(x) for x in m.s_trajectory] == g["s_trajectory"]


def test_block_manager_rollback_and_exhaustion():
    import pytest
    from paper_2402_15678_b200.paged import BlockManager, KVPoolExhausted
    m = BlockManager(n_blocks=6, slots=2, max_blocks=4, block_size=8)
    m.ensure(0, 17)                    # 3 blocks
    m.ensure(1, 8)                     # 1 block
    assert m.used() == 4 and int(m.table[0, 2]) != m.scratch
    assert m.truncate(0, 9) == 1       # positions >= 16 rejected: block 2 freed
    assert int(m.table[0, 2]) == m.scratch and m.used() == 3
    m.ensure(1, 32)                    # 3 more -> 6 used
    with pytest.raises(KVPoolExhausted):
        m.ensure(0, 25)
    assert m.release(1) == 4 and m.used() == 2
