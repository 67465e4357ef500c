"""Tensor-parallel verify on one GPU: t ranks of a TPComm local
group run concurrently (one host thread + CUDA stream per rank) and meet in the
peer-memory reduction kernels — the same kernels and flag protocol as one
process per GPU, with plain device pointers instead of IPC mappings.

Checked: every rank gets the same target argmax; it agrees with the
single-GPU model (the TP sum order differs, so logits agree within bf16
tolerance); the TP forward is deterministic and batch invariant (Q=1 decode
== Q=5 verify, bitwise) — what the lossless engine needs."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run_ranks(fns):
    """Run one callable per rank concurrently, each on its own stream."""
    errs = []
    streams = [torch.cuda.Stream() for _ in fns]

    def body(i):
        try:
            with torch.cuda.stream(streams[i]):
                fns[i]()
            streams[i].synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=body, args=(i,)) for i in range(len(fns))]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=120)
    assert not any(x.is_alive() for x in th), "rank thread hung"
    if errs:
        raise errs[0]


def _setup(t, B=4, T=64, seed=0, name="tiny-llama"):
    from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
    from paper_2402_15678_b200.opt import KVCache
    from paper_2402_15678_b200.tp import LlamaTPModel, TPComm, shard_llama
    cfg = CONFIGS[name]
    w = LlamaWeights.random(cfg, seed, device="cpu", std=0.05, norm_std=0.1)
    full = LlamaModel(w.to("cuda"), max_rows=B * T)
    comms = TPComm.local_group(t, B * T, cfg.d)
    shards = [shard_llama(w, r, t).to("cuda") for r in range(t)]
    models = [LlamaTPModel(shards[r], comms[r], max_rows=B * T) for r in range(t)]
    caches = [KVCache(shards[r].cfg, B, T) for r in range(t)]
    return cfg, full, KVCache(cfg, B, T), models, caches, comms


def _tp_step(models, caches, toks, start, slot):
    B, Q = toks.shape
    t = len(models)
    outs = [torch.zeros(B * Q, dtype=torch.int32, device="cuda") for _ in range(t)]
    logits = [torch.empty(B * Q, models[r].cfg.vocab, device="cuda") for r in range(t)]

    def fn(r):
        return lambda: models[r].argmax(models[r].forward(toks, start, slot, caches[r], logits[r]), outs[r])

    _run_ranks([fn(r) for r in range(t)])
    for m in models:
        m.comm.check()
    return outs, logits


# t <= 4: eight ranks' spin-waiting kernels sharing ONE GPU can starve each
# other of SM resources; with one rank per GPU (the product) that cannot happen.
@pytest.mark.parametrize("t,name", [(2, "tiny-llama"), (4, "tiny-llama-tp")])
def test_tp_forward_matches_single_gpu(t, name):
    cfg, full, fcache, models, caches, _ = _setup(t, name=name)
    B, T0 = 4, 20
    rng = np.random.default_rng(0)
    toks = torch.tensor(rng.integers(0, cfg.vocab, size=(B, T0 + 5)).astype(np.int32), device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    z = torch.zeros(B, dtype=torch.int32, device="cuda")
    # prefill then a Q=5 verify-shaped step, on both paths
    ref_lg = torch.empty(B * T0, cfg.vocab, device="cuda")
    full.forward(toks[:, :T0].contiguous(), z, slot, fcache, ref_lg)
    outs0, lg0 = _tp_step(models, caches, toks[:, :T0].contiguous(), z, slot)
    ref5 = torch.empty(B * 5, cfg.vocab, device="cuda")
    st = torch.full((B,), T0, dtype=torch.int32, device="cuda")
    full.forward(toks[:, T0:].contiguous(), st, slot, fcache, ref5)
    outs5, lg5 = _tp_step(models, caches, toks[:, T0:].contiguous(), st, slot)
    for outs, lg, ref in ((outs0, lg0, ref_lg), (outs5, lg5, ref5)):
        for r in range(1, t):
            assert torch.equal(outs[r], outs[0])  # identical on every rank
        got = torch.cat(lg, dim=1)  # rank slices in vocab order
        err = (got - ref).abs().max().item() / ref.abs().max().item()
        assert err < 3e-2, err
        assert torch.equal(outs[0].long(), got.argmax(-1))  # combine == argmax of the gathered logits
        agree = (outs[0].long() == ref.argmax(-1)).float().mean().item()
        assert agree >= 0.95, agree


def test_tp_forward_batch_invariant_and_deterministic():
    t = 2
    cfg, _, _, models, _, _ = _setup(t, seed=3)
    from paper_2402_15678_b200.opt import KVCache
    B, T0 = 3, 24
    rng = np.random.default_rng(1)
    toks = torch.tensor(rng.integers(0, cfg.vocab, size=(B, T0 + 5)).astype(np.int32), device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")

    def run(chunks):
        caches = [KVCache(m.cfg, B, 64) for m in models]
        res, p = [], 0
        for q in chunks:
            st = torch.full((B,), p, dtype=torch.int32, device="cuda")
            outs, lg = _tp_step(models, caches, toks[:, p:p + q].contiguous(), st, slot)
            res.append((outs[0].view(B, q), [x.view(B, q, -1) for x in lg]))
            p += q
        am = torch.cat([o for o, _ in res], 1)
        lg = [torch.cat([l[r] for _, l in res], 1) for r in range(t)]
        return am, lg

    a_am, a_lg = run([T0, 1, 1, 1, 1, 1])
    b_am, b_lg = run([T0, 5])
    c_am, c_lg = run([T0, 5])
    assert torch.equal(a_am[:, T0:], b_am[:, T0:])
    for r in range(t):
        assert torch.equal(a_lg[r][:, T0:], b_lg[r][:, T0:])
        assert torch.equal(b_lg[r], c_lg[r])
