"""Model-forward kernels against the fp32 CPU reference (oracle/opt_ref.py),
plus the properties the engine relies on: deterministic, batch-invariant rows
and KV-cache incremental decoding equal to a full forward."""
import numpy as np
import pytest
import torch

from conftest import ROOT
from oracle import opt_ref

pytestmark = pytest.mark.gpu


def _ref_linear(x, w, bias=None, residual=None, act=0, out_f32=False):
    y = x.float() @ w.float().T
    if bias is not None:
        y = y + bias.float()
    if act == 1:
        y = torch.relu(y)
    if residual is not None:
        y = y + residual.float()
    return y if out_f32 else y.to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(16, 768, 768), (80, 15360, 5120), (1, 50272, 256),
                                   (300, 1000, 200), (208, 3072, 768), (5, 128, 64),
                                   (256, 5120, 20480), (33, 2304, 768)])
@pytest.mark.parametrize("splits", [0, 1, 3])
def test_linear_vs_torch(M, N, K, splits):
    from paper_2402_15678_b200 import kernels as Kn
    g = torch.Generator().manual_seed(M * 7 + N + K)
    x = torch.randn(M, K, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(N, generator=g).to(torch.bfloat16)
    r = torch.randn(M, N, generator=g).to(torch.bfloat16)
    for act, res, f32 in ((0, None, True), (1, r, False), (0, r, False)):
        got = Kn.linear(x.cuda(), w.cuda(), b.cuda(), None if res is None else res.cuda(), act=act,
                        out_f32=f32, splits=splits).cpu()
        want = _ref_linear(x, w, b, res, act, f32)
        if f32:  # fp32 sums of K products in a different order
            torch.testing.assert_close(got, want, rtol=1e-4, atol=2e-5 * (K ** 0.5))
        else:  # one bf16 rounding of a value whose fp32 sum order differs
            torch.testing.assert_close(got.float(), want.float(), rtol=1.6e-2, atol=1e-2)


@pytest.mark.parametrize("N,K", [(5120, 5120), (50272, 768), (2304, 768)])
def test_linear_rows_independent_of_batch(N, K):
    """A row's result is bitwise the same whatever M (fixed split count)."""
    from paper_2402_15678_b200 import kernels as Kn
    g = torch.Generator().manual_seed(1)
    w = (torch.randn(N, K, generator=g) * 0.02).to(torch.bfloat16).cuda()
    x = torch.randn(300, K, generator=g).to(torch.bfloat16).cuda()
    sp = Kn.linear_splits(N, K)
    full = Kn.linear(x, w, out_f32=True, splits=sp)
    for M in (1, 16, 17, 80, 129, 208):
        part = Kn.linear(x[:M].contiguous(), w, out_f32=True, splits=sp)
        assert torch.equal(part, full[:M]), M
    assert torch.equal(Kn.linear(x, w, out_f32=True, splits=sp), full)  # deterministic


def _tiny(seed=0, cfg_name="tiny-target"):
    from paper_2402_15678_b200.opt import CONFIGS, OPTWeights
    cfg = CONFIGS[cfg_name]
    w_cpu = OPTWeights.random(cfg, seed, device="cpu", std=0.05, bias_std=0.02)
    return cfg, w_cpu


def test_forward_prefill_and_decode_vs_reference():
    from paper_2402_15678_b200.opt import KVCache, OPTModel
    cfg, w_cpu = _tiny()
    model = OPTModel(w_cpu.to("cuda"), max_rows=256)
    B, T0, steps = 4, 24, 6
    rng = np.random.default_rng(0)
    toks = rng.integers(0, cfg.vocab, size=(B, T0 + steps)).astype(np.int32)
    cache = KVCache(cfg, B, 64)
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    # prefill T0 positions
    logits = torch.empty(B * T0, cfg.vocab, device="cuda")
    model.forward(torch.tensor(toks[:, :T0], device="cuda"), torch.zeros(B, dtype=torch.int32, device="cuda"),
                  slot, cache, logits)
    got_pre = logits.view(B, T0, -1).cpu()
    # then one position at a time, then a Q=3 "verify" chunk
    got_dec = []
    for j in range(3):
        lg = torch.empty(B, cfg.vocab, device="cuda")
        model.forward(torch.tensor(toks[:, T0 + j: T0 + j + 1], device="cuda"),
                      torch.full((B,), T0 + j, dtype=torch.int32, device="cuda"), slot, cache, lg)
        got_dec.append(lg.cpu())
    lg3 = torch.empty(B * 3, cfg.vocab, device="cuda")
    model.forward(torch.tensor(toks[:, T0 + 3: T0 + 6], device="cuda"),
                  torch.full((B,), T0 + 3, dtype=torch.int32, device="cuda"), slot, cache, lg3)
    lg3 = lg3.view(B, 3, -1).cpu()
    agree, total, worst = 0, 0, 0.0
    for b in range(B):
        ref = opt_ref.forward(w_cpu.t, cfg, toks[b])
        got = torch.cat([got_pre[b], torch.stack([g[b] for g in got_dec]), lg3[b]])
        err = (got - ref).abs().max().item() / ref.abs().max().item()
        worst = max(worst, err)
        agree += int((got.argmax(-1) == ref.argmax(-1)).sum())
        total += got.shape[0]
    assert worst < 2e-2, worst
    assert agree / total >= 0.97, agree / total


def test_forward_batch_invariant_and_deterministic():
    """Logits of a position are bitwise identical whether it is computed alone
    (Q=1), inside a Q=5 verify chunk, or with other requests in the batch."""
    from paper_2402_15678_b200.opt import KVCache, OPTModel
    cfg, w_cpu = _tiny(1)
    model = OPTModel(w_cpu.to("cuda"), max_rows=256)
    B, T0 = 3, 40
    rng = np.random.default_rng(1)
    toks = torch.tensor(rng.integers(0, cfg.vocab, size=(B, T0 + 5)).astype(np.int32), device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")

    def run(chunks):
        cache = KVCache(cfg, B, 64)
        outs, p = [], 0
        for q in chunks:
            lg = torch.empty(B * q, cfg.vocab, device="cuda")
            model.forward(toks[:, p:p + q].contiguous(), torch.full((B,), p, dtype=torch.int32, device="cuda"),
                          slot, cache, lg)
            outs.append(lg.view(B, q, -1))
            p += q
        return torch.cat(outs, 1)

    a = run([T0, 1, 1, 1, 1, 1])
    b = run([T0, 5])
    c = run([T0, 2, 3])
    assert torch.equal(a[:, T0:], b[:, T0:])
    assert torch.equal(a[:, T0:], c[:, T0:])
    # one request alone in the batch
    cache = KVCache(cfg, 1, 64)
    lg = torch.empty(T0 + 5, cfg.vocab, device="cuda")
    model.forward(toks[1:2], torch.zeros(1, dtype=torch.int32, device="cuda"),
                  torch.zeros(1, dtype=torch.int32, device="cuda"), cache, lg)
    lgb = torch.empty(B * (T0 + 5), cfg.vocab, device="cuda")
    cache = KVCache(cfg, B, 64)
    model.forward(toks, torch.zeros(B, dtype=torch.int32, device="cuda"), slot, cache, lgb)
    assert torch.equal(lg, lgb.view(B, T0 + 5, -1)[1])


def test_head_rows_gather():
    from paper_2402_15678_b200.opt import KVCache, OPTModel
    cfg, w_cpu = _tiny(2, "tiny-ssm")
    model = OPTModel(w_cpu.to("cuda"), max_rows=64)
    B, Q = 4, 6
    toks = torch.randint(0, cfg.vocab, (B, Q), dtype=torch.int32, device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    start = torch.zeros(B, dtype=torch.int32, device="cuda")
    full = torch.empty(B * Q, cfg.vocab, device="cuda")
    model.forward(toks, start, slot, KVCache(cfg, B, 16), full)
    rows = torch.tensor([5, 6, 17, 23], dtype=torch.int32, device="cuda")
    part = torch.empty(4, cfg.vocab, device="cuda")
    model.forward(toks, start, slot, KVCache(cfg, B, 16), part, head_rows=rows)
    assert torch.equal(part, full[rows.long()])


@pytest.mark.parametrize("D,H,Hkv,Q", [(128, 8, 8, 5), (64, 12, 12, 1), (64, 4, 4, 13),
                                      (128, 64, 8, 5), (128, 16, 2, 13), (64, 8, 2, 1)])
def test_attention_split_kv_matches_and_is_batch_invariant(D, H, Hkv, Q):
    """Split over the cache length (chunks fixed by the cache length,
    chunk-order merge; MHA kernel and, Hkv < H, the GQA row kernel) agrees
    with the single-CTA walk and, per query, does not depend on the other
    queries."""
    from paper_2402_15678_b200 import kernels as Kn
    B, T = 6, 512
    g = torch.Generator().manual_seed(D + Q + H)
    kc = (torch.randn(B, Hkv, T, D, generator=g)).to(torch.bfloat16).cuda()
    vc = (torch.randn(B, Hkv, T, D, generator=g)).to(torch.bfloat16).cuda()
    start = torch.tensor([0, 63, 64, 127, 200, 480], dtype=torch.int32, device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, generator=g).to(torch.bfloat16).cuda()
    kw = dict(n_kv_heads=Hkv)
    ws = Kn.AttnWorkspace(B, Q, H, D, T, "cuda", n_kv_heads=Hkv)
    a = Kn.attention(qkv, B, Q, H, D, slot, start, kc.clone(), vc.clone(), D ** -0.5, ws=ws, **kw)
    b = Kn.attention(qkv, B, Q, H, D, slot, start, kc.clone(), vc.clone(), D ** -0.5, ws=None, **kw)
    torch.testing.assert_close(a.float(), b.float(), rtol=2e-2, atol=2e-2)
    assert torch.equal(a, Kn.attention(qkv, B, Q, H, D, slot, start, kc.clone(), vc.clone(), D ** -0.5, ws=ws,
                                       **kw))
    # the first query row of every request alone (Q=1) == row 0 of the Q-row call
    q1 = qkv.view(B, Q, -1)[:, :1].contiguous().view(B, -1)
    ws1 = Kn.AttnWorkspace(B, 1, H, D, T, "cuda", n_kv_heads=Hkv)
    a1 = Kn.attention(q1, B, 1, H, D, slot, start, kc.clone(), vc.clone(), D ** -0.5, ws=ws1, **kw)
    assert torch.equal(a1, a.view(B, Q, -1)[:, 0])


@pytest.mark.parametrize("M,N,K", [(16, 2304, 768), (1, 768, 3072), (16, 768, 3072), (48, 768, 4096),
                                   (33, 3072, 768), (64, 100, 256), (5, 1000, 96)])
def test_gemv_vs_torch_and_row_invariance(M, N, K):
    from paper_2402_15678_b200 import kernels as Kn
    g = torch.Generator().manual_seed(M * 3 + N)
    x = torch.randn(M, K, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(N, generator=g).to(torch.bfloat16)
    r = torch.randn(M, N, generator=g).to(torch.bfloat16)
    for act, res, f32 in ((0, None, True), (1, r, False)):
        got = Kn.gemv(x.cuda(), w.cuda(), b.cuda(), None if res is None else res.cuda(), act=act,
                      out_f32=f32).cpu()
        want = _ref_linear(x, w, b, res, act, f32)
        if f32:
            torch.testing.assert_close(got, want, rtol=1e-4, atol=2e-5 * (K ** 0.5))
        else:
            torch.testing.assert_close(got.float(), want.float(), rtol=1.6e-2, atol=1e-2)
    full = Kn.gemv(x.cuda(), w.cuda(), out_f32=True)
    one = Kn.gemv(x[:1].cuda().contiguous(), w.cuda(), out_f32=True)
    assert torch.equal(one, full[:1])


def test_drafter_forward_small_gemm_vs_reference():
    """The drafter path (ms_gemv for <= 64 rows) against the fp32 reference."""
    from paper_2402_15678_b200.opt import CONFIGS, KVCache, OPTModel, OPTWeights
    cfg = CONFIGS["tiny-ssm"]
    w_cpu = OPTWeights.random(cfg, 3, device="cpu", std=0.05, bias_std=0.02)
    m = OPTModel(w_cpu.to("cuda"), max_rows=256, small_gemm=True)
    B, T0 = 4, 12
    rng = np.random.default_rng(3)
    toks = rng.integers(0, cfg.vocab, size=(B, T0 + 3)).astype(np.int32)
    cache = KVCache(cfg, B, 64)
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    lg = torch.empty(B * T0, cfg.vocab, device="cuda")
    m.forward(torch.tensor(toks[:, :T0], device="cuda"), torch.zeros(B, dtype=torch.int32, device="cuda"),
              slot, cache, lg)
    outs = [lg.view(B, T0, -1).cpu()]
    for j in range(3):
        l1 = torch.empty(B, cfg.vocab, device="cuda")
        m.forward(torch.tensor(toks[:, T0 + j:T0 + j + 1], device="cuda"),
                  torch.full((B,), T0 + j, dtype=torch.int32, device="cuda"), slot, cache, l1)
        outs.append(l1.view(B, 1, -1).cpu())
    got = torch.cat(outs, 1)
    for b in range(B):
        ref = opt_ref.forward(w_cpu.t, cfg, toks[b])
        err = (got[b] - ref).abs().max().item() / ref.abs().max().item()
        assert err < 2e-2, err
