"""Co-resident launch shapes (ms_set_coresident): the drafters' decode-step
kernels sized to fit beside two verify-GEMM CTAs per SM — 64-thread ms_gemv
and the shared-memory-free single-row decode attention — against fp32/fp64
restatements and the default shapes, plus the pipelined engine using them
staying lossless."""
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
BF = torch.bfloat16
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import llama_ref  # noqa: E402
from test_llama_gpu import _ref_attention  # noqa: E402


class _Coresident:
    def __enter__(self):
        from paper_2402_15678_b200 import _native
        self.old = _native.lib.ms_set_coresident(1)

    def __exit__(self, *a):
        from paper_2402_15678_b200 import _native
        _native.lib.ms_set_coresident(self.old)


@pytest.mark.parametrize("H,D,rope", [(12, 64, True), (4, 64, False), (8, 128, True)])
def test_decode_attention_vs_reference_and_default_kernel(H, D, rope):
    from paper_2402_15678_b200 import kernels as Kn
    B, T = 6, 300
    g = torch.Generator().manual_seed(H * 13 + D)
    kc = torch.randn(B, H, T, D, generator=g).to(BF)
    vc = torch.randn(B, H, T, D, generator=g).to(BF)
    qkv = torch.randn(B, 3 * H * D, generator=g).to(BF)
    start = torch.tensor([0, 1, 63, 64, 200, 298], dtype=torch.int32)
    table = llama_ref.rope_table(T + 4, D, 10000.0) if rope else None
    slot = torch.arange(B, dtype=torch.int32).cuda()
    outs, caches = [], []
    for co in (True, False):
        kcd, vcd = kc.cuda(), vc.cuda()
        kw = dict(rope=None if table is None else table.cuda())
        if co:
            with _Coresident():
                o = Kn.attention(qkv.cuda(), B, 1, H, D, slot, start.cuda(), kcd, vcd, D ** -0.5, **kw)
        else:
            o = Kn.attention(qkv.cuda(), B, 1, H, D, slot, start.cuda(), kcd, vcd, D ** -0.5, **kw)
        outs.append(o.cpu().float())
        caches.append((kcd.cpu(), vcd.cpu()))
    want = _ref_attention(qkv, kc, vc, start, B, 1, H, H, D, table)
    torch.testing.assert_close(outs[0], want, rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(outs[0], outs[1], rtol=2e-2, atol=2e-2)
    # the appended (rotated) K / V rows are bitwise the default kernel's
    assert torch.equal(caches[0][0], caches[1][0]) and torch.equal(caches[0][1], caches[1][1])
    # deterministic, and a request's output does not depend on the others
    with _Coresident():
        one = Kn.attention(qkv[4:5].cuda(), 1, 1, H, D, torch.tensor([4], dtype=torch.int32).cuda(), start[4:5].cuda(),
                           kc.cuda(), vc.cuda(), D ** -0.5, rope=None if table is None else table.cuda())
    assert torch.equal(one.cpu().float(), outs[0][4:5])


@pytest.mark.parametrize("M,N,K,act,rms", [(16, 2304, 768, 0, False), (16, 6144, 768, 2, True),
                                            (16, 768, 3072, 0, False), (16, 32000, 768, 0, True),
                                            (40, 512, 256, 0, True)])
def test_coresident_gemv(M, N, K, act, rms):
    from paper_2402_15678_b200 import kernels as Kn
    g = torch.Generator().manual_seed(M + N + K)
    G, eps = 3, 1e-6
    x = (torch.randn(G * M, K, generator=g) * 2).to(BF)
    w = (torch.randn(G, N, K, generator=g) * 0.03).to(BF)
    with _Coresident():
        got = Kn.gemv_grouped(x.cuda(), w.cuda(), G, act=act, out_f32=act == 0,
                              rms_eps=eps if rms else None).cpu().float()
        first = Kn.gemv_grouped(x[:1].contiguous().cuda(), w[:1].contiguous().cuda(), 1, act=act, out_f32=act == 0,
                                rms_eps=eps if rms else None).cpu().float()
    for k in range(G):
        xs = x[k * M:(k + 1) * M].double()
        y = xs @ w[k].double().T
        if rms:
            y = y * torch.rsqrt((xs ** 2).mean(-1, keepdim=True) + eps)
        if act == 2:
            t = y.view(M, -1, 2, 64)
            gt, up = t[:, :, 0].reshape(M, -1), t[:, :, 1].reshape(M, -1)
            y = gt * torch.sigmoid(gt) * up
        torch.testing.assert_close(got[k * M:(k + 1) * M], y.float(), rtol=2e-2, atol=2e-2)
    assert torch.equal(first, got[:1])


def test_pipelined_grouped_drafters_coresident_lossless():
    """Llama target + 3 grouped Llama drafters, pipelined: the drafters' decode
    steps run co-resident (the default there); output == greedy decode."""
    from paper_2402_15678_b200.core import EngineConfig, Request
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights
    tcfg, scfg = CONFIGS["tiny-llama"], CONFIGS["tiny-llama-ssm"]
    target = LlamaWeights.random(tcfg, 0, device="cuda", std=0.05, norm_std=0.1)
    drafters = [LlamaWeights.random(scfg, k + 1, device="cuda", std=0.05, norm_std=0.1) for k in range(3)]
    cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=4, b_ssm=4, s_init=4, initial_weights=(1.0,) * 3,
                       decision_threshold=3)
    eng = SpecEngine(target, drafters, cfg, slots=8, max_len=160, fidelity=[0.9, 0.7, 0.5], pipelined=True)
    assert eng.grouped and eng.draft_coresident
    rng = np.random.default_rng(5)
    reqs = [Request(f"req-{i:03d}", [int(t) for t in rng.integers(0, tcfg.vocab, size=int(rng.integers(4, 9)))], 40)
            for i in range(8)]
    teacher = eng.greedy_teacher([Request(r.id, list(r.prompt), 40) for r in reqs], 40)
    eng.capture_graphs()
    eng.prefill(reqs)
    eng.set_teacher(teacher)
    res = eng.decode()
    assert res.outputs == teacher
    assert res.mean_accepted > 1.0


def test_coresident_default_policy():
    """On by default for grouped drafters in the pipelined schedule with short
    caches only (the one-warp decode attention is slow at 4K contexts)."""
    from paper_2402_15678_b200.core import EngineConfig
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights
    tcfg, scfg = CONFIGS["tiny-llama"], CONFIGS["tiny-llama-ssm"]
    target = LlamaWeights.random(tcfg, 0, device="cuda", std=0.05)
    drafters = [LlamaWeights.random(scfg, k + 1, device="cuda", std=0.05) for k in range(3)]
    cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=2, b_ssm=2, s_init=4, initial_weights=(1.0,) * 3)
    short = SpecEngine(target, drafters, cfg, slots=4, max_len=200, pipelined=True)
    long_ = SpecEngine(target, drafters, cfg, slots=4, max_len=1100, pipelined=True)
    seq = SpecEngine(target, drafters, cfg, slots=4, max_len=200)
    forced = SpecEngine(target, drafters, cfg, slots=4, max_len=1100, pipelined=True, draft_coresident=True)
    assert short.draft_coresident and not long_.draft_coresident and not seq.draft_coresident
    assert forced.draft_coresident
