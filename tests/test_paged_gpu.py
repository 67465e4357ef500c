"""Paged KV cache: attention / KV append through a block
table are bitwise equal to the contiguous cache (only addresses change); the
engine with a paged verifier cache produces the same tokens, frees the
blocks of rejected speculative tokens, and survives an over-subscribed pool."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
BF = torch.bfloat16


@pytest.mark.parametrize("H,Hkv,D,Q,T,bs", [(8, 2, 128, 5, 96, 16), (12, 12, 64, 1, 96, 16), (8, 8, 128, 20, 96, 16),
                                           (64, 8, 128, 11, 96, 16), (64, 8, 128, 7, 320, 32),
                                           # prompt-prefill tiles through the block table (Q * G > 128)
                                           (64, 8, 128, 40, 320, 32), (40, 40, 128, 130, 640, 64)])
@pytest.mark.parametrize("tc", [False, "auto"])
def test_paged_attention_bitwise_equals_contiguous(H, Hkv, D, Q, T, bs, tc, monkeypatch):
    """Either GQA kernel (the row kernel, or the tcgen05 one where "auto"
    selects it: 70B-style heads, caches <= 384 positions)."""
    from paper_2402_15678_b200 import kernels as Kn
    B = 3
    nb = T // bs
    g = torch.Generator().manual_seed(H + Q)
    kc = torch.randn(B, Hkv, T, D, generator=g).to(BF).cuda()
    vc = torch.randn(B, Hkv, T, D, generator=g).to(BF).cuda()
    # scatter the contiguous cache into a pool through a random block table
    perm = torch.randperm(B * nb + 2, generator=g)[: B * nb].view(B, nb).to(torch.int32)
    kp = torch.zeros(B * nb + 3, Hkv, bs, D, dtype=BF, device="cuda")
    vp = torch.zeros_like(kp)
    for b in range(B):
        for j in range(nb):
            kp[perm[b, j]] = kc[b, :, j * bs:(j + 1) * bs]
            vp[perm[b, j]] = vc[b, :, j * bs:(j + 1) * bs]
    table = perm.cuda()
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, generator=g).to(BF).cuda()
    start = torch.tensor([0, 33, T - Q - 1], dtype=torch.int32, device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    tab = Kn.rope_table(T, D, device="cuda")
    monkeypatch.setattr(Kn, "TC_ATTENTION", tc)
    a = Kn.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, n_kv_heads=Hkv, rope=tab)
    p = Kn.attention(qkv, B, Q, H, D, slot, start, kp, vp, D ** -0.5, n_kv_heads=Hkv, rope=tab, page=(table, bs))
    assert torch.equal(a, p)
    # the appended rows landed in the right blocks
    for b in range(B):
        for t in range(int(start[b]), int(start[b]) + Q):
            blk, row = int(perm[b, t // bs]), t % bs
            assert torch.equal(kp[blk, :, row], kc[b, :, t]) and torch.equal(vp[blk, :, row], vc[b, :, t])


@pytest.mark.parametrize("pipelined", [False, True])
def test_engine_paged_kv_same_tokens_and_frees_rejected(pipelined):
    from paper_2402_15678_b200.core import EngineConfig, Request
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights
    tcfg, scfg = CONFIGS["tiny-llama"], CONFIGS["tiny-llama-ssm"]
    target = LlamaWeights.random(tcfg, 0, device="cuda", std=0.05)
    drafters = [LlamaWeights.random(scfg, k + 1, device="cuda", std=0.05) for k in range(3)]
    outs = []
    for bs in (0, 16):
        cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=4, b_ssm=4, s_init=4, initial_weights=(1.0,) * 3)
        eng = SpecEngine(target, drafters, cfg, slots=4, max_len=128, fidelity=[0.9, 0.6, 0.3], adaptive=False,
                         kv_block_size=bs, pipelined=pipelined)
        eng.capture_graphs([4])
        rng = np.random.default_rng(1)
        reqs = [Request(f"req-{i:03d}", [int(t) for t in rng.integers(0, tcfg.vocab, size=int(rng.integers(5, 30)))],
                        48) for i in range(4)]
        teacher = eng.greedy_teacher([Request(r.id, list(r.prompt), 48) for r in reqs], 48)
        eng.prefill(reqs)
        eng.set_teacher(teacher)
        res = eng.decode()
        assert res.outputs == teacher
        outs.append(res.outputs)
        if bs:
            assert eng.t_cache.mgr.used() == 0  # every request finished: all blocks back in the pool
    assert outs[0] == outs[1]


def test_chunked_prefill_same_generation():
    """Prompt prefill in 8-position chunks (SURVEY §8f chunked prefill) gives
    exactly the generations of a one-chunk prefill (the prefill GEMMs,
    ms_linear_wide, accumulate the full K in k order whatever the chunk's row
    count, and the other kernels are batch-invariant)."""
    from paper_2402_15678_b200.core import EngineConfig, Request
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights
    tcfg, scfg = CONFIGS["tiny-llama"], CONFIGS["tiny-llama-ssm"]
    target = LlamaWeights.random(tcfg, 3, device="cuda", std=0.05)
    drafters = [LlamaWeights.random(scfg, k + 5, device="cuda", std=0.05) for k in range(3)]
    outs = []
    for chunk in (1024, 8):
        cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=4, b_ssm=4, s_init=3, initial_weights=(1.0,) * 3)
        eng = SpecEngine(target, drafters, cfg, slots=4, max_len=128, fidelity=[0.9, 0.6, 0.3], adaptive=False)
        eng.PREFILL_CHUNK = chunk
        rng = np.random.default_rng(2)
        reqs = [Request(f"req-{i:03d}", [int(t) for t in rng.integers(0, tcfg.vocab, size=int(rng.integers(20, 40)))],
                        24) for i in range(4)]
        teacher = eng.greedy_teacher([Request(r.id, list(r.prompt), 24) for r in reqs], 24)
        eng.prefill(reqs)
        eng.set_teacher(teacher)
        res = eng.decode()
        assert res.outputs == teacher
        outs.append((teacher, res.outputs))
    assert outs[0] == outs[1]
