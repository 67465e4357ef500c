"""Target for ncu captures of the small hot-path kernels:
vote (K4), greedy accept from logits (K8 + K9) and one grouped drafter decode
step (3 x Llama-160M, 16 requests, 200-position caches: rmsnorm, gemv QKV /
O / gate-up, cluster GEMM down-proj, GQA/MHA attention, LM head, argmax).

usage: python tools/ncu_small.py [vote|accept|va|draft|draftco|all]
(draftco: the co-resident launch shapes the pipelined engine uses)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2402_15678_b200 import _native

what = sys.argv[1] if len(sys.argv) > 1 else "all"
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
rng = np.random.default_rng(0)

if what in ("vote", "va", "all"):
    for B, K, s in [(16, 3, 6), (256, 8, 16)]:
        tok = torch.tensor(rng.integers(0, 6, size=(B, K, s)).astype(np.int32), device="cuda")
        w = torch.tensor(1.25 ** rng.integers(-3, 4, size=K), dtype=torch.float64, device="cuda")
        path = torch.zeros(B, s, dtype=torch.int32, device="cuda")
        voted = torch.zeros(B, dtype=torch.int32, device="cuda")
        for _ in range(3):
            _native.call("ms_vote", tok.data_ptr(), w.data_ptr(), None, B, K, s, path.data_ptr(),
                         voted.data_ptr(), st())

if what in ("accept", "va", "all"):
    V = 32000
    for B, s in [(16, 6), (256, 16)]:
        path = torch.tensor(rng.integers(0, 4, size=(B, s)).astype(np.int32), device="cuda")
        logits = torch.randn(B, s + 1, V, device="cuda")
        rem = torch.full((B,), 1000, dtype=torch.int32, device="cuda")
        tgt = torch.zeros(B * (s + 1), dtype=torch.int32, device="cuda")
        ws = torch.zeros(B * (s + 1), dtype=torch.int64, device="cuda")
        n_acc, n_emit, fin = (torch.zeros(B, dtype=torch.int32, device="cuda") for _ in range(3))
        emitted = torch.zeros(B, s + 1, dtype=torch.int32, device="cuda")
        for _ in range(3):
            _native.call("ms_accept_greedy_logits", path.data_ptr(), logits.data_ptr(), 0, V, rem.data_ptr(), -1,
                         B, s, tgt.data_ptr(), ws.data_ptr(), n_acc.data_ptr(), emitted.data_ptr(),
                         n_emit.data_ptr(), fin.data_ptr(), None, st())

if what in ("draft", "draftco", "all"):
    from paper_2402_15678_b200.llama import GroupedLlamaModel
    from paper_2402_15678_b200.weights import CONFIGS, KVCache, LlamaWeights
    c = CONFIGS["llama-160m"]
    G, B, T = 3, 16, 200
    m = GroupedLlamaModel([LlamaWeights.random(c, k + 1) for k in range(G)], max_rows=B * 16)
    cache = KVCache(c, G * B, 512)
    tokens = torch.randint(0, c.vocab, (G * B, 1), dtype=torch.int32, device="cuda")
    start = torch.full((G * B,), T, dtype=torch.int32, device="cuda")
    slot = torch.arange(G * B, dtype=torch.int32, device="cuda")
    logits = torch.empty(G * B, c.vocab, device="cuda")
    am = torch.zeros(G * B, dtype=torch.int32, device="cuda")
    aws = torch.zeros(G * B, dtype=torch.int64, device="cuda")
    if what == "draftco":  # the pipelined engine's co-resident decode shapes
        _native.lib.ms_set_coresident(1)
        m.coresident = True
    for _ in range(3):
        m.forward(tokens, start, slot, cache, logits)
        _native.call("ms_argmax_rows", logits.data_ptr(), 0, G * B, c.vocab, c.vocab, am.data_ptr(),
                     aws.data_ptr(), st())
torch.cuda.synchronize()
print("ok")
