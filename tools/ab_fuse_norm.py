"""A/B of the folded RMSNorm on the Llama-2-70B verify forward (same weights,
same process): graph-replayed forward time, fuse_norm on vs off, interleaved."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache
c = CONFIGS["llama-2-70b"]
w = LlamaWeights.random(c, 0)
B = 16
for Q in (5, 7, 9, 11):
    ms = {}
    models = {"fused": LlamaModel(w, max_rows=B * Q, fuse_norm=True), "explicit": LlamaModel(w, max_rows=B * Q, fuse_norm=False)}
    cache = KVCache(c, B, 512)
    tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
    start = torch.full((B,), 190, dtype=torch.int32, device="cuda")
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    logits = torch.empty(B * Q, c.vocab, device="cuda")
    graphs = {}
    for k, m in models.items():
        m.forward(tok, start, slot, cache, logits); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            m.forward(tok, start, slot, cache, logits)
        graphs[k] = g
    t = {k: [] for k in graphs}
    for rep in range(6):
        for k, g in graphs.items():
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            t[k].append(e0.elapsed_time(e1))
    print(Q, {k: round(sorted(v)[len(v) // 2], 3) for k, v in t.items()}, flush=True)
    del models, graphs
    torch.cuda.empty_cache()
