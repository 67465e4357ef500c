"""A/B of the drafters' decode attention (grouped Llama-160M drafters: G x B
rows, 12 heads, D = 64, one position) with and without split-KV over the
cache length, L-layer chains as CUDA graphs, replays interleaved.
usage: python tools/draft_attn_split_ab.py [ctx,...] [G=5] [B=16]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K

ctxs = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "200,1000,4096").split(",")]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 5
B = int(sys.argv[3]) if len(sys.argv) > 3 else 16
H, D, L, Q = 12, 64, 12, 1
R = G * B
for ctx in ctxs:
    T = ctx + 64
    caches = [(torch.randn(R, H, T, D, device="cuda").to(torch.bfloat16),
               torch.randn(R, H, T, D, device="cuda").to(torch.bfloat16)) for _ in range(L)]
    qkv = torch.randn(R * Q, 3 * H * D, device="cuda").to(torch.bfloat16)
    out = torch.empty(R * Q, H * D, device="cuda", dtype=torch.bfloat16)
    slot = torch.arange(R, dtype=torch.int32, device="cuda")
    start = torch.full((R,), ctx, dtype=torch.int32, device="cuda")
    rope = K.rope_table(T + 8, D, 10000.0)
    ws = K.AttnWorkspace(R, Q, H, D, T, "cuda")
    outs, graphs = {}, {}
    for split in (False, True):
        def f():
            for kc, vc in caches:
                K.attention(qkv, R, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out, rope=rope,
                            ws=ws if split else None, append=False)
        f(); torch.cuda.synchronize()
        outs[split] = out.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[split] = g
    res = {k: [] for k in graphs}
    for rep in range(5):
        for k, g in graphs.items():
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3 / L)
    kvb = R * H * ctx * D * 2 * 2
    print(json.dumps({"G": G, "B": B, "ctx": ctx,
                      "whole_us": round(min(res[False]), 2), "split_us": round(min(res[True]), 2),
                      "whole_GBs": round(kvb / (min(res[False]) * 1e-6) / 1e9),
                      "split_GBs": round(kvb / (min(res[True]) * 1e-6) / 1e9),
                      "max_abs_diff": float((outs[True].float() - outs[False].float()).abs().max())}), flush=True)
    del caches, graphs
    torch.cuda.empty_cache()
