"""A/B of the 70B verify attention: the tcgen05 kernel (csrc/attention_tc.cu)
vs the warp-MMA row kernel, 80-layer chains (one KV cache per layer, B=16)
captured as CUDA graphs, replays interleaved; µs per layer and KV GB/s.
usage: python tools/attn_tc_ab.py ["Q:ctx,..."] ["H:Hkv:B:L"]   (default 64:8:16:80, the
70B heads; 40:40:16:40 = Llama-2-13B's multi-head attention, cfg5)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
cases = [tuple(int(v) for v in c.split(":")) for c in (sys.argv[1] if len(sys.argv) > 1 else
         "5:190,7:190,9:190,13:190,7:1000,5:4096").split(",")]
H, Hkv, B, L = (int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "64:8:16:80").split(":"))
D = 128
for Q, ctx in cases:
    T = ctx + 32
    caches = [(torch.zeros(B, Hkv, T, D, device="cuda", dtype=torch.bfloat16),
               torch.zeros(B, Hkv, T, D, device="cuda", dtype=torch.bfloat16)) for _ in range(L)]
    for kc, vc in caches:
        kc.normal_(); vc.normal_()
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
    out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    rope = K.rope_table(T + 8, D, 10000.0)
    graphs = {}
    for tc_on in (False, True):
        K.TC_ATTENTION = tc_on
        def f():
            for kc, vc in caches:
                K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out, n_kv_heads=Hkv, rope=rope)
        f(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[tc_on] = g
    K.TC_ATTENTION = "auto"
    res = {k: [] for k in graphs}
    for rep in range(3):
        for k, g in graphs.items():
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3 / L)
    kvb = B * Hkv * (ctx + Q) * D * 2 * 2
    row = {"H": H, "Hkv": Hkv, "B": B, "Q": Q, "ctx": ctx}
    for k, v in res.items():
        us = min(v)
        row["tc" if k else "rows"] = {"us_per_layer": round(us, 2), "GBs": round(kvb / (us * 1e-6) / 1e9)}
    print(json.dumps(row), flush=True)
    del caches, graphs
    torch.cuda.empty_cache()
