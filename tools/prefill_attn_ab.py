"""Prompt-prefill attention: tcgen05 query tiles (kernels.TC_PREFILL) vs the
warp-MMA row kernel, per layer (L-layer chains as CUDA graphs), for the
configs' prefill chunks.  usage: python tools/prefill_attn_ab.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K

cases = [  # (name, H, Hkv, B, Q, start, T, L, D)
    ("13b 4K chunk 4", 40, 40, 32, 1024, 3072, 4160, 4, 128),
    ("13b 4K chunk 1", 40, 40, 32, 1024, 0, 4160, 4, 128),
    ("70b 128-token prompts", 64, 8, 32, 127, 0, 272, 8, 128),
    ("5 x 160m 4K chunk 4 (D = 64: row kernel only)", 12, 12, 160, 1024, 3072, 4160, 2, 64),
]
if len(sys.argv) > 1:
    cases = [c for c in cases if sys.argv[1] in c[0]]
for name, H, Hkv, B, Q, st, T, L, D in cases:
    caches = [(torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16),
               torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)) for _ in range(L)]
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
    out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    start = torch.full((B,), st, dtype=torch.int32, device="cuda")
    rope = K.rope_table(T + 8, D, 10000.0)
    graphs, outs = {}, {}
    for tc in (False, True):
        K.TC_PREFILL = tc
        def f():
            for kc, vc in caches:
                K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out, n_kv_heads=Hkv, rope=rope)
        f(); torch.cuda.synchronize()
        outs[tc] = out.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[tc] = g
    K.TC_PREFILL = True
    res = {k: [] for k in graphs}
    for rep in range(3):
        for k, g in graphs.items():
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3 / L)
    keys = st + Q / 2
    fl = 4 * B * H * Q * keys * D
    print(json.dumps({"case": name, "rows_us": round(min(res[False]), 1), "tc_us": round(min(res[True]), 1),
                      "tc_TFLOPs": round(fl / (min(res[True]) * 1e-6) / 1e12, 1),
                      "rows_TFLOPs": round(fl / (min(res[False]) * 1e-6) / 1e12, 1),
                      "max_abs_diff": float((outs[True].float() - outs[False].float()).abs().max())}), flush=True)
    del caches, graphs
    torch.cuda.empty_cache()
