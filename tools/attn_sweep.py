"""Verify/decode attention over the KV cache: device time (CUDA-graph replay)
and achieved HBM GB/s (algorithmic bytes = the K/V rows read, B*Hkv*ctx*D*2*2)
at decode contexts and at cfg5-like long contexts.
usage: attn_sweep.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K

cases = [  # name, B, Q, H, Hkv, D, ctx, rope, splitkv
    ("70b verify ctx190", 16, 11, 64, 8, 128, 190, True, False),
    ("70b verify ctx1k", 16, 11, 64, 8, 128, 1024, True, False),
    ("70b verify ctx4k", 16, 11, 64, 8, 128, 4096, True, False),
    ("13b(cfg5) verify ctx4k", 64, 5, 40, 40, 128, 4096, True, False),
    ("13b(cfg5) verify ctx4k splitkv", 64, 5, 40, 40, 128, 4096, True, True),
    ("160m decode ctx200 x3", 48, 1, 12, 12, 64, 200, True, False),
    ("160m decode ctx4k x5", 320, 1, 12, 12, 64, 4096, True, False),
]
for name, B, Q, H, Hkv, D, ctx, rope, skv in cases:
    T = ctx + Q + 8
    kc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
    vc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
    tab = K.rope_table(T, D, device="cuda") if rope else None
    ws = K.AttnWorkspace(B, Q, H, D, T, "cuda", n_kv_heads=Hkv) if skv else None
    def run():
        K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out, n_kv_heads=Hkv, rope=tab, ws=ws)
    run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            run()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    byts = B * Hkv * (ctx + Q) * D * 2 * 2
    print(f"{name:32s} {t*1e6:9.1f} us  {byts/1e6:9.1f} MB  {byts/t/1e9:7.0f} GB/s", flush=True)
    del kc, vc
    torch.cuda.empty_cache()
