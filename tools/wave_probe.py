"""Is the gate/up GEMM limited by wave quantization?  Time ms_linear (gated)
at M rows for N = k * 2 * 148 tiles (full waves at 2 CTAs/SM) vs 448 tiles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
for M in (112, 176):
    for tiles in (148, 296, 448, 592):
        N = tiles * 128
        L = max(4, min(16, int(8e9 // (N * 8192 * 2))))
        ws = [(torch.randn(N, 8192, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
        x = torch.randn(M, 8192, device="cuda").to(torch.bfloat16)
        out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        def run():
            for w in ws:
                K.linear(x, w, out=out, act=2)
        run(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); g.replay(); g.replay(); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / (2 * L)
        print(f"M={M} tiles={tiles} N={N}: {t*1e6:8.1f} us  {N*8192*2/t/1e9:7.0f} GB/s", flush=True)
        del ws
        torch.cuda.empty_cache()
