"""Large-M (prefill) GEMM: ms_linear vs cuBLAS (torch.matmul) on the 70B
shapes at M = B * prompt tokens, each as a CUDA-graph replay of L launches.
usage: prefill_gemm_probe.py [M]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
M = int(sys.argv[1]) if len(sys.argv) > 1 else 2032
for name, N, Kd, act in (("qkv", 10240, 8192, 0), ("o", 8192, 8192, 0), ("gu", 57344, 8192, 2), ("down", 8192, 28672, 0)):
    L = 4
    ws = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
    x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N // 2 if act == 2 else N, device="cuda", dtype=torch.bfloat16)
    full = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for impl in ("ms", "cublas"):
        def run():
            for w in ws:
                if impl == "ms":
                    K.linear(x, w, out=out, act=act)
                else:
                    torch.matmul(x, w.t(), out=full)
        run(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / (3 * L)
        print(f"M={M} {name:5s} N={N} K={Kd} {impl:6s} {t*1e6:9.1f} us  {2*M*N*Kd/t/1e12:7.1f} TFLOP/s", flush=True)
    del ws
