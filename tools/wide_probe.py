"""ms_linear_wide (2-CTA tcgen05 prefill GEMM) vs cuBLAS (torch.mm) vs the
weight-streaming ms_linear at prefill shapes: TFLOP/s per launch, CUDA-graph
replays of L launches over L weight copies.

usage: python tools/wide_probe.py [M,M,...] > profiles/r2_wide_probe.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2402_15678_b200 import kernels as K

Ms = [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["512", "1024", "2048", "4096"])]
SHAPES = [("70b qkv", 10240, 8192, 0), ("70b o", 8192, 8192, 0), ("70b gu", 57344, 8192, 2),
          ("70b down", 8192, 28672, 0), ("13b qkv", 15360, 5120, 0), ("13b gu", 27648, 5120, 2),
          ("160m gu", 6144, 768, 2)]


def tgraph(fn, L, reps=3):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3 / L)
    return best


for name, N, Kd, act in SHAPES:
    L = max(2, min(8, int(4e9 // (N * Kd * 2))))
    ws = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
    for M in Ms:
        x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
        No = N // 2 if act == 2 else N
        o = torch.empty(M, No, device="cuda", dtype=torch.bfloat16)
        o32 = torch.empty(M, N, device="cuda", dtype=torch.float32)
        t_w = tgraph(lambda: [K.linear_wide(x, w, act=act, out=o) for w in ws], L)
        t_l = tgraph(lambda: [K.linear(x, w, act=act, out=o) for w in ws], L)
        t_c = tgraph(lambda: [torch.mm(x, w.t(), out_dtype=torch.float32, out=o32) for w in ws], L)
        fl = 2.0 * M * N * Kd
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": Kd, "act": act,
                          "wide_tflops": round(fl / t_w / 1e12, 1), "linear_tflops": round(fl / t_l / 1e12, 1),
                          "cublas_tflops": round(fl / t_c / 1e12, 1), "wide_us": round(t_w * 1e6, 1)}), flush=True)
    del ws
    torch.cuda.empty_cache()
