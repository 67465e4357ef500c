"""A/B of the weight layout for the verify GEMMs (70B shapes): nn.Linear
row-major [N, K] vs tile-blocked [N/128][K/64][128][64] (every 128 x 64 TMA
tile one contiguous 16 KB run).  Same kernel, same launch, interleaved CUDA-
graph replays of L back-to-back launches over L distinct weight copies (like
L layers), so weights stream from HBM.  Checks the outputs are bitwise equal.

usage: python tools/wblock_probe.py [M,M,...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2402_15678_b200 import kernels as K

Ms = [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["16", "80", "112", "176"])]
SHAPES = [("qkv", 10240, 8192, 0), ("o", 8192, 8192, 0), ("gu", 57344, 8192, 2), ("down", 8192, 28672, 0),
          ("head", 32000, 8192, 0)]


blocked = K.block_weight


def graph_of(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def timeit(g, L, reps=3):
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / (reps * L)


for name, N, Kd, act in SHAPES:
    L = max(4, min(24, int(6e9 // (N * Kd * 2))))
    ws = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
    wb = [blocked(w) for w in ws]
    f32 = name == "head"
    for M in Ms:
        x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
        Nout = N // 2 if act == 2 else N
        outs = [torch.empty(M, Nout, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16) for _ in range(2)]

        def run(wl, o, blk):
            def f():
                for w in wl:
                    K.linear(x, w, out=o, out_f32=f32, act=act, w_blocked=blk)
            return f
        g_row = graph_of(run(ws, outs[0], False))
        g_blk = graph_of(run(wb, outs[1], True))
        same = bool(torch.equal(outs[0], outs[1]))
        tr, tb = [], []
        for _ in range(3):
            tr.append(timeit(g_row, L))
            tb.append(timeit(g_blk, L))
        byts = N * Kd * 2 + M * Kd * 2 + M * Nout * (4 if f32 else 2)
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": Kd, "L": L, "row_us": round(min(tr) * 1e6, 2),
                          "blocked_us": round(min(tb) * 1e6, 2), "row_GBs": round(byts / min(tr) / 1e9),
                          "blocked_GBs": round(byts / min(tb) / 1e9), "bitwise_equal": same}), flush=True)
    del ws, wb
    torch.cuda.empty_cache()
