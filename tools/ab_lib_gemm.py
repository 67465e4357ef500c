"""Same-process A/B of ms_linear between two builds of libminions (the
round-2 start, commit 07e7419, vs the current library): CUDA-graph replays
of L back-to-back launches over L weight copies, interleaved.

usage: python tools/ab_lib_gemm.py [old.so]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2402_15678_b200 import _native

old_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "ablib", "libminions_r2start.so")
old = ctypes.CDLL(old_path)
P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
old.ms_linear.argtypes = [P, I64, P, P, P, I64, P, I64, I, I, I, I, I, I, P, I64, P, I, P]
new = _native.lib


def call_old(x, w, out, M, N, K, act, st):
    r = old.ms_linear(x.data_ptr(), K, w.data_ptr(), None, None, 0, out.data_ptr(), out.stride(0), 0, M, N, K, act,
                      0, None, 0, None, 0, st)
    assert r == 0, r


def call_new(x, w, out, M, N, K, act, st):
    r = new.ms_linear(x.data_ptr(), K, w.data_ptr(), None, None, 0, out.data_ptr(), out.stride(0), 0, M, N, K, act,
                      0, st)
    assert r == 0, r


def graph(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    return g


def t(g, L):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / L


for name, N, Kd, act in [("qkv", 10240, 8192, 0), ("o", 8192, 8192, 0), ("gu", 57344, 8192, 2),
                         ("down", 8192, 28672, 0)]:
    L = max(4, min(24, int(6e9 // (N * Kd * 2))))
    ws = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
    for M in (16, 80, 176):
        x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
        o1 = torch.empty(M, N // 2 if act == 2 else N, device="cuda", dtype=torch.bfloat16)
        o2 = torch.empty_like(o1)

        def f_old():
            st = torch.cuda.current_stream().cuda_stream
            for w in ws:
                call_old(x, w, o1, M, N, Kd, act, st)

        def f_new():
            st = torch.cuda.current_stream().cuda_stream
            for w in ws:
                call_new(x, w, o2, M, N, Kd, act, st)
        go, gn = graph(f_old), graph(f_new)
        same = bool(torch.equal(o1, o2))
        to, tn = [], []
        for _ in range(4):
            to.append(t(go, L))
            tn.append(t(gn, L))
        byts = N * Kd * 2
        print(json.dumps({"gemm": name, "M": M, "old_us": round(min(to), 2), "new_us": round(min(tn), 2),
                          "old_TBs": round(byts / min(to) / 1e6, 2), "new_TBs": round(byts / min(tn) / 1e6, 2),
                          "bitwise_equal": same}), flush=True)
    del ws
    torch.cuda.empty_cache()
