"""Would the CTA-pair GEMM (ms_linear_wide: cta_group::2, 256-feature tiles,
persistent, double-buffered TMEM) stream the verify's gate/up weights faster
than ms_linear?  80 distinct 70B gate/up weights [57344, 8192], a CUDA graph
of 80 launches per kernel, replays interleaved; µs per layer and TB/s.
usage: python tools/wide_verify_probe.py [M,...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
Ms = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "16,80,112").split(",")]
L, N, Kd = 80, 2 * 28672, 8192
ws = []
for _ in range(L):
    w = torch.empty(N, Kd, device="cuda", dtype=torch.bfloat16)
    w.normal_(0, 0.02)
    ws.append(w)
for M in Ms:
    x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    graphs = {}
    for name, f in (("linear", lambda w: K.linear(x, w, act=2, out=out)),
                    ("wide", lambda w: K.linear_wide(x, w, act=2, out=out))):
        def chain(f=f):
            for w in ws:
                f(w)
        chain(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            chain()
        graphs[name] = g
    res = {k: [] for k in graphs}
    for rep in range(5):
        for k, g in graphs.items():
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3 / L)
    row = {"M": M}
    for k, v in res.items():
        us = sorted(v)[len(v) // 2]
        row[k] = {"us": round(us, 1), "TBs": round(N * Kd * 2 / (us * 1e-6) / 1e12, 2)}
    print(json.dumps(row), flush=True)
