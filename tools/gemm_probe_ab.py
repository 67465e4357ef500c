"""Where does the verify GEMM's time go?  80-layer graph chains of the 70B
gate/up and down GEMMs at M rows under ms_set_gemm_probe: 0 full, 1 weight
stream only (no MMA, no token loads), 2 weight + token loads without MMA,
3 MMAs without token loads.  usage: python tools/gemm_probe_ab.py [M=112]
(Measurement probe of round 2: the ms_set_gemm_trace / ms_set_gemm_probe /
ms_set_ring hooks it needs were removed from the product library after the
measurement — results in profiles/r2_epilogue_trace.txt.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native, kernels as K
from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights

M = int(sys.argv[1]) if len(sys.argv) > 1 else 112
MODES = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,3,4,5").split(",")]
c = CONFIGS["llama-2-70b"]
w = LlamaWeights.random(c, 0)
L = c.n_layers
h = torch.randn(M, c.d, device="cuda").to(torch.bfloat16)
x = torch.randn(M, c.d, device="cuda").to(torch.bfloat16)
ff = torch.randn(M, c.ffn, device="cuda").to(torch.bfloat16)
ffo = torch.empty(M, c.ffn, device="cuda", dtype=torch.bfloat16)
qkv = torch.empty(M, c.qkv_out, device="cuda", dtype=torch.bfloat16)
def chain(kind):
    def f():
        for i in range(L):
            p = f"l{i}."
            if kind == "gu":
                K.linear(h, w[p + "w_gu"], act=2, out=ffo)
            elif kind == "qkv":
                K.linear(h, w[p + "w_qkv"], out=qkv)
            else:
                K.linear(ff, w[p + "w_down"], residual=x, out=x)
    return f
size = {"gu": 2 * c.d * c.ffn, "down": c.d * c.ffn, "qkv": c.d * c.qkv_out}
for kind in ("gu", "down", "qkv"):
    graphs = {}
    for mode in MODES:
        _native.lib.ms_set_gemm_probe(mode)
        f = chain(kind)
        f(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[mode] = g
    _native.lib.ms_set_gemm_probe(0)
    res = {k: [] for k in graphs}
    for rep in range(3):
        for k, g in graphs.items():
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g.replay(); g.replay(); e1.record(); torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) / 2)
    for k, v in res.items():
        us = min(v) * 1e3 / L
        print(json.dumps({"gemm": kind, "M": M, "probe": k, "us_per_layer": round(us, 2),
                          "TBs": round(2 * size[kind] / (us * 1e-6) / 1e12, 3)}), flush=True)
    del graphs
