"""Weight-stream rate of the gate/up GEMM vs ring depth, with the MMA and token
loads switched off (ms_set_gemm_probe(1)) or on (0): 80-layer graph chains at
M rows with ring overrides sw:sx (ms_set_ring).
usage: python tools/ring_probe.py M "sw:sx,..." [probe=1]
(Measurement probe of round 2: the ms_set_gemm_trace / ms_set_gemm_probe /
ms_set_ring hooks it needs were removed from the product library after the
measurement — results in profiles/r2_epilogue_trace.txt.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native, kernels as K
from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights
M = int(sys.argv[1])
cfgs = [tuple(int(v) for v in c.split(":")) for c in sys.argv[2].split(",")]
probe = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = CONFIGS["llama-2-70b"]
w = LlamaWeights.random(c, 0)
h = torch.randn(M, c.d, device="cuda").to(torch.bfloat16)
ffo = torch.empty(M, c.ffn, device="cuda", dtype=torch.bfloat16)
graphs = {}
_native.lib.ms_set_gemm_probe(probe)
for sw, sx in cfgs:
    _native.lib.ms_set_ring(sw, sx)
    f = lambda: [K.linear(h, w[f"l{i}.w_gu"], act=2, out=ffo) for i in range(c.n_layers)]  # noqa: E731
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    graphs[(sw, sx)] = g
_native.lib.ms_set_ring(0, 0)
_native.lib.ms_set_gemm_probe(0)
res = {k: [] for k in graphs}
for rep in range(3):
    for k, g in graphs.items():
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); g.replay(); g.replay(); e1.record(); torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1) / 2)
for k, v in res.items():
    us = min(v) * 1e3 / c.n_layers
    print(json.dumps({"M": M, "probe": probe, "sw": k[0], "sx": k[1], "us": round(us, 1),
                      "TBs": round(2 * 2 * c.d * c.ffn / (us * 1e-6) / 1e12, 3)}), flush=True)
