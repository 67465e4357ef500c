"""Split-K sweep of the four 70B verify GEMMs (80-layer sequences captured as
CUDA graphs, interleaved replays): time per layer and weight GB/s for each
forced split count.  usage: python tools/split_sweep.py [Ms=80,112] [splits=1,2,3,4,5,6,8]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
from paper_2402_15678_b200.llama import CONFIGS, LlamaWeights

Ms = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "80,112").split(",")]
sps = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,4,5,6,8").split(",")]
c = CONFIGS["llama-2-70b"]
w = LlamaWeights.random(c, 0)
L = c.n_layers
Mx = max(Ms)
h = torch.randn(Mx, c.d, device="cuda").to(torch.bfloat16)
x = torch.randn(Mx, c.d, device="cuda").to(torch.bfloat16)
at = torch.randn(Mx, c.d, device="cuda").to(torch.bfloat16)
ff = torch.randn(Mx, c.ffn, device="cuda").to(torch.bfloat16)
qkv = torch.empty(Mx, c.qkv_out, device="cuda", dtype=torch.bfloat16)
for M in Ms:
    def mk(kind, sp):
        def f():
            for i in range(L):
                p = f"l{i}."
                if kind == "qkv":
                    K.linear(h[:M], w[p + "w_qkv"], out=qkv[:M], splits=sp)
                elif kind == "o":
                    K.linear(at[:M], w[p + "w_o"], residual=x[:M], out=x[:M], splits=sp)
                elif kind == "gu":
                    K.linear(h[:M], w[p + "w_gu"], act=2, out=ff[:M], splits=sp)
                else:
                    K.linear(ff[:M], w[p + "w_down"], residual=x[:M], out=x[:M], splits=sp)
        return f
    size = {"qkv": c.d * c.qkv_out, "o": c.d * c.d, "gu": 2 * c.d * c.ffn, "down": c.d * c.ffn}
    auto = {"qkv": K.linear_splits(c.qkv_out, c.d), "o": K.linear_splits(c.d, c.d),
            "gu": K.linear_splits(2 * c.ffn, c.d), "down": K.linear_splits(c.d, c.ffn)}
    for kind in ("qkv", "o", "gu", "down"):
        graphs = {}
        for sp in sps:
            f = mk(kind, sp)
            f(); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                f()
            graphs[sp] = g
        res = {sp: [] for sp in sps}
        for rep in range(3):
            for sp in sps:
                g = graphs[sp]
                g.replay(); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(); g.replay(); g.replay(); e1.record(); torch.cuda.synchronize()
                res[sp].append(e0.elapsed_time(e1) / 2)
        out = {sp: round(min(v) * 1e3 / L, 2) for sp, v in res.items()}
        gbs = {sp: round(2 * size[kind] / (us * 1e-6) / 1e9) for sp, us in out.items()}
        print(json.dumps({"M": M, "gemm": kind, "auto_split": auto[kind], "us_per_layer": out, "GBs": gbs}), flush=True)
        del graphs
