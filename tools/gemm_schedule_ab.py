"""A/B of the gate/up GEMM schedule (ms_set_gated_persistent: 0 = one tile
per CTA, 448 tiles = 1.51 waves; 1 = persistent two-per-SM CTAs with
double-buffered TMEM, gemm_gated.cuh) on the 70B verify forward (B=16, ctx 190)
and its four GEMM kinds: one CUDA graph per (schedule, what), replayed
interleaved.  (The same harness ran round 2's L2-prefetch, stream-K and
tail-split A/Bs, profiles/r2_*_ab.jsonl, whose knobs were removed.)
usage: python tools/gemm_schedule_ab.py [Qs=5,7,9]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native, kernels as K
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache

dists = [0, 1]
Qs = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "5,7,9").split(",")]
c = CONFIGS["llama-2-70b"]
B, ctx = 16, 190
w = LlamaWeights.random(c, 0)
m = LlamaModel(w, max_rows=B * max(Qs))
cache = KVCache(c, B, 512)
slot = torch.arange(B, dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
for Q in Qs:
    R = B * Q
    tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
    logits = torch.empty(R, c.vocab, device="cuda")
    x, h, qkv, at, ff = m.x[:R], m.h[:R], m.qkv[:R], m.attn[:R], m.ff[:R]
    def full():
        m.forward(tok, start, slot, cache, logits)
    def gemm(kind):
        def f():
            for i in range(c.n_layers):
                p = f"l{i}."
                if kind == "qkv":
                    K.linear(h, w[p + "w_qkv"], out=qkv)
                elif kind == "o":
                    K.linear(at, w[p + "w_o"], residual=x, out=x)
                elif kind == "gu":
                    K.linear(h, w[p + "w_gu"], act=2, out=ff)
                else:
                    K.linear(ff, w[p + "w_down"], residual=x, out=x)
        return f
    fns = [("full", full)] + [(k, gemm(k)) for k in ("qkv", "o", "gu", "down")]
    graphs = {}
    for d in dists:
        _native.lib.ms_set_gated_persistent(d)
        for nm, fn in fns:
            fn(); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            graphs[(d, nm)] = g
    _native.lib.ms_set_gated_persistent(1)
    res = {}
    for rep in range(3):
        for nm, _ in fns:
            for d in dists:
                g = graphs[(d, nm)]
                g.replay(); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for _ in range(3):
                    g.replay()
                e1.record(); torch.cuda.synchronize()
                res.setdefault((d, nm), []).append(e0.elapsed_time(e1) / 3)
    for nm, _ in fns:
        print(json.dumps({"Q": Q, "what": nm, "ms": {d: round(min(res[(d, nm)]), 3) for d in dists}}), flush=True)
    del graphs
