"""Warm per-op timing of the grouped drafter decode step (3 x Llama-160M, 16
requests each, one position, ctx keys): each op kind as a 12-layer chain
captured in a CUDA graph (PDL on), µs per layer, and the op's algorithmic
bytes / time.  usage: python tools/draft_breakdown.py [ctx=200] [B=16] [G=3] [co]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native, kernels as K
from paper_2402_15678_b200.llama import GroupedLlamaModel
from paper_2402_15678_b200.weights import CONFIGS, KVCache, LlamaWeights

T = int(sys.argv[1]) if len(sys.argv) > 1 else 200
CO = len(sys.argv) > 4 and sys.argv[4] == "co"  # the co-resident launch shapes (ms_set_coresident)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
G = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = CONFIGS["llama-160m"]
m = GroupedLlamaModel([LlamaWeights.random(c, k + 1) for k in range(G)], max_rows=B * 16)
cache = KVCache(c, G * B, T + 64)
R = G * B
tokens = torch.randint(0, c.vocab, (R, 1), dtype=torch.int32, device="cuda")
start = torch.full((R,), T, dtype=torch.int32, device="cuda")
slot = torch.arange(R, dtype=torch.int32, device="cuda")
logits = torch.empty(R, c.vocab, device="cuda")
t = m.t
x, h, qkv, at, ff = m.x[:R], m.h[:R], m.qkv[:R], m.attn[:R], m.ff[:R]
for z in (x, h, qkv, at, ff):
    z.normal_()
L = c.n_layers


def lin(xx, name, **kw):
    wt = t[name]
    if B <= 64 and wt.shape[2] <= K.GEMV_MAX_K:
        return K.gemv_grouped(xx, wt, G, **kw)
    return K.linear_grouped(xx, wt.view(-1, wt.shape[2]), G, **kw)


ops = {
    "rmsnorm": (lambda i: K.rmsnorm_grouped(x, t[f"l{i}.attn_norm"], B, c.eps, out=h), 4 * R * c.d),
    "qkv": (lambda i: lin(h, f"l{i}.w_qkv", out=qkv), 2 * G * c.d * c.qkv_out),
    "attention": (lambda i: K.attention(qkv, R, 1, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], m.scale,
                                        out=at, n_kv_heads=c.n_kv_heads, rope=m.rope),
                  R * T * c.n_kv_heads * c.head_dim * 4),
    "o": (lambda i: lin(at, f"l{i}.w_o", residual=x, out=x), 2 * G * c.d * c.d),
    "gate_up": (lambda i: lin(h, f"l{i}.w_gu", act=2, out=ff), 2 * G * c.d * 2 * c.ffn),
    "down": (lambda i: lin(ff, f"l{i}.w_down", residual=x, out=x), 2 * G * c.d * c.ffn),
}
out = {}
if CO:
    _native.lib.ms_set_coresident(1)
for nm, (fn, byt) in ops.items():
    def chain():
        for i in range(L):
            fn(i)
    chain(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        chain()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 10 / L
    print(json.dumps({"op": nm, "us_per_layer": round(us, 2), "MB": round(byt / 1e6, 2),
                      "GBs": round(byt / (us * 1e-6) / 1e9)}), flush=True)
def head():
    K.rmsnorm_grouped(x, t["norm_f"], B, c.eps, out=h)
    hd = t["lm_head"]
    K.linear_grouped(h, hd.view(-1, hd.shape[2]), G, out=logits, out_f32=True)
head(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    head()
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    g.replay()
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 10
print(json.dumps({"op": "norm+lm_head", "us": round(us, 2), "MB": round(2 * G * c.vocab * c.d / 1e6, 1)}), flush=True)
