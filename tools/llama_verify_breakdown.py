"""Warm per-category timing of a Llama verify forward (B requests, Q=s+1 rows
each, ctx keys): each category captured as its own CUDA graph and replayed —
full forward, the four GEMM kinds, attention, RMSNorms, LM head.
usage: python tools/llama_verify_breakdown.py [model] [Q] [ctx] [B]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache

name = sys.argv[1] if len(sys.argv) > 1 else "llama-2-70b"
Q = int(sys.argv[2]) if len(sys.argv) > 2 else 7
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 190
B = int(sys.argv[4]) if len(sys.argv) > 4 else 16
c = CONFIGS[name]
w = LlamaWeights.random(c, 0)
m = LlamaModel(w, max_rows=B * Q)
cache = KVCache(c, B, max(512, ctx + Q + 16))
tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
logits = torch.empty(B * Q, c.vocab, device="cuda")
R = B * Q
x, h, qkv, at, ff = m.x[:R], m.h[:R], m.qkv[:R], m.attn[:R], m.ff[:R]
x.normal_()
h.normal_()
at.normal_()
ff.normal_()

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

def attn():
    for i in range(c.n_layers):
        K.attention(qkv, B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], m.scale, out=at,
                    n_kv_heads=c.n_kv_heads, rope=m.rope)

def norms():
    for i in range(c.n_layers):
        K.rmsnorm(x, w[f"l{i}.attn_norm"], c.eps, out=h)
        K.rmsnorm(x, w[f"l{i}.mlp_norm"], c.eps, out=h)

def head():
    K.rmsnorm(x, w["norm_f"], c.eps, out=h)
    K.linear(h, w["lm_head"], out=logits, out_f32=True)

P = c.matmul_params()
sizes = {"qkv": c.d * c.qkv_out, "o": c.d * c.d, "gu": 2 * c.d * c.ffn, "down": c.d * c.ffn}
for nm, fn in [("full", full)] + [(k, gemm(k)) for k in ("qkv", "o", "gu", "down")] + \
        [("attention", attn), ("rmsnorm", norms), ("head", head)]:
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    extra = ""
    if nm in sizes:
        extra = f"  {2 * sizes[nm] * c.n_layers / ms / 1e9:7.0f} GB/s weights"
    if nm == "full":
        extra = f"  {2 * P / ms / 1e9:7.0f} GB/s weights"
    print(f"{name} B={B} Q={Q} ctx={ctx}: {nm:10s} {ms:8.3f} ms{extra}", flush=True)
