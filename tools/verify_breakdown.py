"""Warm per-category timing of the OPT-13B verify forward (B=16, Q=s+1), each
category captured as its own CUDA graph and replayed: full forward, GEMMs only,
attention only, LayerNorms only, LM head only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
from paper_2402_15678_b200.opt import CONFIGS, KVCache, OPTModel, OPTWeights

name = sys.argv[1] if len(sys.argv) > 1 else "opt-13b"
B, Q, ctx = 16, int(sys.argv[2]) if len(sys.argv) > 2 else 5, 190
c = CONFIGS[name]
w = OPTWeights.random(c, 0)
m = OPTModel(w, max_rows=B * Q)
cache = KVCache(c, B, 512)
tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
logits = torch.empty(B * Q, c.vocab, device="cuda")
R = B * Q
x, h, qkv, at, ff = m.x[:R], m.h[:R], m.qkv[:R], m.attn[:R], m.ff[:R]

def full():
    m.forward(tok, start, slot, cache, logits)

def gemms():
    for i in range(c.n_layers):
        p = f"l{i}."
        K.linear(h, w[p + "w_qkv"], w[p + "b_qkv"], out=qkv)
        K.linear(at, w[p + "w_o"], w[p + "b_o"], residual=x, out=x)
        K.linear(h, w[p + "w_fc1"], w[p + "b_fc1"], act=1, out=ff)
        K.linear(ff, w[p + "w_fc2"], w[p + "b_fc2"], residual=x, out=x)

def attn():
    for i in range(c.n_layers):
        K.attention(qkv, B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], m.scale, out=at,
                    ws=m._attn_ws(B, Q, cache.max_len) if os.environ.get("MS_SPLITKV", "0") == "1" else None)

def lns():
    for i in range(c.n_layers):
        p = f"l{i}."
        K.layernorm(x, w[p + "ln1_g"], w[p + "ln1_b"], c.eps, out=h)
        K.layernorm(x, w[p + "ln2_g"], w[p + "ln2_b"], c.eps, out=h)

def head():
    K.layernorm(x, w["lnf_g"], w["lnf_b"], c.eps, out=h)
    K.linear(h, w["tok_emb"], out=logits, out_f32=True)

for nm, fn in (("full", full), ("gemms", gemms), ("attention", attn), ("layernorm", lns), ("head", head)):
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
    print(f"{name} B={B} Q={Q} ctx={ctx}: {nm:10s} {e0.elapsed_time(e1) / 5:8.3f} ms", flush=True)
