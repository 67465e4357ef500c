"""Same-process A/B of the 70B verify forward with the row-kernel attention vs
the tcgen05 attention (kernels.TC_ATTENTION False / "auto"): B requests x Q
rows, ctx cached keys, a bench-sized cache (T = 272), full forward and the
80-layer attention chain each captured as CUDA graphs, replays interleaved.
usage: python tools/verify_attn_ab.py [Q] [ctx] [B] [T]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 190
B = int(sys.argv[3]) if len(sys.argv) > 3 else 16
T = int(sys.argv[4]) if len(sys.argv) > 4 else 272
c = CONFIGS["llama-2-70b"]
w = LlamaWeights.random(c, 0)
m = LlamaModel(w, max_rows=B * Q)
cache = KVCache(c, B, T)
for k, v in zip(cache.k, cache.v):
    k.normal_(); v.normal_()
tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
logits = torch.empty(B * Q, c.vocab, device="cuda")
R = B * Q
m.qkv[:R].normal_()

def full():
    m.forward(tok, start, slot, cache, logits)

def attn():
    for i in range(c.n_layers):
        K.attention(m.qkv[:R], B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], m.scale,
                    out=m.attn[:R], n_kv_heads=c.n_kv_heads, rope=m.rope)

graphs = {}
for arm in (False, "auto"):
    K.TC_ATTENTION = arm
    for name, f in (("full", full), ("attention", attn)):
        f(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[(str(arm), name)] = g
K.TC_ATTENTION = "auto"
res = {k: [] for k in graphs}
for rep in range(7):
    for k, g in graphs.items():
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1))
out = {"Q": Q, "ctx": ctx, "B": B, "T": T}
for (arm, name), v in res.items():
    v = sorted(v)
    out[f"{name}_{'rows' if arm == 'False' else 'tc'}_ms"] = round(v[len(v) // 2], 3)
print(json.dumps(out), flush=True)
