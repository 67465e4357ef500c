"""Isolated drafter decode step (VERDICT r1 #4 metric): 3 x Llama-160M as one
grouped model, 16 requests per drafter, one position, KV caches at `ctx`
positions — forward + LM head + argmax, captured as one CUDA graph and
replayed; prints device µs per step and the step's algorithmic bytes / time.
usage: python tools/draft_step.py [ctx=200] [B=16] [G=3]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native
from paper_2402_15678_b200.llama import GroupedLlamaModel
from paper_2402_15678_b200.weights import CONFIGS, KVCache, LlamaWeights

T = int(sys.argv[1]) if len(sys.argv) > 1 else 200
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
G = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = CONFIGS["llama-160m"]
m = GroupedLlamaModel([LlamaWeights.random(c, k + 1) for k in range(G)], max_rows=B * 16)
cache = KVCache(c, G * B, T + 64)
tokens = torch.randint(0, c.vocab, (G * B, 1), dtype=torch.int32, device="cuda")
start = torch.full((G * B,), T, dtype=torch.int32, device="cuda")
slot = torch.arange(G * B, dtype=torch.int32, device="cuda")
logits = torch.empty(G * B, c.vocab, device="cuda")
am = torch.zeros(G * B, dtype=torch.int32, device="cuda")
aws = torch.zeros(G * B, dtype=torch.int64, device="cuda")
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def step():
    m.forward(tokens, start, slot, cache, logits)
    _native.call("ms_argmax_rows", logits.data_ptr(), 0, G * B, c.vocab, c.vocab, am.data_ptr(), aws.data_ptr(), st())


params = sum(t[0].numel() for k, t in m.t.items() if "norm" not in k) - m.t["tok_emb"][0].numel()
wbytes = 2 * G * params
kvbytes = G * B * T * c.n_layers * c.n_kv_heads * c.head_dim * 2 * 2
res = {}
for pdl in (1, 0):
    _native.lib.ms_set_pdl(pdl)
    n0 = _native.launch_count()
    step(); torch.cuda.synchronize()
    nk = _native.launch_count() - n0
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    res[pdl] = us
    print(json.dumps({"pdl": pdl, "G": G, "B": B, "ctx": T, "kernels": nk, "us_per_step": round(us, 1),
                      "weight_MB": round(wbytes / 1e6, 1), "kv_MB": round(kvbytes / 1e6, 1),
                      "GBs": round((wbytes + kvbytes) / (us * 1e-6) / 1e9)}), flush=True)
_native.lib.ms_set_pdl(1)
