"""One 70B verify forward (for ncu): python tools/verify_one.py [Q] [ctx]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 190
c = CONFIGS["llama-2-70b"]
B = 16
m = LlamaModel(LlamaWeights.random(c, 0), max_rows=B * Q)
cache = KVCache(c, B, 512)
tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
logits = torch.empty(B * Q, c.vocab, device="cuda")
for _ in range(2):
    m.forward(tok, start, slot, cache, logits)
torch.cuda.synchronize()
print("ok")
