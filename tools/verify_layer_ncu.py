"""ncu driver: three eager 70B verify forwards (B = 16, Q given, ctx 190);
capture one layer's kernels of the third with
  ncu --set full -k regex:"linear_kernel|linear_gated_kernel|attention_tc_short" -s 807 -c 5
(401 matching launches per forward: 80 x (QKV, attention, O, gate/up, down) + LM head).
usage: python tools/verify_layer_ncu.py [Q]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 7
c = CONFIGS["llama-2-70b"]
B, ctx = 16, 190
m = LlamaModel(LlamaWeights.random(c, 0), max_rows=B * Q)
cache = KVCache(c, B, 272)
tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
logits = torch.empty(B * Q, c.vocab, device="cuda")
for _ in range(3):
    m.forward(tok, start, slot, cache, logits)
torch.cuda.synchronize()
print("ok")
