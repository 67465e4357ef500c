"""Time one prompt prefill of the bench workload (Llama-2-70B target, B slots x
P positions) and its grouped-drafter prefill with CUDA events.
usage: prefill_time.py [B] [P]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
P = int(sys.argv[2]) if len(sys.argv) > 2 else 127
c = CONFIGS["llama-2-70b"]
m = LlamaModel(LlamaWeights.random(c, 0), max_rows=B * P)
cache = KVCache(c, B, 300)
tok = torch.randint(0, c.vocab, (B, P), dtype=torch.int32, device="cuda")
st = torch.zeros(B, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
empty = torch.zeros(0, dtype=torch.int32, device="cuda")
dummy = torch.empty(0, c.vocab, device="cuda")
for _ in range(2):
    m.forward(tok, st, slot, cache, dummy, head_rows=empty, prefill=True)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    m.forward(tok, st, slot, cache, dummy, head_rows=empty, prefill=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
fl = 2 * c.matmul_params() * B * P
print(f"prefill B={B} P={P}: {min(ts):.1f} ms, matmul {fl / 1e12:.0f} TFLOP -> {fl / min(ts) / 1e9:.0f} TFLOP/s overall", flush=True)
