"""DRAM traffic of one Llama verify forward (all its kernels), for the bench's
roofline.traffic: run under
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv
usage: verify_traffic.py [model] [Q] [ctx] [B]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache

name = sys.argv[1] if len(sys.argv) > 1 else "llama-2-70b"
Q = int(sys.argv[2]) if len(sys.argv) > 2 else 11
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 190
B = int(sys.argv[4]) if len(sys.argv) > 4 else 16
c = CONFIGS[name]
m = LlamaModel(LlamaWeights.random(c, 0), max_rows=B * Q)
cache = KVCache(c, B, 512)
tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
logits = torch.empty(B * Q, c.vocab, device="cuda")
m.forward(tok, start, slot, cache, logits)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.forward(tok, start, slot, cache, logits)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("algorithmic bytes", 2 * c.matmul_params() + B * ctx * c.kv_bytes_per_token() + B * Q * c.kv_bytes_per_token())
