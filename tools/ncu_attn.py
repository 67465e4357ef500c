"""Small driver for ncu captures of the 70B verify attention (B=16, Hkv=8,
H=64, D=128): a few launches of the tcgen05 kernel and the row kernel at
the given Q / context.  usage: python tools/ncu_attn.py [Q] [ctx]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 190
H, Hkv, D, B = 64, 8, 128, 16
T = ctx + 32
kc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
vc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
slot = torch.arange(B, dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
rope = K.rope_table(T + 8, D, 10000.0)
for tc in ("auto", False):
    K.TC_ATTENTION = tc
    for _ in range(3):
        K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out, n_kv_heads=Hkv, rope=rope)
torch.cuda.synchronize()
print("ok")
