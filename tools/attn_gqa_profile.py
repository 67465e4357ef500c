"""Launch the 70B verify GQA attention (B=16, H=64, Hkv=8, D=128, RoPE) a few
times for ncu.  usage: attn_gqa_profile.py [Q] [ctx]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 190
B, H, Hkv, D = 16, 64, 8, 128
T = 512
kc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
vc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
tab = K.rope_table(T, D, device="cuda")
for _ in range(5):
    K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out, n_kv_heads=Hkv, rope=tab)
torch.cuda.synchronize()
