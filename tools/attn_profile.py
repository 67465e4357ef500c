"""Launch the verify attention (OPT-13B shape) a few times for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
B, Q, H, D, T, ctx = 16, int(sys.argv[1]) if len(sys.argv) > 1 else 5, 40, 128, 512, 190
if len(sys.argv) > 2:
    H, D = 12, 64
kc = torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16)
vc = torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16)
qkv = torch.randn(B * Q, 3 * H * D, device="cuda").to(torch.bfloat16)
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out)
torch.cuda.synchronize()
