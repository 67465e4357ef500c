"""Debug run of the tcgen05 attention with bounded barrier waits (build with
-DATC_DEBUG into lib/ab/libminions_atcdbg.so; MS_LIB points at it)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as Kn
H, Hkv, D, T, Q, B = 64, 8, 128, 320, 5, 1
kc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
vc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
start = torch.tensor([int(sys.argv[1]) if len(sys.argv) > 1 else 60], dtype=torch.int32, device="cuda")
Kn.TC_ATTENTION = True
out = Kn.attention(qkv, B, Q, H, D, torch.arange(B, dtype=torch.int32, device="cuda"), start, kc, vc, D ** -0.5,
                   n_kv_heads=Hkv)
torch.cuda.synchronize()
print("done", out.float().abs().mean().item())
