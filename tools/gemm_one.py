"""One ms_linear launch (after a warm-up launch) for ncu: usage
python tools/gemm_one.py M N K [act=0] — e.g. 320 57344 8192 2 = the 70B
gate/up projection at 320 token rows (a B=64 verify at s=4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
M, N, Kd = (int(v) for v in sys.argv[1:4])
act = int(sys.argv[4]) if len(sys.argv) > 4 else 0
x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16)
for _ in range(2):
    K.linear(x, w, act=act)
torch.cuda.synchronize()
print("ok")
