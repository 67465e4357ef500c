"""Run one GEMM shape a few times (for ncu): python tools/gemm_one.py M N K act [splits] [reps]
splits = -1: the persistent stream-K schedule (a Workspace is passed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K
M, N, Kd, act = (int(a) for a in sys.argv[1:5])
splits = int(sys.argv[5]) if len(sys.argv) > 5 else 0
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
ws = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(reps)]
x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
out = torch.empty(M, N // 2 if act == 2 else N, device="cuda", dtype=torch.bfloat16)
wsp = None
if splits < 0:
    wsp = K.Workspace("cuda")
    wsp.fit(M, N, Kd)
    splits = 0
for w in ws:
    K.linear(x, w, out=out, act=act, splits=splits, ws=wsp)
torch.cuda.synchronize()
print("ok")
