"""ncu target: single ms_linear launches on the 70B verify shapes (gate/up,
down, QKV) at M = 16 / 80 / 176, to read DRAM vs L2 (LTS) throughput.
usage: ncu --metrics ... python tools/gemm_l2_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2402_15678_b200 import kernels as K

for name, N, Kd, act in [("gu", 57344, 8192, 2), ("down", 8192, 28672, 0), ("qkv", 10240, 8192, 0)]:
    w = (torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16)
    for M in (16, 80, 176):
        x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
        out = torch.empty(M, N // 2 if act == 2 else N, device="cuda", dtype=torch.bfloat16)
        K.linear(x, w, act=act, out=out)
    torch.cuda.synchronize()
print("ok")
