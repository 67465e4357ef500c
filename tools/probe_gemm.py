"""Time ms_linear on the OPT-13B / OPT-125M verify and decode shapes (CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K

torch.manual_seed(0)
shapes = [("13b qkv", 15360, 5120), ("13b o", 5120, 5120), ("13b fc1", 20480, 5120),
          ("13b fc2", 5120, 20480), ("13b head", 50272, 5120), ("125m qkv", 2304, 768),
          ("125m fc1", 3072, 768), ("125m fc2", 768, 3072), ("125m head", 50272, 768)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for M in [int(a) for a in (sys.argv[1:] or ["16", "80"])]:
    for name, N, Kd in shapes:
        w = (torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
        f32 = "head" in name
        out = torch.empty(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
        for sp in sorted({K.linear_splits(N, Kd), 1}):
            for _ in range(3):
                K.linear(x, w, out=out, out_f32=f32, splits=sp)
            ts = []
            for _ in range(10):
                flush.zero_()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(); K.linear(x, w, out=out, out_f32=f32, splits=sp); e1.record()
                torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            t = sorted(ts)[len(ts) // 2] * 1e-3
            byts = N * Kd * 2 + M * Kd * 2 + M * N * (4 if f32 else 2)
            print(f"M={M:4d} {name:10s} N={N:6d} K={Kd:6d} splits={sp} {t*1e6:8.1f} us  {byts/t/1e9:7.0f} GB/s")
