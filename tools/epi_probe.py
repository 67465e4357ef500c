"""Single-launch device time of the 70B gate/up GEMM (ms_linear act=2) at M
rows, normal vs probe modes (ms_set_gemm_probe: 4 = no epilogue), each
launch on a cold weight slice (L2 holds < 1 of the 8 weight copies).
(Measurement probe of round 2: the ms_set_gemm_trace / ms_set_gemm_probe /
ms_set_ring hooks it needs were removed from the product library after the
measurement — results in profiles/r2_epilogue_trace.txt.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native, kernels as K
N, Kd = 57344, 8192
ws = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(8)]
for M in (16, 48, 80, 112, 160):
    x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    row = {"M": M}
    for mode in (0, 4, 5):
        _native.lib.ms_set_gemm_probe(mode)
        ts = []
        for it in range(24):
            w = ws[it % 8]
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda.synchronize()
            e0.record(); K.linear(x, w, act=2, out=out); e1.record(); torch.cuda.synchronize()
            if it >= 8:
                ts.append(e0.elapsed_time(e1) * 1e3)
        row[f"mode{mode}_us"] = round(sorted(ts)[len(ts) // 2], 1)
    _native.lib.ms_set_gemm_probe(0)
    print(json.dumps(row), flush=True)
