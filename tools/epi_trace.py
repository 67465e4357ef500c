"""Per-CTA phase timestamps (ms_set_gemm_trace) of one 70B gate/up launch at M
rows: when CTAs start, finish streaming, finish the MMAs, and how long the
gated epilogue phases take.  usage: python tools/epi_trace.py [M=112] [N=57344] [K=8192] [act=2]
(Measurement probe of round 2: the ms_set_gemm_trace / ms_set_gemm_probe /
ms_set_ring hooks it needs were removed from the product library after the
measurement — results in profiles/r2_epilogue_trace.txt.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_15678_b200 import _native, kernels as K
M = int(sys.argv[1]) if len(sys.argv) > 1 else 112
N = int(sys.argv[2]) if len(sys.argv) > 2 else 57344
Kd = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
act = int(sys.argv[4]) if len(sys.argv) > 4 else 2
rms = len(sys.argv) > 5 and sys.argv[5] == "rms"  # residual + folded-norm partials (the verify's O / down)
w = (torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16)
x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
out = torch.empty(M, N // 2 if act == 2 else N, device="cuda", dtype=torch.bfloat16)
n_cta = ((N + 127) // 128) * K.linear_splits(N, Kd)
buf = torch.zeros(n_cta * 12, dtype=torch.int64, device="cuda")
res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
parts = torch.zeros(M, (N + 127) // 128, device="cuda")
def run():
    if rms:
        K.linear_rms(x, w, residual=res, out=res, rms_out=parts)
    else:
        K.linear(x, w, act=act, out=out)
run(); torch.cuda.synchronize()
_native.lib.ms_set_gemm_trace(buf.data_ptr())
run(); torch.cuda.synchronize()
_native.lib.ms_set_gemm_trace(None)
t = buf.view(n_cta, 12).cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
first = t[:, 0] < np.median(t[:, 0]) + 5
def q(a):
    return [round(float(np.percentile(a, p)), 1) for p in (0, 50, 100)]
print(json.dumps({"M": M, "N": N, "K": Kd, "ctas": n_cta, "start": q(t[:, 0]), "last_w_issue": q(t[:, 1]), "raw8": q(t[:, 8]), "mma_issued": q(t[:, 2]),
                  "acc_done": q(t[:, 3]), "phase_a": q(t[:, 4] - t[:, 3]), "phase_b": q(t[:, 5] - t[:, 4]),
                  "stores": q(t[:, 6] - t[:, 5]), "to_loaded": q(t[:, 8] - t[:, 5]), "to_stored": q(t[:, 9] - t[:, 5]), "exit": q(t[:, 7]), "epilogue_total": q(t[:, 7] - t[:, 3]),
                  "n_second_wave": int((t[:, 0] > 20).sum())}))
