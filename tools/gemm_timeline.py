"""Per-CTA timeline of one ms_linear launch (diagnostic build -DMS_EXP_TIMING,
MS_LIB=.../libminions_T.so): mainloop and epilogue durations, wave structure.
usage: MS_LIB=... python tools/gemm_timeline.py M N K act"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_15678_b200 import _native, kernels as K
M, N, Kd, act = (int(a) for a in sys.argv[1:5])
w = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(3)]
x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
r = None if act == 2 else torch.randn(M, N, device="cuda").to(torch.bfloat16)
out = torch.empty(M, N // 2 if act == 2 else N, device="cuda", dtype=torch.bfloat16)
for i in range(3):
    K.linear(x, w[i], residual=r, act=act, out=out)
torch.cuda.synchronize()
lib = _native.lib
lib.ms_exp_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = 4096
st = np.zeros(n * 4, np.uint64)
lib.ms_exp_stamps(st.ctypes.data, n)
st = st.reshape(n, 4).astype(np.int64)
st = st[st[:, 0] > 0]
t0 = st[:, 0].min()
start, main_end, end = (st[:, 0] - t0) / 1e3, (st[:, 1] - t0) / 1e3, (st[:, 2] - t0) / 1e3
ml = main_end - start
ep = end - main_end
print(f"CTAs {len(st)}  kernel span {end.max():.1f} us")
print(f"mainloop us: median {np.median(ml):.1f} p10 {np.percentile(ml, 10):.1f} p90 {np.percentile(ml, 90):.1f}")
print(f"epilogue us: median {np.median(ep):.2f} p10 {np.percentile(ep, 10):.2f} p90 {np.percentile(ep, 90):.2f}")
print(f"start us:  first-wave end ~{np.percentile(end, 50):.1f}; last start {start.max():.1f}; last end {end.max():.1f}")
hist = np.histogram(start, bins=10)
print("start histogram:", list(hist[0]), [round(b, 1) for b in hist[1]])
