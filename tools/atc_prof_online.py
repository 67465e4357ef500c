"""Phase timeline of the online-softmax tcgen05 attention (long caches) from
the diagnostic build (tools/build_atcprof.sh, -DATC_PROF): thread 0 (key
group 0's TMA / MMA issuer) stamps per CTA of the chain's last launch.
usage: MS_LIB=paper_2402_15678_b200/lib/ab/libminions_atcprof.so python tools/atc_prof_online.py [Q] [ctx]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_15678_b200 import _native, kernels as K
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
H, Hkv, D, B, L = 64, 8, 128, 16, 8
T = ctx + 32
caches = [(torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16),
           torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)) for _ in range(L)]
qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
slot = torch.arange(B, dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
rope = K.rope_table(T + 8, D, 10000.0)
K.TC_ATTENTION = True
def f():
    for kc, vc in caches:
        K.attention(qkv, B, Q, H, D, slot, start, kc, vc, D ** -0.5, out=out, n_kv_heads=Hkv, rope=rope)
f(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    f()
for _ in range(3):
    g.replay()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
buf = np.zeros((4096, 12), dtype=np.uint64)
assert _native.lib.ms_atc_prof_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
n = B * Hkv
t = buf[:n].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = {0: "entry", 1: "staged", 4: "s4", 2: "it4_S_loaded", 3: "it4_max", 6: "it4_pv_prev_done",
         8: "it4_rescaled", 10: "it4_half1", 11: "it4_bar", 7: "it4_pv_done", 5: "s8", 9: "exit"}
med = {names[i]: round(float(np.median(rel[:, i])), 2) for i in names}
print(json.dumps({"Q": Q, "ctx": ctx, "us_per_launch": round(e0.elapsed_time(e1) * 1e3 / L, 2),
                  "median_abs_us": med,
                  "per_iter_us_s4_s8": round(float(np.median(rel[:, 5] - rel[:, 4])) / 4, 3),
                  "max_exit_us": round(float(rel[:, 9].max()), 2)}))
