"""Per-launch time of ms_linear on the verify/decode shapes, measured as CUDA-graph
replays of L back-to-back launches over L distinct weight copies (like L layers),
so weights stream from HBM and launch gaps are those of the real forward."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import kernels as K

M_list = [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["16", "80"])]
split_opts = [a for a in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["sk"])]
SHAPES = {
    "opt": [("13b qkv", 15360, 5120), ("13b o", 5120, 5120), ("13b fc1", 20480, 5120),
            ("13b fc2", 5120, 20480), ("13b head", 50272, 5120), ("125m qkv", 2304, 768),
            ("125m o", 768, 768), ("125m fc1", 3072, 768), ("125m fc2", 768, 3072), ("125m head", 50272, 768)],
    "llama": [("70b qkv", 10240, 8192), ("70b o", 8192, 8192), ("70b gu", 57344, 8192),
              ("70b down", 8192, 28672), ("70b head", 32000, 8192), ("160m qkv", 2304, 768),
              ("160m gu", 6144, 768), ("160m down", 768, 3072), ("160m head", 32000, 768)],
}
shapes = SHAPES[sys.argv[3] if len(sys.argv) > 3 else "opt"]
for M in M_list:
    for name, N, Kd in shapes:
        L = max(4, min(40, int(8e9 // (N * Kd * 2))))
        ws = [(torch.randn(N, Kd, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(L)]
        x = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
        f32 = "head" in name
        out = torch.empty(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
        for sp in split_opts:
            wsp = None
            act = 2 if " gu" in name else 0
            if act == 2:
                out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
            if sp == "gemv":
                def run():
                    for w in ws:
                        K.gemv(x, w, out=out, out_f32=f32, act=act)
                spv = 0
            elif sp == "sk":
                wsp = K.Workspace("cuda")
                wsp.fit(M, N, Kd)
                spv = 0
            elif sp == "auto":  # splits=0, no workspace (MS_PK=1: whole-tile persistent)
                spv = 0
            else:
                spv = int(sp) or K.linear_splits(N, Kd)
            if sp != "gemv":
                def run():
                    for w in ws:
                        K.linear(x, w, out=out, out_f32=f32, splits=spv, ws=wsp, act=act)
            run(); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run()
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(3):
                g.replay()
            e1.record(); torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e-3 / (3 * L)
            byts = N * Kd * 2 + M * Kd * 2 + M * N * (4 if f32 else 2)
            print(f"M={M:4d} {name:10s} N={N:6d} K={Kd:6d} splits={sp if sp in ("sk", "gemv", "auto") else spv} L={L:3d} {t*1e6:8.2f} us/launch {byts/t/1e9:7.0f} GB/s", flush=True)
        del ws
        torch.cuda.empty_cache()
