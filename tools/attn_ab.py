"""A/B of the GQA verify attention (ms_attention_gqa, Llama-2-70B heads,
RoPE) between builds of libminions (raw ctypes, so an older build works):
device time per call (back-to-back launches over L distinct KV caches, like
L layers, so K/V stream from HBM as in a forward) and the max |difference| of
each build's output vs the first build's.
usage: python tools/attn_ab.py lib_a.so lib_b.so ..."""
import ctypes, os, sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
P, I, I64, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
libs = [ctypes.CDLL(p) for p in sys.argv[1:]]
for lib in libs:
    lib.ms_attention_gqa.argtypes = [P, I64, I, I, I, I, I, P, P, I, P, P, P, F, I, P, I64, P, I64, P, I, P]


def rope_table(T, D, theta=10000.0):
    inv = 1.0 / (theta ** (torch.arange(0, D, 2, dtype=torch.float64) / D))
    ang = torch.arange(T, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.stack([ang.cos(), ang.sin()], -1).float().cuda().contiguous()


print("case", [p.split("/")[-1] for p in sys.argv[1:]], "us; max|diff| vs first", flush=True)
for ctx in (190, 1024, 4096):
    for Q in (1, 5, 8, 11):
        B, H, Hkv, D = 16, 64, 8, 128
        T = ctx + Q + 8
        torch.manual_seed(0)
        L = max(2, min(40, int(4e9 // (B * Hkv * T * D * 4))))
        kcs = [torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
        vcs = [torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
        qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
        slot = torch.arange(B, dtype=torch.int32, device="cuda")
        start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
        tab = rope_table(T, D)
        res, outs = [], []
        wsb, wsc = None, None
        if os.environ.get("AB_WS") == "1":  # split over the cache length (scratch sized by the last build)
            b_, c_ = ctypes.c_int64(), ctypes.c_int()
            libs[-1].ms_attention_workspace_gqa(B, Q, H, Hkv, D, T, ctypes.byref(b_), ctypes.byref(c_))
            wsb = torch.empty(b_.value // 4 + 1, dtype=torch.float32, device="cuda")
            wsc = torch.zeros(c_.value, dtype=torch.int32, device="cuda")
        for lib in libs:
            out = torch.zeros(B * Q, H * D, device="cuda", dtype=torch.bfloat16)

            def run(i=0):
                st = torch.cuda.current_stream().cuda_stream
                assert lib.ms_attention_gqa(qkv.data_ptr(), qkv.stride(0), B, Q, H, Hkv, D, slot.data_ptr(),
                                            start.data_ptr(), T, kcs[i].data_ptr(), vcs[i].data_ptr(), tab.data_ptr(),
                                            D ** -0.5, 1, out.data_ptr(), out.stride(0),
                                            None if wsb is None else wsb.data_ptr(), 0 if wsb is None else wsb.numel() * 4,
                                            None if wsc is None else wsc.data_ptr(), 0 if wsc is None else wsc.numel(),
                                            st) == 0
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for i in range(L):
                    run(i)
                e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / L * 1e3)
            res.append(round(sorted(ts)[2], 1))
            outs.append(out.float())
        diffs = [round((o - outs[0]).abs().max().item(), 5) for o in outs[1:]]
        byts = B * Hkv * (ctx + Q) * D * 4
        print(f"ctx={ctx:5d} Q={Q:2d}", res, diffs, [f"{byts / t / 1e3:.0f} GB/s" for t in res], flush=True)
        del kcs, vcs
        torch.cuda.empty_cache()
