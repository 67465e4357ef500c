"""A/B of ms_attention_gqa between two builds of libminions (raw ctypes, so
an older ABI works): python tools/attn_ab.py lib_a.so lib_b.so"""
import ctypes, sys
import torch
P, I, I64, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
libs = [ctypes.CDLL(p) for p in sys.argv[1:]]
for lib in libs:
    lib.ms_attention_gqa.argtypes = [P, I64, I, I, I, I, I, P, P, I, P, P, P, F, I, P, I64, P, I64, P, I, P]
for name, B, Q, H, Hkv, D, ctx in (("70b ctx190", 16, 11, 64, 8, 128, 190), ("70b ctx1k", 16, 11, 64, 8, 128, 1024),
                                  ("160m ctx200", 48, 1, 12, 12, 64, 200)):
    T = ctx + Q + 8
    kc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
    vc = torch.randn(B, Hkv, T, D, device="cuda").to(torch.bfloat16)
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
    slot = torch.arange(B, dtype=torch.int32, device="cuda")
    start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    out = torch.empty(B * Q, H * D, device="cuda", dtype=torch.bfloat16)
    res = []
    for li, lib in enumerate(libs):
        def run():
            st = torch.cuda.current_stream().cuda_stream
            assert lib.ms_attention_gqa(qkv.data_ptr(), qkv.stride(0), B, Q, H, Hkv, D, slot.data_ptr(),
                                        start.data_ptr(), T, kc.data_ptr(), vc.data_ptr(), None, D ** -0.5, 1,
                                        out.data_ptr(), out.stride(0), None, 0, None, 0, st) == 0
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(20):
                run()
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 20 * 1e3)
        res.append(round(sorted(ts)[2], 1))
    print(name, res, flush=True)
