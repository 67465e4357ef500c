"""Same-process A/B of the 70B verify forward between two builds of
libminions (default: the session-start library of round 2's last leg, built
from commit 1e503a6 into lib/ab/) — one CUDA graph per (library, Q), captured
with kernels.py routed to that library, replays interleaved.
usage: python tools/verify_ab_lib.py [old.so] [Qs=5,7,9]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native
from paper_2402_15678_b200.llama import CONFIGS, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache

old_path = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] else os.path.join(os.path.dirname(_native.LIB_PATH), "ab", "libminions_r2start.so")
Qs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "5,7,9").split(",")]
old = ctypes.CDLL(old_path)
for name, args in _native._SIGS.items():
    if hasattr(old, name):
        fn = getattr(old, name)
        fn.argtypes = args
        fn.restype = _native._RESTYPE.get(name, ctypes.c_int)
new = _native.lib
c = CONFIGS["llama-2-70b"]
B, ctx = 16, 190
m = LlamaModel(LlamaWeights.random(c, 0), max_rows=B * max(Qs))
cache = KVCache(c, B, 512)
slot = torch.arange(B, dtype=torch.int32, device="cuda")
start = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
for Q in Qs:
    tok = torch.randint(0, c.vocab, (B, Q), dtype=torch.int32, device="cuda")
    logits = torch.empty(B * Q, c.vocab, device="cuda")
    graphs = {}
    for tag, lib in (("old", old), ("new", new)):
        _native.lib = lib
        for _ in range(2):
            m.forward(tok, start, slot, cache, logits)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            m.forward(tok, start, slot, cache, logits)
        graphs[tag] = g
    _native.lib = new
    res = {k: [] for k in graphs}
    for rep in range(4):
        for k, g in graphs.items():
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g.replay(); g.replay(); e1.record(); torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) / 2)
    print(json.dumps({"Q": Q, "M": B * Q, "verify_forward_ms": {k: round(min(v), 3) for k, v in res.items()},
                      "old_lib": os.path.basename(old_path)}), flush=True)
