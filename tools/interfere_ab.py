"""Where does drafting slow the verifier down?  70B verify forward (B = 16,
Q = 7, ctx 190, T = 272) alone and concurrently with (a) the grouped
3 x Llama-160M catch-up step (qc rows per request, head rows only, the
pipelined engine's draft step 0) and (b) five co-resident decode steps
(steps 1..5), each on its own stream, all as CUDA graphs; device ms.
usage: python tools/interfere_ab.py [qc=7] [reps=5]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_15678_b200 import _native
from paper_2402_15678_b200.llama import CONFIGS, GroupedLlamaModel, LlamaModel, LlamaWeights
from paper_2402_15678_b200.opt import KVCache

qc = int(sys.argv[1]) if len(sys.argv) > 1 else 7
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
B, Q, ctx, T, G = 16, 7, 190, 272, 3
tc = CONFIGS["llama-2-70b"]
tgt = LlamaModel(LlamaWeights.random(tc, 0), max_rows=B * Q)
tcache = KVCache(tc, B, T)
ttok = torch.randint(0, tc.vocab, (B, Q), dtype=torch.int32, device="cuda")
tstart = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
tslot = torch.arange(B, dtype=torch.int32, device="cuda")
tlog = torch.empty(B * Q, tc.vocab, device="cuda")
sc = CONFIGS["llama-160m"]
dm = GroupedLlamaModel([LlamaWeights.random(sc, k + 1) for k in range(G)], max_rows=B * 16)
dcache = KVCache(sc, G * B, T)
dslot = torch.arange(G * B, dtype=torch.int32, device="cuda")
ctok = torch.randint(0, sc.vocab, (G * B, qc), dtype=torch.int32, device="cuda")
cstart = torch.full((G * B,), ctx - qc, dtype=torch.int32, device="cuda")
chead = (torch.arange(G * B, device="cuda") * qc + qc - 1).to(torch.int32)
stok = torch.randint(0, sc.vocab, (G * B, 1), dtype=torch.int32, device="cuda")
sstart = torch.full((G * B,), ctx, dtype=torch.int32, device="cuda")
dlog = torch.empty(G * B * qc, sc.vocab, device="cuda")

def verify():
    tgt.forward(ttok, tstart, tslot, tcache, tlog)

def catchup():
    dm.forward(ctok, cstart, dslot, dcache, dlog, head_rows=chead)

def decode():
    co = _native.lib.ms_set_coresident(1)
    dm.coresident = True
    try:
        for _ in range(5):
            dm.forward(stok, sstart, dslot, dcache, dlog[: G * B])
    finally:
        _native.lib.ms_set_coresident(co)
        dm.coresident = False

graphs = {}
for name, f in (("verify", verify), ("catchup", catchup), ("decode5", decode)):
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    graphs[name] = g
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timed(names):
    ev = {n: (torch.cuda.Event(True), torch.cuda.Event(True)) for n in names}
    torch.cuda.synchronize()
    for n, st in zip(names, (s1, s2)):
        with torch.cuda.stream(st):
            ev[n][0].record(); graphs[n].replay(); ev[n][1].record()
    torch.cuda.synchronize()
    return {n: e0.elapsed_time(e1) for n, (e0, e1) in ev.items()}

arms = [("verify",), ("catchup",), ("decode5",), ("verify", "catchup"), ("verify", "decode5")]
res = {a: [] for a in arms}
for r in range(reps + 1):
    for a in arms:
        t = timed(a)
        if r:
            res[a].append(t)
out = {"qc": qc}
for a, ts in res.items():
    for n in a:
        v = sorted(t[n] for t in ts)
        out["+".join(a) + ":" + n] = round(v[len(v) // 2], 3)
print(json.dumps(out), flush=True)
