"""cfg4 of BASELINE.json — vote + verify microbench sweep: SSM count K 1-8,
speculation length s 1-16, batch B 1-256 (V = 32,000, Llama vocabulary).

Per cell, on the device (CUDA events over a CUDA-graph replay of 50 calls,
inputs resident in HBM):
  vote    ms_vote (K4) over drafts [B, K, s]           bytes = 4BKs + 8K + 4B(s+1)
  accept  ms_accept_greedy_logits (K8 + K9) over fp32 target logits [B, s+1, V]
          bytes = 4 B (s+1) V + 4Bs + 4B(s+2)  -> GB/s against HBM
Checked against the oracle (oracle/aggspec_oracle.py, the CPU restatement of
merge/select_majority/verify) on every cell; the reference's own CPU loop
(oracle port, one Python thread) is timed beside it on a bounded sample.
Multi-GPU: vote/accept shard by request — per-GPU numbers at
B/N requests are the per-rank cost; no collective.

usage: python tools/vote_verify_sweep.py [--quick] > profiles/cfg4_sweep.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import aggspec_oracle as O
from paper_2402_15678_b200 import _native

V = 32000


def timed(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps  # us per call


def cell(K, s, B, rng, peak):
    tok = torch.tensor(rng.integers(0, 6, size=(B, K, s)).astype(np.int32), device="cuda")
    w = torch.tensor(1.25 ** rng.integers(-3, 4, size=K), dtype=torch.float64, device="cuda")
    path = torch.zeros(B, s, dtype=torch.int32, device="cuda")
    voted = torch.zeros(B, dtype=torch.int32, device="cuda")
    logits = torch.randn(B, s + 1, V, device="cuda")
    rem = torch.full((B,), 1000, dtype=torch.int32, device="cuda")
    tgt = torch.zeros(B * (s + 1), dtype=torch.int32, device="cuda")
    ws = torch.zeros(B * (s + 1), dtype=torch.int64, device="cuda")
    n_acc, n_emit, fin = (torch.zeros(B, dtype=torch.int32, device="cuda") for _ in range(3))
    emitted = torch.zeros(B, s + 1, dtype=torch.int32, device="cuda")

    def vote():
        _native.call("ms_vote", tok.data_ptr(), w.data_ptr(), None, B, K, s, path.data_ptr(), voted.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)

    def accept():
        _native.call("ms_accept_greedy_logits", path.data_ptr(), logits.data_ptr(), 0, V, rem.data_ptr(), -1, B, s,
                     tgt.data_ptr(), ws.data_ptr(), n_acc.data_ptr(), emitted.data_ptr(), n_emit.data_ptr(),
                     fin.data_ptr(), None, torch.cuda.current_stream().cuda_stream)

    t_vote = timed(vote)
    t_acc = timed(accept)
    # parity against the oracle on this cell
    p_ref, v_ref = O.vote_batch(tok.cpu().numpy(), w.cpu().numpy())
    assert np.array_equal(path.cpu().numpy(), p_ref) and np.array_equal(voted.cpu().numpy(), v_ref)
    t_ref = logits.argmax(-1).to(torch.int32).cpu().numpy()
    a_ref, e_ref, ne_ref, _ = O.accept_greedy_batch(p_ref, t_ref, rem.cpu().numpy(), None)
    assert np.array_equal(n_acc.cpu().numpy(), a_ref) and np.array_equal(emitted.cpu().numpy(), e_ref)
    # reference CPU loop (oracle port, one thread) on a bounded sample of requests
    nb = min(B, 16)
    tk, wn, lg = tok.cpu().numpy(), w.cpu().numpy(), t_ref
    t0 = time.perf_counter()
    for b in range(nb):
        pth, _ = O.vote_one(tk[b], wn)
        O.verify_greedy_one(pth, lg[b])
    t_cpu = (time.perf_counter() - t0) / nb * B * 1e6
    vb = 4 * B * K * s + 8 * K + 4 * B * (s + 1)
    ab = 4 * B * (s + 1) * V + 4 * B * s + 4 * B * (s + 2)
    return {"K": K, "s": s, "B": B, "vote_us": round(t_vote, 2), "vote_bytes": vb,
            "accept_us": round(t_acc, 2), "accept_bytes": ab, "accept_gbs": round(ab / t_acc / 1e3, 1),
            "accept_frac_hbm": round(ab / t_acc / 1e3 / peak, 3),
            "cpu_ref_us": round(t_cpu, 1), "cpu_ref_note": "oracle port vote+greedy verify loop, 1 thread "
                                                         "(logit argmax excluded)", "parity": "ok"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    peak = 6650.0
    try:
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    rng = np.random.default_rng(0)
    Ks = [1, 3, 8] if a.quick else [1, 2, 3, 5, 8]
    ss = [1, 4, 16] if a.quick else [1, 2, 4, 8, 12, 16]
    Bs = [1, 16, 256] if a.quick else [1, 4, 16, 64, 256]
    for K in Ks:
        for s in ss:
            for B in Bs:
                print(json.dumps(cell(K, s, B, rng, peak)), flush=True)


if __name__ == "__main__":
    main()
