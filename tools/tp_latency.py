"""Latency of the tensor-parallel reduction protocol (csrc/tp.cu) per call,
two ranks as threads + streams of ONE process on one GPU.

One call = what a row-parallel layer output costs after its GEMM:
ms_tp_signal -> ms_tp_reduce_gather (rank-order sum of the fp32 partials,
bf16 all-gather) -> ms_tp_signal -> ms_rmsnorm_wait (70B: d = 8192).
Timed as CUDA-graph replays of 50 back-to-back calls per rank (both ranks'
graphs launched concurrently), so the number is device time per call.

(Two PROCESSES sharing one GPU cannot measure this: without MPS the GPU
time-slices between their contexts, so a spin-wait only completes after a
context switch — that is the 38.5 ms tiny-model verify of round 1's
gpurun_out/tpbench2.log, not the protocol's cost.)

usage: python tools/tp_latency.py > profiles/r2_tp_latency.jsonl
"""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2402_15678_b200.tp import TPComm

t, d, N = 2, 8192, 50
for R in (16, 80, 176):
    comms = TPComm.local_group(t, 256, d)
    gamma = torch.ones(d, dtype=torch.bfloat16, device="cuda")
    outs = [torch.empty(R, d, dtype=torch.bfloat16, device="cuda") for _ in range(t)]
    streams = [torch.cuda.Stream() for _ in range(t)]
    graphs = [torch.cuda.CUDAGraph() for _ in range(t)]

    def body(r, capture):
        try:
            _body(r, capture)
        except Exception as e:  # surface thread errors
            errs.append(e)

    errs = []

    def _body(r, capture):
        with torch.cuda.stream(streams[r]):
            if capture:
                with torch.cuda.graph(graphs[r], stream=streams[r], capture_error_mode="thread_local"):
                    for _ in range(N):
                        comms[r].allreduce_norm(R, gamma, 1e-5, outs[r])
            else:
                for _ in range(N):
                    comms[r].allreduce_norm(R, gamma, 1e-5, outs[r])
        streams[r].synchronize()

    def both(capture):
        th = [threading.Thread(target=body, args=(r, capture)) for r in range(t)]
        for x in th:
            x.start()
        for x in th:
            x.join(timeout=60)

    both(False)  # warm (eager)
    both(True)   # capture (no kernels run)
    if errs:
        raise errs[0]
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(t)]
    torch.cuda.synchronize()
    for rep in range(2):
        for r in range(t):
            with torch.cuda.stream(streams[r]):
                ev[r][0].record()
                graphs[r].replay()
                ev[r][1].record()
        torch.cuda.synchronize()
    for c in comms:
        c.check()
    us = max(e0.elapsed_time(e1) for e0, e1 in ev) * 1e3 / N
    byts = R * d * 4 * (t - 1) / t + R * d * 2 * (t - 1) / t  # per rank, peer reads + writes
    print(json.dumps({"t": t, "rows": R, "d": d, "us_per_allreduce_norm": round(us, 2),
                      "kernels_per_call": 4, "peer_bytes_per_rank": int(byts),
                      "mode": "2 ranks as threads+streams on one GPU, CUDA-graph replay of 50 calls"}), flush=True)
