"""Ablation in the structure of the paper's Fig. 8,
on MEASURED device time instead of the reference's cost model
(aggspec/bench.py:255-268 runs the same ladder on its simulated clock):

  default      one drafter, fixed s = 4, sequential      (plain speculative decoding)
  +majority    K drafters + weighted majority vote, fixed s = 4
  +selector    + adaptive speculation length (maybe_adjust)
  +pipeline    + pipelined drafting / verification (two request groups)

Prints one JSON line per variant: output tokens/s (decode, CUDA events),
mean accepted length, and the reference's RunMetrics computed from the
device-timed trace (trace.collect_metrics).  Writes each variant's trace
JSONL next to --out.
usage: python tools/ablation.py [--target llama-2-70b] [--ssm llama-160m] [--out profiles/ablation]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2402_15678_b200.core import EngineConfig
from paper_2402_15678_b200.engine import SpecEngine
from paper_2402_15678_b200.models import config, random_weights
from paper_2402_15678_b200.trace import write_trace


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--target", default="llama-2-70b")
    ap.add_argument("--ssm", default="llama-160m")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--new-tokens", type=int, default=128)
    ap.add_argument("--fidelity", default="0.9,0.85,0.8")
    ap.add_argument("--out", default="gpurun_out/ablation")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    tcfg, scfg = config(a.target), config(a.ssm)
    fid = [float(x) for x in a.fidelity.split(",")]
    target = random_weights(tcfg, 0)
    drafters = [random_weights(scfg, k + 1) for k in range(len(fid))]
    variants = [("default", 1, False, False), ("+majority", len(fid), False, False),
                ("+selector", len(fid), True, False), ("+pipeline", len(fid), True, True)]
    for name, K, adaptive, pipelined in variants:
        cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=a.batch, b_ssm=a.batch, s_init=4, s_min=1, s_max=12,
                           initial_weights=(1.0,) * K, seed=0)
        n_req = a.batch * (2 if pipelined else 1)
        max_len = 128 + a.new_tokens + cfg.s_max + 4
        eng = SpecEngine(target, drafters[:K], cfg, slots=n_req, max_len=max_len, fidelity=fid[:K],
                         pipelined=pipelined, adaptive=adaptive)
        eng.capture_graphs()
        reqs = bench.make_requests(n_req, 128, a.new_tokens, tcfg.vocab)
        teacher = eng.greedy_teacher(bench.fresh(reqs), a.new_tokens)
        for _ in range(2):  # warm-up (selector / weights adapt, as in the bench)
            eng.prefill(bench.fresh(reqs))
            eng.set_teacher(teacher)
            eng.decode()
        rs = bench.fresh(reqs)
        eng.prefill(rs)
        eng.set_teacher(teacher)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        res = eng.decode()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        m = res.metrics(rs)
        write_trace(res.trace(), f"{a.out}_{name.strip('+')}.jsonl")
        print(json.dumps({"variant": name, "drafters": K, "adaptive": adaptive, "pipelined": pipelined,
                          "requests": n_req, "tokens_per_s": round(res.tokens / t, 1),
                          "mean_accepted_length": round(res.mean_accepted, 3),
                          "lossless_vs_greedy": res.outputs == teacher,
                          "trace_throughput": round(m.throughput, 1), "llm_utilization": round(m.llm_utilization, 3),
                          "mean_acceptance": round(m.mean_acceptance, 4),
                          "per_ssm_acceptance": {str(k): round(v, 4) for k, v in m.per_ssm_acceptance.items()},
                          "final_s": m.s_trajectory[-1][1] if m.s_trajectory else None}), flush=True)
        del eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
