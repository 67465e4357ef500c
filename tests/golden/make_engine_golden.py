"""Engine-level golden streams: the UNMODIFIED reference engine driven by fp32
CPU transformer oracles (SURVEY §8c golden #5, VERDICT r1 "next round" #1).

Run in the dev container, where the reference is importable:

    python tests/golden/make_engine_golden.py      # imports /root/reference/pkg/src

For each scenario it builds the cfg1 models (BASELINE.json configs[0]: tiny
OPT-style target, 4 layers, d=256, + 3 one-layer drafters; random init with
torch.manual_seed-style generators on the CPU, the exact weights the GPU tests
rebuild), wraps them as ModelOracles (oracle/model_oracle.py, exact fp32: the
fp32 verification-mode contract) and runs aggspec.run_sequential /
aggspec.run_pipelined (aggspec/engine.py:619-671; simulated clock, so the
selector sees the reference CostModel's t_llm) over make_requests-style
prompts (aggspec/bench.py:177-186).  Recorded per scenario:

  * the final token streams per request,
  * every verify event of the trace (request ids, s, accepted, emitted,
    voted, decision, s_next, weights — aggspec/engine.py:385-409),
  * every draft_sequence call's tokens, per (round of the request, drafter)
    — by wrapping aggspec.engine.draft_sequence with a recorder (the engine
    itself is not modified),
  * the smallest argmax margin (top-1 minus top-2 logit) any oracle call saw
    — the fp32 parity headroom, stated in the golden.

Modes: "greedy" (point-mass oracles, the fp32 verification mode's greedy
streams) and "sample" (softmax oracles: draft_sequence SAMPLES with each
request's draft/{rid}/{sid} stream and verify() runs speculative sampling
with verify/{rid} — the reference engine's stochastic path, which
SpecEngine(sampling=True) reproduces).

Scenarios: "random" = the configs[0] drafters verbatim (independent random
init: acceptance ~0, every round rolls the drafters back); "layerskip" =
drafter k is the target's embedding + its layer k (a random-init layer-skip
drafter: partial acceptance, exercises accept > 0, lcp rollback, weight
updates and selector moves).  Output: tests/golden/engine_streams.json.
"""
from __future__ import annotations

import json
import os
import re
import sys
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("AGGSPEC_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import aggspec.engine as ref_engine  # noqa: E402
from aggspec.core import EngineConfig, Request, seeded_rng  # noqa: E402
from aggspec.oracles import CostModel  # noqa: E402

from oracle.model_oracle import CPUModelOracle  # noqa: E402
from paper_2402_15678_b200.weights import CONFIGS, OPTWeights  # noqa: E402

COST = dict(c0=2.5, c1=0.1, d0=56.5, d1=0.75, d2=0.25)  # tests/test_acceptance.py:65 of the reference
N_REQ, NEW_TOKENS, SEED = 4, 64, 0


def build_models(kind: str):
    """cfg1 weights (bf16 values; the oracles compute in fp32)."""
    tc, sc = CONFIGS["tiny-target"], CONFIGS["tiny-ssm"]
    target = OPTWeights.random(tc, 0, device="cpu")
    if kind == "random":
        drafters = [OPTWeights.random(sc, k + 1, device="cpu") for k in range(3)]
    elif kind == "layerskip":
        drafters = []
        for k in range(3):
            t = {n: v.clone() for n, v in target.t.items() if not re.match(r"l\d+\.", n)}
            for n, v in target.t.items():
                if n.startswith(f"l{k}."):
                    t["l0." + n.split(".", 1)[1]] = v.clone()
            drafters.append(OPTWeights(sc, t))
    else:
        raise ValueError(kind)
    return target, drafters


def make_requests(vocab: int, seed: int = SEED) -> list[Request]:
    """aggspec/bench.py:177-186 with prompt_len U[4, 8] (cfg1)."""
    rng = seeded_rng(seed, "workload")
    out = []
    for i in range(N_REQ):
        n = int(rng.integers(4, 8 + 1))
        out.append(Request(id=f"req-{i:03d}", prompt=[int(t) for t in rng.integers(0, vocab, size=n)],
                           max_new_tokens=NEW_TOKENS))
    return out


def run(kind: str, schedule: str, adaptive: bool = True, mode: str = "greedy"):
    target, drafters = build_models(kind)
    tc = target.cfg
    llm = CPUModelOracle(target.t, tc, exact=True, mode=mode)
    ssms = [CPUModelOracle(w.t, w.cfg, exact=True, mode=mode) for w in drafters]
    b = N_REQ if schedule == "sequential" else N_REQ // 2
    cfg = EngineConfig(vocab_size=tc.vocab, b_llm=b, b_ssm=b, s_init=4, s_min=1, s_max=12,
                       initial_weights=(1.0, 1.0, 1.0), seed=SEED)
    reqs = make_requests(tc.vocab)
    prompts = {r.id: list(r.prompt) for r in reqs}
    drafts: dict = {}
    orig = ref_engine.draft_sequence

    def recording_draft_sequence(oracle, context, s, rng):
        toks, dists = orig(oracle, context, s, rng)
        sid = ssms.index(oracle)
        rid = next(r.id for r in reqs if list(r.prompt) + list(r.generated) == list(context))
        rounds = drafts.setdefault(rid, [])
        if sid == 0:  # _do_draft_batch drafts with ssm 0..K-1 in order per request
            rounds.append({})
        rounds[-1][sid] = [int(t) for t in toks]
        return toks, dists

    ref_engine.draft_sequence = recording_draft_sequence
    try:
        runner = ref_engine.run_sequential if schedule == "sequential" else ref_engine.run_pipelined
        t0 = time.time()
        metrics, trace = runner(reqs, ssms, llm, CostModel(**COST), cfg, adaptive=adaptive, clock="simulated")
        wall = time.time() - t0
    finally:
        ref_engine.draft_sequence = orig
    verify = [dict(round_index=e.round_index, request_ids=list(e.request_ids), s=e.s, accepted=list(e.accepted),
                   emitted=list(e.emitted), voted=list(e.voted), decision=e.decision, s_next=e.s_next,
                   weights={str(k): v for k, v in e.weights.items()})
              for e in trace if e.kind == "verify"]
    return dict(kind=kind, schedule=schedule, adaptive=adaptive, mode=mode, cost=COST,
                cfg=dict(b_llm=b, b_ssm=b, s_init=4, s_min=1, s_max=12, seed=SEED),
                prompts=prompts, outputs={r.id: list(r.generated) for r in reqs},
                verify=verify, drafts={rid: [[d[k] for k in sorted(d)] for d in v] for rid, v in drafts.items()},
                mean_accepted=float(np.mean([a for e in verify for a in e["accepted"]])),
                margin_min=min(o.min_margin for o in [llm] + ssms), oracle_calls=llm.calls + sum(o.calls for o in ssms),
                wall_s=round(wall, 1))


def main():
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    out = {"generator": "tests/golden/make_engine_golden.py", "reference": "aggspec (/root/reference/pkg/src)",
           "models": "cfg1: tiny-target (OPT 4L d256) + 3 x tiny-ssm (1L), weights OPTWeights.random(cfg, seed, "
                     "device='cpu') seeds 0 / 1..3 (std 0.02)",
           "scenarios": []}
    for mode in ("greedy", "sample"):
      for kind in ("random", "layerskip"):
        for schedule in ("sequential", "pipelined"):
            sc = run(kind, schedule, mode=mode)
            print(mode, kind, schedule, "rounds", len(sc["verify"]), "mean_acc", round(sc["mean_accepted"], 3),
                  "s_path", [v["s"] for v in sc["verify"]][:24], "margin", sc["margin_min"],
                  "wall", sc["wall_s"], flush=True)
            out["scenarios"].append(sc)
    with open(os.path.join(HERE, "engine_streams.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
