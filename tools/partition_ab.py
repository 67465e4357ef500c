"""A/B of pipelined-schedule placement options on the bench workload (cfg3:
Llama-2-70B + 3 x Llama-160M, two groups of 16, fidelity injection), in one
process, arms interleaved so clock drift hits every arm alike.  An arm is a
comma list of SpecEngine options: draft_sms=N (SM partition, csrc/
partition.cu), draft_pdl=0|1 (programmatic dependent launch of the drafter
kernels), draft_coresident=0|1, gated_persistent=0|1 (gate/up schedule,
ms_set_gated_persistent), stream_priority=0|1|2 (equal / verify / draft
high), tc_attention=0|1|2 (kernels.TC_ATTENTION False / True / "auto").
usage: python tools/partition_ab.py ["draft_sms=0;draft_sms=16;draft_pdl=0"] [fixed_s=6] [reps=2] [new_tokens=128]
prints one JSON line per (rep, arm)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2402_15678_b200.core import EngineConfig
from paper_2402_15678_b200.engine import SpecEngine
from paper_2402_15678_b200.models import config, make_model, random_weights

arms = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in a.split(",") if kv)
        for a in (sys.argv[1] if len(sys.argv) > 1 else "draft_sms=0;draft_sms=16;draft_pdl=0").split(";")]
fixed_s = int(sys.argv[2]) if len(sys.argv) > 2 else 6
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
new_tokens = int(sys.argv[4]) if len(sys.argv) > 4 else 128
tcfg, scfg = config("llama-2-70b"), config("llama-160m")
fid = [0.9, 0.85, 0.8]
cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=16, b_ssm=16, s_init=fixed_s or 4, s_min=1, s_max=12,
                   initial_weights=(1.0,) * 3, seed=0)
max_len = 128 + new_tokens + cfg.s_max + 4
tw = random_weights(tcfg, 0)
target = make_model(tw, max_rows=max(32 * (cfg.s_max + 1), 32 * max_len))
drafters = [random_weights(scfg, k + 1) for k in range(3)]
reqs = bench.make_requests(32, 128, new_tokens, tcfg.vocab)
teacher = None
for rep in range(reps):
    for arm in arms:
        kw = {"draft_sms": arm.get("draft_sms", 0), "draft_pdl": bool(arm.get("draft_pdl", 1)),
              "stream_priority": ("equal", "verify", "draft")[arm.get("stream_priority", 0)],
              "draft_coresident": bool(arm["draft_coresident"]) if "draft_coresident" in arm else None}
        from paper_2402_15678_b200 import _native
        _native.lib.ms_set_gated_persistent(arm.get("gated_persistent", 1))  # baked into the captured graphs
        from paper_2402_15678_b200 import kernels as _K
        if "tc_attention" in arm:  # 0: row kernel, 1: tcgen05 everywhere, 2: auto (by cache length)
            _K.TC_ATTENTION = {0: False, 1: True, 2: "auto"}[arm["tc_attention"]]
        eng = SpecEngine(target, drafters, cfg, slots=32, max_len=max_len, fidelity=fid, pipelined=True,
                         adaptive=not fixed_s, **kw)
        eng.capture_graphs()
        # the greedy teacher of this arm's kernels (arms that change the target's
        # arithmetic, e.g. tc_attention, have their own greedy continuation)
        teacher = eng.greedy_teacher(bench.fresh(reqs), new_tokens)
        out = []
        for it in range(3):
            rs = bench.fresh(reqs)
            eng.prefill(rs)
            eng.set_teacher(teacher)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            res = eng.decode()
            e1.record()
            torch.cuda.synchronize()
            if it == 0:
                continue  # warm-up
            out.append((res.tokens / (e0.elapsed_time(e1) * 1e-3), res))
        tps = sum(o[0] for o in out) / len(out)
        rounds = [rd for _, r in out for rd in r.rounds]
        print(json.dumps({"rep": rep, "arm": arm, "got_sms": [eng.draft_sms, eng.verify_sms],
                          "fixed_s": fixed_s, "tokens_per_s": round(tps, 1),
                          "lossless": all(r.outputs == teacher for _, r in out),
                          "verify_ms": round(sum(r.t_verify_ms for r in rounds) / len(rounds), 3),
                          "draft_ms": round(sum(r.t_draft_ms for r in rounds) / len(rounds), 3),
                          "mean_s": round(sum(r.s for r in rounds) / len(rounds), 2)}), flush=True)
        del eng
        torch.cuda.empty_cache()
