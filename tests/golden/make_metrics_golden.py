"""Golden vector for trace.collect_metrics: the reference's collect_metrics
(aggspec/engine.py:117-168) on a fixed synthetic trace.  Run in the build
container (imports the reference from /root/reference/pkg/src):
    python tests/golden/make_metrics_golden.py"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from aggspec.core import Request  # noqa: E402
from aggspec.engine import TraceEvent, collect_metrics  # noqa: E402


def synthetic():
    evs, seq, t = [], 0, 0.0
    w = {0: 1.0, 1: 1.0, 2: 1.0}
    for rnd in range(6):
        s = 3 + rnd % 3
        evs.append(TraceEvent(seq, "draft", t, t + 1.5 + 0.1 * rnd, s, ["req-000", "req-001"], 0))
        seq += 1
        t += 1.5 + 0.1 * rnd
        acc = [rnd % (s + 1), (rnd * 2) % (s + 1)]
        w = {k: v * (1.25 if k == rnd % 3 else 1.0) for k, v in w.items()}
        evs.append(TraceEvent(seq, "verify", t, t + 4.0, s, ["req-000", "req-001"], 1, rnd, acc,
                              [a + 1 for a in acc], [rnd % 3, (rnd + 1) % 3], 2.5, "hold", s, dict(w)))
        seq += 1
        t += 4.0
    reqs = [Request("req-000", [1, 2], 20), Request("req-001", [3], 20)]
    reqs[0].generated = list(range(11))
    reqs[1].generated = list(range(7))
    reqs[0].finish_time = 30.0
    return evs, reqs


evs, reqs = synthetic()
m = collect_metrics(evs, reqs)
out = {"events": [json.loads(e.to_json()) for e in evs],
       "requests": [{"id": r.id, "generated": r.generated, "finish_time": r.finish_time} for r in reqs],
       "metrics": {k: getattr(m, k) for k in ("total_time", "tokens_emitted", "throughput", "normalized_latency",
                                              "llm_busy_time", "ssm_busy_time", "llm_utilization",
                                              "llm_utilization_steady", "mean_acceptance")},
       "per_ssm_acceptance": {str(k): v for k, v in m.per_ssm_acceptance.items()},
       "s_trajectory": m.s_trajectory}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "metrics_golden.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print("ok")
