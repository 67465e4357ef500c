"""Trace events and run metrics in the reference's format
(TraceEvent / write_trace / RunMetrics / collect_metrics,
aggspec/engine.py:49-168), produced from the device engine's rounds with
MEASURED device time: every timestamp is milliseconds since the decode's
first kernel, read from CUDA events on the draft / verify streams — not the
reference's cost-model clock.

One speculation round of a request group yields a "draft" event (the K
drafters' s steps + vote + verifier-input pack) and a "verify" event (the
verify forward + greedy accept).  `collect_metrics` is the reference's
arithmetic verbatim (throughput, normalized latency, LLM utilisation,
per-SSM acceptance, weight and s trajectories).
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Sequence

import numpy as np


@dataclass
class TraceEvent:
    """One completed engine activity (aggspec/engine.py:49-90)."""

    seq: int
    kind: str  # "draft" | "verify"
    start: float
    end: float
    s: int
    request_ids: list
    pool_depth: int
    round_index: int | None = None
    accepted: list | None = None
    emitted: list | None = None
    voted: list | None = None
    vl: float | None = None
    decision: str | None = None
    s_next: int | None = None
    weights: dict | None = None

    def to_json(self) -> str:
        payload = {"seq": self.seq, "kind": self.kind, "start": self.start, "end": self.end, "s": self.s,
                   "request_ids": self.request_ids, "pool_depth": self.pool_depth}
        if self.kind == "verify":
            payload.update(round=self.round_index, accepted=self.accepted, emitted=self.emitted,
                           voted=self.voted, vl=self.vl, decision=self.decision, s_next=self.s_next,
                           weights=self.weights)
        return json.dumps(payload)


def write_trace(trace: Sequence[TraceEvent], path) -> None:
    with open(path, "w") as fh:
        for ev in trace:
            fh.write(ev.to_json())
            fh.write("\n")


@dataclass
class RunMetrics:
    """aggspec/engine.py:100-114 (times in ms of device time)."""

    total_time: float
    tokens_emitted: int
    throughput: float
    normalized_latency: float
    llm_busy_time: float
    ssm_busy_time: float
    llm_utilization: float
    llm_utilization_steady: float
    mean_acceptance: float
    per_ssm_acceptance: dict
    weight_trajectory: list
    s_trajectory: list


def collect_metrics(trace: Sequence[TraceEvent], requests) -> RunMetrics:
    """The reference's metric arithmetic (aggspec/engine.py:117-168)."""
    total_time = max((ev.end for ev in trace), default=0.0)
    tokens = sum(len(r.generated) for r in requests)
    throughput = tokens / (total_time / 1000.0) if total_time > 0 else 0.0
    latencies = []
    for r in requests:
        if len(r.generated) == 0:
            continue
        finish = r.finish_time if r.finish_time is not None else total_time
        latencies.append((finish - r.arrival_time) / len(r.generated))
    normalized_latency = float(np.mean(latencies)) if latencies else 0.0
    llm_busy = sum(ev.end - ev.start for ev in trace if ev.kind == "verify")
    ssm_busy = sum(ev.end - ev.start for ev in trace if ev.kind == "draft")
    llm_util = llm_busy / total_time if total_time > 0 else 0.0
    verify_events = [ev for ev in trace if ev.kind == "verify"]
    if verify_events:
        window = max(ev.end for ev in verify_events) - min(ev.start for ev in verify_events)
        llm_util_steady = llm_busy / window if window > 0 else 1.0
    else:
        llm_util_steady = 0.0
    rates: dict = {}
    all_rates: list = []
    weight_traj, s_traj = [], []
    for ev in verify_events:
        for voted, acc in zip(ev.voted, ev.accepted):
            r = acc / ev.s
            rates.setdefault(voted, []).append(r)
            all_rates.append(r)
        weight_traj.append((ev.round_index, dict(ev.weights)))
        s_traj.append((ev.round_index, ev.s_next))
    per_ssm = {k: float(np.mean(v)) for k, v in sorted(rates.items(), key=lambda kv: str(kv[0]))}
    mean_acc = float(np.mean(all_rates)) if all_rates else 0.0
    return RunMetrics(total_time=total_time, tokens_emitted=tokens, throughput=throughput,
                      normalized_latency=normalized_latency, llm_busy_time=llm_busy, ssm_busy_time=ssm_busy,
                      llm_utilization=llm_util, llm_utilization_steady=llm_util_steady, mean_acceptance=mean_acc,
                      per_ssm_acceptance=per_ssm, weight_trajectory=weight_traj, s_trajectory=s_traj)


def trace_from_rounds(rounds) -> list[TraceEvent]:
    """Device-timed TraceEvents of an engine run (RoundStats with timestamps)."""
    evs = []
    for rd in rounds:
        if rd.draft_start is None:
            continue
        evs.append(TraceEvent(seq=0, kind="draft", start=rd.draft_start, end=rd.draft_end, s=rd.s,
                              request_ids=list(rd.request_ids), pool_depth=rd.pool_depth))
        evs.append(TraceEvent(seq=0, kind="verify", start=rd.verify_start, end=rd.verify_end, s=rd.s,
                              request_ids=list(rd.request_ids), pool_depth=rd.pool_depth,
                              round_index=rd.round_index, accepted=list(rd.accepted), emitted=list(rd.emitted),
                              voted=list(rd.voted), vl=rd.vl, decision=rd.decision, s_next=rd.s_next,
                              weights=dict(rd.weights)))
    evs.sort(key=lambda e: (e.end, e.kind != "draft"))
    for i, e in enumerate(evs):
        e.seq = i
    return evs
