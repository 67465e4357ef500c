"""Host bookkeeping of one verified round — the reference's _do_verify_batch
tail (aggspec/engine.py:297-330) over the device's per-request results.

Pure host code (no device, no libminions): SpecEngine calls it after reading
back a group's results, and the multi-rank tests drive it directly — in the
tensor-parallel engine every rank runs it on bitwise-identical device results
and a selector time made identical by `sync_time` (the max over ranks), so
every rank takes the same decisions without any other exchange.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import AggSpecError, EngineConfig, Request, RequestState
from .selector import Decision, MonitorSample, SelectorState, maybe_adjust, observe
from .voting import WeightTable, record_acr, update_weights


class NoProgress(AggSpecError):  # aggspec/engine.py:44
    pass


@dataclass
class RoundOutcome:
    accepted: list
    emitted: list
    voted: list
    vl: float
    decision: Decision
    s_next: int


def commit_round(requests: list[Request], ctx: list[list[int]], ssm_cached: list[list[int]], active: list[int],
                 s: int, n_acc, n_emit, emitted, voted, drafts, weights: WeightTable, selector: SelectorState,
                 cfg: EngineConfig, t_sel: float, rnd: int, adaptive: bool, finish_time=None) -> RoundOutcome:
    """Apply one round's device results (n_acc [B], n_emit [B], emitted [B, s+1],
    voted [B], drafts [B, K, s]) to the requests, the per-drafter cached
    lengths, the drafter weights and the selector:

      * use = emitted[:n_emit] (K9 already cut at remaining / the stop token),
        appended; FINISHED on the stop token or an exhausted budget
        (aggspec/engine.py:300-315);
      * record_acr(voted, accepted / s) per request, update_weights once per
        batch (aggspec/voting.py:142-170);
      * drafter k's cache stays valid up to lcp(drafts[b, k], use) (capped at
        s - 1 and len(use) - 1: the last context token is always re-fed);
      * observe(MonitorSample(t_llm=t_sel, vl=mean emitted)), maybe_adjust
        when adaptive (aggspec/selector.py:82-170)."""
    accs, ems, vts = [], [], []
    K = len(ssm_cached)
    for b in active:
        r = requests[b]
        r.advance(RequestState.AWAITING_VERIFICATION)
        acc = int(n_acc[b])
        use = [int(t) for t in emitted[b, : n_emit[b]]]
        record_acr(weights, int(voted[b]), acc / s)
        if len(use) == 0:
            raise NoProgress(f"request {r.id} made no progress")
        len_before = len(ctx[b])
        r.generated.extend(use)
        ctx[b].extend(use)
        stopped = cfg.stop_token is not None and cfg.stop_token in use
        if stopped or r.remaining <= 0:
            r.advance(RequestState.FINISHED)
            r.finish_time = finish_time
        else:
            r.advance(RequestState.RUNNING)
        for k in range(K):
            mlen = 0
            lim = min(s - 1, len(use) - 1)
            while mlen < lim and drafts[b, k, mlen] == use[mlen]:
                mlen += 1
            ssm_cached[k][b] = len_before + mlen
        accs.append(acc)
        ems.append(len(use))
        vts.append(int(voted[b]))
    update_weights(weights, cfg)
    vl = float(np.mean(ems)) if ems else 1.0
    observe(selector, MonitorSample(round_index=rnd, t_llm=t_sel, vl=vl, s_used=s))
    decision = Decision.HOLD
    if adaptive:
        _, decision = maybe_adjust(selector)
    return RoundOutcome(accs, ems, vts, vl, decision, selector.current_s)
