"""Speculate-vote-verify runtime on one B200: the device form of
SpeculationEngine._do_draft_batch / _do_verify_batch (aggspec/engine.py:252-330)
and of its two schedules, sequential and pipelined (aggspec/engine.py:337-342,
494-576).

One round of a request group, entirely on the device (two CUDA graphs per
(s, Qc): draft and verify):

  for each SSM k (K drafters, own weights + KV cache, own stream):
      step 0   catch-up forward of the Qc context tokens the SSM has not cached
               (rollback: an SSM's cache is valid only up to its longest prefix
               agreement with the emitted tokens), logits of the last row
      step j   one-token decode of its previous draft           (K1/K2/K7)
      argmax + draft_commit -> drafts[B, K, s]                   (K3)
  vote (fp64 weights, reference tie rules) -> path[B, s], voted  (K4)
  pack [last token | path] -> verify forward of s+1 rows          (K5/K6/K7)
  LM head logits -> argmax -> greedy accept + commit              (K8/K9)

then one device->host copy of the group's results, after which the host
replays the reference's bookkeeping verbatim: record_acr / update_weights
(fp64), the Request lifecycle, the remaining-budget / stop-token commit and the
adaptive speculation length (observe / maybe_adjust) fed with the MEASURED
verify time (CUDA events), not a cost model.

Schedules:
  sequential  one group holding every slot: draft, then verify, per round.
  pipelined   two groups (the reference's pool of depth b_llm, throttle
              len(pool) < b_llm): while the LLM verifies group A on the verify
              stream, the drafters draft group B on the draft stream; each
              phase ends with the verified group's results on the host.
              Weights are snapshotted at draft start, so a vote may use weights
              one verify stale — the reference's pipelined semantics.

KV rollback is length arithmetic: the LLM's cache is valid for the first
len(context) - 1 positions (the verify forward rewrites the rest), an SSM's for
len(context_before_round) + lcp(its draft, emitted) positions.
"""
from __future__ import annotations

import ctypes
import time
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev
from . import _native
from .core import AggSpecError, EngineConfig, Request, RequestState, seeded_rng, validate_config

from .llama import GroupedLlamaModel
from .models import make_model
from .opt import KVCache
from .rounds import NoProgress, commit_round  # noqa: F401  (NoProgress: public name)
from .selector import SelectorState
from .verification import AcceptOut, peek_uniforms
from .voting import WeightTable

I32 = torch.int32


class EngineFinished(AggSpecError):  # aggspec/engine.py:37
    pass


class DeadlockError(AggSpecError):  # aggspec/engine.py:41
    pass


@dataclass
class RoundStats:
    s: int
    qc: int
    t_verify_ms: float
    t_round_ms: float
    t_draft_ms: float
    accepted: list
    emitted: list
    voted: list
    vl: float
    decision: str
    s_next: int
    weights: dict
    group: int = 0
    trace: dict | None = None  # per-round device arrays when record=True
    # device timestamps (ms since the decode's first kernel) for the trace
    round_index: int = 0
    request_ids: tuple = ()
    pool_depth: int = 0
    draft_start: float | None = None
    draft_end: float | None = None
    verify_start: float | None = None
    verify_end: float | None = None


@dataclass
class RunResult:
    outputs: dict                     # request id -> generated tokens
    rounds: list = field(default_factory=list)
    tokens: int = 0
    wall_s: float = 0.0

    @property
    def mean_accepted(self) -> float:
        acc = [a for r in self.rounds for a in r.accepted]
        return float(np.mean(acc)) if acc else 0.0

    @property
    def mean_emitted(self) -> float:
        em = [e for r in self.rounds for e in r.emitted]
        return float(np.mean(em)) if em else 0.0

    def trace(self):
        """Device-timed TraceEvents in the reference's format (trace.py)."""
        from .trace import trace_from_rounds
        return trace_from_rounds(self.rounds)

    def metrics(self, requests):
        """RunMetrics (aggspec/engine.py:100-168) from the device-timed trace;
        request finish times are the device end of their last verify."""
        from .trace import collect_metrics
        return collect_metrics(self.trace(), requests)


class _Group:
    """Per-group device buffers (one pinned upload / one download per round),
    host request state and the drafts awaiting verification.  Slots
    [slot0, slot0 + B)."""

    def __init__(self, eng: "SpecEngine", gid: int, slot0: int, B: int):
        self.gid, self.slot0, self.B = gid, slot0, B
        dev, K, s_cap, V = eng.dev, eng.K, eng.cfg.s_max, eng.V
        z = lambda *sh: torch.zeros(sh, dtype=I32, device=dev)  # noqa: E731
        sizes = [("w", 2 * K)]
        if eng.sampling:  # fp64 uniforms (even int32 offsets: right after the fp64 weights)
            sizes += [("u_draft", 2 * K * B * s_cap), ("u_verify", 2 * B * (s_cap + 1))]
        sizes += [("ctx_len", B), ("c_start", B), ("c_head", B), ("v_start", B),
                  ("last", B), ("remaining", B), ("step_start", s_cap * B), ("c_tok", B * (s_cap + 1))]
        if eng.grouped:  # the drafters' inputs replicated per row group (drafter)
            sizes += [("g_c_start", K * B), ("g_c_head", K * B), ("g_step_start", s_cap * K * B),
                      ("g_c_tok", K * B * (s_cap + 1))]
        self.meta, self.meta_h, self.meta_off = self._packed(sizes, dev)
        mv = lambda n: self.meta[self.meta_off[n][0]: sum(self.meta_off[n])]  # noqa: E731
        if eng.grouped:
            self.g_c_start, self.g_c_head = mv("g_c_start"), mv("g_c_head")
            self.g_step_start = mv("g_step_start").view(s_cap, K * B)
            self.g_c_tok = mv("g_c_tok")
            self.g_slot = torch.tensor([k * eng.B + slot0 + b for k in range(K) for b in range(B)], dtype=I32,
                                       device=dev)
            self.g_step_tok = z(K * B, 1)
            self.g_argmax = z(K * B)
            self.g_ws = torch.zeros(K * B, dtype=torch.int64, device=dev)
            self.g_logits = torch.empty(K * B, V, device=dev)
        self.w_dev = mv("w").view(torch.float64)
        if eng.sampling:
            # stochastic drafting / verification (K3 stochastic + K10): per-round
            # uniforms of the reference's per-request streams, the K drafters'
            # distributions [K, B, s, V] (kept for the verifier), the voted
            # drafter's [B, s, V], the target's [B, s+1, V], K10 scratch
            self.u_draft = mv("u_draft").view(torch.float64)    # [K*B, s_cap]
            self.u_verify = mv("u_verify").view(torch.float64)  # [B, s+1] compact per round
            f64 = lambda *sh: torch.zeros(sh, dtype=torch.float64, device=dev)  # noqa: E731
            self.q = f64(K * B * s_cap * V)
            self.qv = f64(B * s_cap * V)
            self.o = f64(B * (s_cap + 1) * V)
            self.k10_scratch = f64(B * V)
        self.ctx_len, self.c_start, self.c_head = mv("ctx_len"), mv("c_start"), mv("c_head")
        self.v_start, self.last, self.remaining = mv("v_start"), mv("last"), mv("remaining")
        self.step_start = mv("step_start").view(s_cap, B)
        self.c_tok = mv("c_tok")
        rsz = [("n_acc", B), ("n_emit", B), ("finished", B), ("voted", B), ("n_draws", B),
               ("emitted", B * (s_cap + 1)), ("tgt", B * (s_cap + 1)), ("drafts", B * K * s_cap),
               ("path", B * s_cap)]
        self.res, self.res_h, self.res_off = self._packed(rsz, dev)
        rv = lambda n: self.res[self.res_off[n][0]: sum(self.res_off[n])]  # noqa: E731
        self.drafts, self.path, self.voted = rv("drafts"), rv("path"), rv("voted")
        self.n_draws = rv("n_draws")
        self.acc = AcceptOut(rv("n_acc"), rv("emitted"), rv("n_emit"), rv("finished"), rv("tgt"))
        self.slot = torch.arange(slot0, slot0 + B, dtype=I32, device=dev)
        self.req_key = z(B)
        self.step_tok = [z(B, 1) for _ in range(K)]
        self.argmax = [z(B) for _ in range(K)]
        self.ssm_ws = [torch.zeros(B, dtype=torch.int64, device=dev) for _ in range(K)]
        self.ssm_logits = [torch.empty(B, V, device=dev) for _ in range(K)]
        self.argmax_ws = torch.zeros(B * (s_cap + 1), dtype=torch.int64, device=dev)
        self.vin = z(B, s_cap + 1)
        self.v_logits = torch.empty(B * (s_cap + 1), eng.Vt, device=dev)  # target's vocab slice
        self.ev_d0 = torch.cuda.Event(enable_timing=True)
        self.ev_d1 = torch.cuda.Event(enable_timing=True)
        self.ev_v0 = torch.cuda.Event(enable_timing=True)
        self.ev_v1 = torch.cuda.Event(enable_timing=True)
        self.ev_res = torch.cuda.Event()
        self.K = K
        # host state
        self.requests: list[Request] = []
        self.ctx: list[list[int]] = []
        self.ssm_cached: list[list[int]] = []
        self.pending = None  # (s, qc, active, t_start) of drafts awaiting verification
        self.prev_states: list = []  # request states before the pending draft (discard)

    @staticmethod
    def _packed(sizes, dev):
        n = sum(m for _, m in sizes)
        off, o = {}, 0
        for name, m in sizes:
            off[name] = (o, m)
            o += m
        return (torch.zeros(n, dtype=I32, device=dev), torch.zeros(n, dtype=I32, pin_memory=True), off)

    def drafts_s(self, s):
        # drafts buffer viewed as [B, K, s] contiguous (the first B*K*s ints)
        return self.drafts[: self.B * self.K * s].view(self.B, self.K, s)

    def active(self):
        return [b for b, r in enumerate(self.requests) if r.state != RequestState.FINISHED]


class SpecEngine:
    """Greedy speculative decoding with K voting drafters on one GPU."""

    PREFILL_CHUNK = 1024  # prompt positions per prefill forward

    def __init__(self, target, drafters: list, cfg: EngineConfig,
                 slots: int, max_len: int, device="cuda", use_graphs: bool = True,
                 fidelity: list[float] | None = None, inject_seed: int = 0, adaptive: bool = True,
                 record: bool = False, pipelined: bool = False, sync_time=None,
                 kv_block_size: int = 0, kv_blocks: int | None = None, precision: str = "bf16",
                 selector_time: str = "verify", sim_cost=None, sampling: bool = False,
                 draft_sms: int = 0, draft_pdl: bool = True, draft_coresident: bool | None = None,
                 grouped_drafters: bool = True, stream_priority: str = "equal"):
        """target: weights (a model is built here) or a prebuilt model — e.g. a
        tp.LlamaTPModel rank, whose forward yields its vocab slice and whose
        argmax() combines across ranks.  sync_time(ms) -> ms: makes the
        selector's verify time identical on every rank (tensor parallel: every
        rank must take the same decisions); None = local time.
        kv_block_size > 0: the verifier's KV cache is paged (paged.PagedKVCache,
        kv_blocks pool blocks; default = slots x max_len worth): blocks are
        grown before each round and the blocks past the accepted length —
        the KV of rejected speculative tokens — are freed after it.
        precision "fp32": the fp32 verification mode (fp32.py) — every model
        runs with fp32 activations and an fp32 KV cache; the parity mode
        against the reference engine driven by fp32 oracles.
        selector_time: what MonitorSample.t_llm gets — "verify" (default, as
        the reference: the verify's device time, aggspec/engine.py:322),
        "round" (verify + draft device time: the sequential schedule's round
        period).  sim_cost: an object with t_llm(b, s) -> ms (the reference's
        CostModel, aggspec/oracles.py:157-183); when given the selector is fed
        t_llm(len(batch), s) exactly as the reference's simulated clock does,
        which makes the s trajectory reproducible across runs (parity tests).
        sampling: stochastic decoding as the reference engine does it — every
        drafter step SAMPLES from softmax(logits) with the request's
        draft/{rid}/{sid} stream (draft_sequence, aggspec/oracles.py:135-153)
        and keeps its distributions; the verifier runs speculative sampling
        (K10, verify() of aggspec/verification.py:29-77) on the voted
        drafter's and the target's distributions with the verify/{rid}
        stream, advanced by the draws the device made (aggspec/engine.py:
        232-248, 285-330).  Greedy (False) is the point-mass special case.
        draft_sms > 0 (pipelined): the draft and verify streams live on two
        green contexts splitting the GPU's SMs — draft_sms for the drafters,
        the rest for the verifier (ms_sm_partition): the drafters' small
        kernels no longer wait for, or displace, the verify GEMMs' CTAs.
        draft_pdl=False: the drafters' kernels launch without programmatic
        dependent launch (a PDL-launched kernel's CTAs occupy SM slots while
        they wait for their predecessor — slots the concurrent verify could
        use).
        draft_coresident (default: on for grouped Llama drafters in the
        pipelined schedule with caches <= 1,024 positions): the drafters' decode
        steps run in co-resident launch shapes (ms_set_coresident: 64-thread
        gemv / decode-attention CTAs, the LM head on gemv) that fit on an SM
        beside two verify-GEMM CTAs.
        grouped_drafters: K Llama drafters of one architecture run as row
        groups of one model (one launch per op for all drafters; False: one
        model per drafter on its own stream).  stream_priority ("equal",
        "verify", "draft"): CUDA stream priorities of the pipelined schedule
        (A/Bs in DESIGN §8)."""
        validate_config(cfg)
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"precision must be 'bf16' or 'fp32', got {precision!r}")
        if selector_time not in ("verify", "round"):
            raise ValueError("selector_time must be 'verify' or 'round'")
        if precision == "fp32" and kv_block_size > 0:
            raise ValueError("the fp32 verification mode uses a contiguous KV cache")
        if sampling and fidelity is not None:
            raise ValueError("fidelity injection replaces drafted tokens: greedy decoding only")
        self.sampling = bool(sampling)
        self.precision = precision
        self.selector_time = selector_time
        self.sim_cost = sim_cost
        kv_dtype = torch.float32 if precision == "fp32" else torch.bfloat16
        if len(cfg.initial_weights) != len(drafters):
            raise ValueError("initial_weights must have one entry per drafter")
        if pipelined and slots % 2:
            raise ValueError("pipelined mode needs an even number of slots (two groups)")
        self.dev = torch.device(device)
        _dev.require_cuda()
        self.cfg = cfg
        self.K = len(drafters)
        self.B = slots
        self.max_len = max_len
        self.adaptive = adaptive
        self.record = record
        self.pipelined = pipelined
        s_cap = cfg.s_max
        if hasattr(target, "forward"):
            self.target = target
        else:
            rows_t = max(slots * (s_cap + 1), slots * min(max_len, self.PREFILL_CHUNK))
            self.target = make_model(target, max_rows=rows_t, device=device, precision=precision)
        self.tp = hasattr(self.target, "comm")
        if self.tp and sampling:
            raise ValueError("stochastic decoding needs full-vocabulary target logits (not tensor parallel)")
        self.Vt = self.target.cfg.vocab                       # width of the target's logits
        V = self.Vt * (self.target.tp if self.tp else 1)      # full vocabulary
        if any(w.cfg.vocab != V for w in drafters):
            raise ValueError("drafters and target must share a vocabulary")
        self.V = V
        self.sync_time = sync_time
        # K Llama drafters of one architecture run as row groups of one model
        # (one launch per op for all drafters)
        self.grouped = (len(drafters) > 1 and all(getattr(w.cfg, "family", "") == "llama" for w in drafters)
                        and all(w.cfg == drafters[0].cfg for w in drafters)
                        and bool(grouped_drafters) and precision == "bf16")
        rows = slots * min(max_len, max(self.PREFILL_CHUNK, cfg.s_max + 2))
        self.ssms = [] if self.grouped else [make_model(w, max_rows=rows, device=device, small_gemm=True,
                                                        precision=precision) for w in drafters]
        if self.grouped:
            self.ssm_g = GroupedLlamaModel(drafters, max_rows=rows, device=device)
            self.s_cache_g = KVCache(drafters[0].cfg, self.K * slots, max_len, device)
            self.fid_arr = None
        if kv_block_size > 0:
            from .paged import PagedKVCache
            self.t_cache = PagedKVCache(self.target.cfg, slots, max_len, kv_block_size, kv_blocks, device)
        else:
            self.t_cache = KVCache(self.target.cfg, slots, max_len, device, dtype=kv_dtype)
        self.paged = kv_block_size > 0
        self.s_caches = [] if self.grouped else [KVCache(w.cfg, slots, max_len, device, dtype=kv_dtype)
                                                 for w in drafters]
        ng = 2 if pipelined else 1
        gb = slots // ng
        self.groups = [_Group(self, g, g * gb, gb) for g in range(ng)]
        self.slot = torch.arange(slots, dtype=I32, device=self.dev)
        self.fidelity = list(fidelity) if fidelity is not None else None
        self.inject_seed = inject_seed
        self.teacher = (torch.full((slots, max_len), -1, dtype=I32, device=self.dev)
                        if fidelity is not None else None)
        self.use_graphs = use_graphs
        self.graphs: dict = {}
        self.graph_kernels: dict = {}   # kernels per captured graph (launch accounting)
        self.kernel_launches = 0        # kernels this engine issued (eager + replayed)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.ssm_streams = [torch.cuda.Stream(self.dev) for _ in range(self.K)]
        # stream priorities for the pipelined schedule (CTA scheduling order when
        # both streams' kernels wait for SM slots): equal by default
        if stream_priority not in ("equal", "verify", "draft"):
            raise ValueError("stream_priority must be 'equal', 'verify' or 'draft'")
        hi = lambda k: -1 if stream_priority == k else 0  # noqa: E731
        self.draft_pdl = bool(draft_pdl)
        # co-resident drafter shapes by default only for short caches: their
        # one-warp-per-(request, head) decode attention streams ~1.9 TB/s, fine
        # beside the verifier at a few hundred keys but the critical path of a
        # draft-bound 4K-context round (cfg5: attention 307 vs 111 us per layer)
        self.draft_coresident = bool((pipelined and self.grouped and max_len <= 1024)
                                     if draft_coresident is None else draft_coresident)
        self.draft_sms = self.verify_sms = 0
        if draft_sms > 0:
            if not pipelined:
                raise ValueError("draft_sms partitions the SMs between concurrent drafting and "
                                 "verification: pipelined schedule only")
            self.draft_stream, self.verify_stream, self.draft_sms, self.verify_sms = _dev.sm_partition_streams(
                draft_sms, self.dev, hi("draft"), hi("verify"))
        else:
            self.draft_stream = torch.cuda.Stream(self.dev, priority=hi("draft"))
            self.verify_stream = torch.cuda.Stream(self.dev, priority=hi("verify"))
        self.requests: list[Request] = []
        self._run_t0 = None

    # ------------------------------------------------------------------ setup
    def prefill(self, requests: list[Request]) -> None:
        """Assign slots (request i -> slot i; a group is a slot range) and cache
        every prompt position but the last (the first round feeds the last
        prompt token)."""
        if len(requests) > self.B:
            raise ValueError(f"{len(requests)} requests exceed {self.B} slots")
        self.requests = list(requests)
        if self.sampling:  # the reference's per-request streams (aggspec/engine.py:232-248)
            self._draft_rngs = {(r.id, k): seeded_rng(self.cfg.seed, f"draft/{r.id}/{k}")
                                for r in requests for k in range(self.K)}
            self._verify_rngs = {r.id: seeded_rng(self.cfg.seed, f"verify/{r.id}") for r in requests}
        ctx = [list(r.prompt) + list(r.generated) for r in requests]
        if min(len(c) for c in ctx) < 1:
            raise ValueError("context must be non-empty")
        if any(len(c) + r.remaining + self.cfg.s_max + 2 > self.max_len for c, r in zip(ctx, requests)):
            raise ValueError("max_len too small for prompt + max_new_tokens + s_max")
        for g in self.groups:
            idx = range(g.slot0, min(g.slot0 + g.B, len(requests)))
            g.requests = [requests[i] for i in idx]
            g.ctx = [ctx[i] for i in idx]
            g.ssm_cached = [[len(c) - 1 for c in g.ctx] + [0] * (g.B - len(g.ctx)) for _ in range(self.K)]
            keys = np.zeros(g.B, np.int32)
            for b, r in enumerate(g.requests):
                keys[b] = zlib.crc32(str(r.id).encode()) & 0x7FFFFFFF
            g.req_key.copy_(torch.from_numpy(keys))
            g.pending = None
        P = max(len(c) for c in ctx) - 1
        if self.paged:  # a fresh batch: every slot's blocks back to the pool, prompts' blocks in
            mgr = self.t_cache.mgr
            for b in range(self.B):
                mgr.release(b)
            for b in range(self.B):  # padding slots too: the prefill forward writes P rows for every slot
                mgr.ensure(b, max(P, 1))
            self.h2d_bytes += self.t_cache.upload()
        if P > 0:
            toks = np.zeros((self.B, P), np.int32)
            for b, c in enumerate(ctx):
                toks[b, : len(c) - 1] = c[:-1]
            t = torch.from_numpy(toks).to(self.dev)
            self.h2d_bytes += toks.nbytes
            self._prefill_chunks(t)
        for r in requests:
            if r.remaining <= 0 and r.state != RequestState.FINISHED:
                r.state = RequestState.FINISHED
        torch.cuda.synchronize(self.dev)

    def _prefill_chunks(self, t: torch.Tensor) -> None:
        """Cache prompt positions 0..P-1 (t [B, P]) in every model, PREFILL_CHUNK
        positions at a time (chunked prefill — activation buffers
        and GEMM temporaries are sized for a chunk, not a 4K-token prompt);
        each chunk's queries attend to the cached earlier chunks."""
        B, P = t.shape
        empty = torch.zeros(0, dtype=I32, device=self.dev)
        tgt_dummy = torch.empty(0, self.Vt, device=self.dev)
        dummy = torch.empty(0, self.V, device=self.dev)
        G = self.K
        gslot = torch.arange(G * B, dtype=I32, device=self.dev)
        for c0 in range(0, P, self.PREFILL_CHUNK):
            tc = t[:, c0: c0 + self.PREFILL_CHUNK].contiguous()
            st = torch.full((B,), c0, dtype=I32, device=self.dev)
            self.target.forward(tc, st, self.slot, self.t_cache, tgt_dummy, head_rows=empty, prefill=True)
            for m, c in zip(self.ssms, self.s_caches):
                m.forward(tc, st, self.slot, c, dummy, head_rows=empty, prefill=True)
            if self.grouped:
                self.ssm_g.forward(tc.repeat(G, 1), st.repeat(G), gslot, self.s_cache_g, dummy, head_rows=empty,
                                   prefill=True)

    def set_teacher(self, teacher: dict) -> None:
        """Target greedy continuations (request id -> tokens after the prompt)
        for fidelity injection."""
        if self.teacher is None:
            raise ValueError("engine was built without fidelity injection")
        t = np.full((self.B, self.max_len), -1, np.int32)
        for b, r in enumerate(self.requests):
            seq = teacher[r.id]
            p0 = len(r.prompt)
            t[b, p0: p0 + len(seq)] = seq
        self.teacher.copy_(torch.from_numpy(t))

    # --------------------------------------------------------- device work
    def _device_draft(self, g: _Group, s: int, qc: int) -> None:
        """K drafters (concurrent streams) + vote + verifier input rows."""
        main = torch.cuda.current_stream(self.dev)
        if self.grouped:
            self._draft_grouped(g, s, qc)
            sp = _dev.stream_ptr(main)
            _native.call("ms_vote", g.drafts_s(s).data_ptr(), g.w_dev.data_ptr(), None, g.B, self.K, s,
                         g.path.data_ptr(), g.voted.data_ptr(), sp)
            _native.call("ms_pack_verify", g.last.data_ptr(), g.path.data_ptr(), g.B, s, g.vin.data_ptr(), sp)
            return
        ev0 = torch.cuda.Event()
        ev0.record(main)
        done = []
        for k in range(self.K):
            st = self.ssm_streams[k]
            st.wait_event(ev0)
            with torch.cuda.stream(st):
                self._draft(g, k, s, qc, st)
                e = torch.cuda.Event()
                e.record(st)
                done.append(e)
        for e in done:
            main.wait_event(e)
        sp = _dev.stream_ptr(main)
        _native.call("ms_vote", g.drafts_s(s).data_ptr(), g.w_dev.data_ptr(), None, g.B, self.K, s,
                     g.path.data_ptr(), g.voted.data_ptr(), sp)
        _native.call("ms_pack_verify", g.last.data_ptr(), g.path.data_ptr(), g.B, s, g.vin.data_ptr(), sp)

    def _draft_grouped(self, g: _Group, s: int, qc: int) -> None:
        """All K drafters' s steps as row groups of one model (one launch per op)."""
        B, G, m = g.B, self.K, self.ssm_g
        sp = _dev.stream_ptr()
        dr = g.drafts_s(s)
        tok_in = g.g_c_tok[: G * B * qc].view(G * B, qc)
        teacher = None
        if self.teacher is not None:
            teacher = self.teacher.data_ptr() + g.slot0 * self.max_len * 4
        fid = (ctypes.c_float * 8)(*([float(f) for f in self.fidelity] if self.fidelity else [0.0] * G))
        for j in range(s):
            if j == 0:
                m.forward(tok_in, g.g_c_start, g.g_slot, self.s_cache_g, g.g_logits, head_rows=g.g_c_head)
            else:
                m.forward(g.g_step_tok, g.g_step_start[j - 1], g.g_slot, self.s_cache_g, g.g_logits)
            if self.sampling:  # row k*B + b: drafter k, request b; q laid out [K, B, s, V]
                _native.call("ms_softmax_sample", g.g_logits.data_ptr(), self.V, G * B, self.V,
                             g.u_draft.data_ptr() + j * 8, self.cfg.s_max, g.q.data_ptr() + j * self.V * 8,
                             s * self.V, g.g_argmax.data_ptr(), sp)
            else:
                _native.call("ms_argmax_rows", g.g_logits.data_ptr(), 0, G * B, self.V, self.V,
                             g.g_argmax.data_ptr(), g.g_ws.data_ptr(), sp)
            _native.call("ms_draft_commit_grouped", g.g_argmax.data_ptr(), g.ctx_len.data_ptr(), B, j, G, s,
                         teacher, self.max_len, g.req_key.data_ptr(), fid if self.fidelity else None,
                         self.inject_seed, dr.data_ptr(), g.g_step_tok.data_ptr(), sp)

    def _put_grouped_meta(self, g: _Group, put, start, c_head, steps, c_tok, qc) -> None:
        """Replicate the drafters' round inputs per row group (drafter)."""
        if not self.grouped:
            return
        G, B = self.K, g.B
        put("g_c_start", np.tile(np.asarray(start).reshape(-1), G))
        put("g_c_head", np.concatenate([k * B * qc + np.asarray(c_head).reshape(-1) for k in range(G)]))
        put("g_step_start", np.tile(np.asarray(steps).reshape(steps.shape[0], -1), (1, G)))
        if c_tok is not None:
            put("g_c_tok", np.tile(np.asarray(c_tok).reshape(B, -1), (G, 1)))

    def _draft(self, g: _Group, k: int, s: int, qc: int, st) -> None:
        B, m, cache = g.B, self.ssms[k], self.s_caches[k]
        sp = _dev.stream_ptr(st)
        dr = g.drafts_s(s)
        tok_in = g.c_tok[: B * qc].view(B, qc)
        teacher = None
        if self.teacher is not None:
            teacher = self.teacher.data_ptr() + g.slot0 * self.max_len * 4  # the group's rows
        f = float(self.fidelity[k]) if self.fidelity is not None else 0.0
        for j in range(s):
            if j == 0:
                m.forward(tok_in, g.c_start, g.slot, cache, g.ssm_logits[k], head_rows=g.c_head, stream=st)
            else:
                m.forward(g.step_tok[k], g.step_start[j - 1], g.slot, cache, g.ssm_logits[k], stream=st)
            if self.sampling:
                _native.call("ms_softmax_sample", g.ssm_logits[k].data_ptr(), self.V, B, self.V,
                             g.u_draft.data_ptr() + (k * B * self.cfg.s_max + j) * 8, self.cfg.s_max,
                             g.q.data_ptr() + (k * B * s * self.V + j * self.V) * 8, s * self.V,
                             g.argmax[k].data_ptr(), sp)
            else:
                _native.call("ms_argmax_rows", g.ssm_logits[k].data_ptr(), 0, B, self.V, self.V,
                             g.argmax[k].data_ptr(), g.ssm_ws[k].data_ptr(), sp)
            _native.call("ms_draft_commit", g.argmax[k].data_ptr(), g.ctx_len.data_ptr(), B, j, k,
                         self.K, s, teacher, self.max_len, g.req_key.data_ptr(), f,
                         self.inject_seed, dr.data_ptr(), g.step_tok[k].data_ptr(), sp)

    def _device_verify(self, g: _Group, s: int) -> None:
        """Verify forward of s+1 rows per request + greedy accept."""
        B, V = g.B, self.V
        sp = _dev.stream_ptr()
        vin = g.vin.view(-1)[: B * (s + 1)].view(B, s + 1)
        logits = g.v_logits[: B * (s + 1)]
        self.target.forward(vin, g.v_start, g.slot, self.t_cache, logits)
        a = g.acc
        if self.sampling:  # target distributions, the voted drafter's, speculative sampling (K10)
            _native.call("ms_softmax_sample", logits.data_ptr(), V, B * (s + 1), V, None, 0, g.o.data_ptr(), V,
                         None, sp)
            _native.call("ms_gather_voted", g.q.data_ptr(), g.voted.data_ptr(), self.K, B, s, V, g.qv.data_ptr(),
                         sp)
            _native.call("ms_accept_stochastic", g.path.data_ptr(), g.qv.data_ptr(), g.o.data_ptr(),
                         g.u_verify.data_ptr(), g.remaining.data_ptr(),
                         -1 if self.cfg.stop_token is None else self.cfg.stop_token, B, s, V,
                         g.k10_scratch.data_ptr(), a.n_acc.data_ptr(), a.emitted.data_ptr(), a.n_emit.data_ptr(),
                         a.finished.data_ptr(), g.n_draws.data_ptr(), sp)
            return
        if self.tp:  # vocab-parallel logits: cross-rank argmax, then accept
            R = B * (s + 1)
            self.target.argmax(logits, a.tgt_argmax[:R])
            _native.call("ms_accept_greedy", g.path.data_ptr(), a.tgt_argmax.data_ptr(), g.remaining.data_ptr(),
                         -1 if self.cfg.stop_token is None else self.cfg.stop_token, B, s, a.n_acc.data_ptr(),
                         a.emitted.data_ptr(), a.n_emit.data_ptr(), a.finished.data_ptr(), None, sp)
            return
        _native.call("ms_accept_greedy_logits", g.path.data_ptr(), logits.data_ptr(), 0, V,
                     g.remaining.data_ptr(), -1 if self.cfg.stop_token is None else self.cfg.stop_token,
                     B, s, a.tgt_argmax.data_ptr(), g.argmax_ws.data_ptr(), a.n_acc.data_ptr(),
                     a.emitted.data_ptr(), a.n_emit.data_ptr(), a.finished.data_ptr(), None, sp)

    def _replay(self, key, fn) -> None:
        """Run fn eagerly the first time (sets kernel attributes, produces this
        round's results), capture it as a CUDA graph for the next times."""
        n0 = _native.launch_count()
        if not self.use_graphs:
            fn()
            self.kernel_launches += _native.launch_count() - n0
            return
        gr = self.graphs.get(key)
        if gr is None:
            fn()
            torch.cuda.current_stream(self.dev).synchronize()
            self.kernel_launches += _native.launch_count() - n0
            gr = torch.cuda.CUDAGraph()
            n1 = _native.launch_count()
            with torch.cuda.graph(gr, stream=torch.cuda.current_stream(self.dev), capture_error_mode="thread_local"):
                fn()
            self.graph_kernels[key] = _native.launch_count() - n1
            self.graphs[key] = gr
            return
        gr.replay()
        self.kernel_launches += self.graph_kernels[key]

    def _launch_draft(self, g: _Group, s: int, qc: int) -> None:
        with torch.cuda.stream(self.draft_stream):
            g.ev_d0.record()
            # launch policies baked into the captured graph
            pdl = None if self.draft_pdl else _native.lib.ms_set_pdl(0)
            co = _native.lib.ms_set_coresident(1) if self.draft_coresident else None
            if self.grouped:
                self.ssm_g.coresident = self.draft_coresident
            try:
                self._replay(("draft", g.gid, s, qc), lambda: self._device_draft(g, s, qc))
            finally:
                if pdl is not None:
                    _native.lib.ms_set_pdl(pdl)
                if co is not None:
                    _native.lib.ms_set_coresident(co)
                if self.grouped:
                    self.ssm_g.coresident = False
            g.ev_d1.record()

    def _launch_verify(self, g: _Group, s: int) -> None:
        with torch.cuda.stream(self.verify_stream):
            self.verify_stream.wait_event(g.ev_d1)  # this group's drafts
            g.ev_v0.record()
            self._replay(("verify", g.gid, s), lambda: self._device_verify(g, s))
            g.ev_v1.record()
            g.res_h.copy_(g.res, non_blocking=True)  # one D2H for the whole round
            g.ev_res.record()

    def capture_graphs(self, s_values=None) -> None:
        """Capture the draft and verify graphs of every s up front (call before
        prefill: the capture runs each graph once on dummy rows, writing
        scratch K/V that prefill / decode overwrite before anything reads it),
        so no capture lands inside a timed decode when the selector moves s."""
        if not self.use_graphs:
            return
        s_values = s_values or range(self.cfg.s_min, self.cfg.s_max + 1)
        if self.paged:  # the dummy rounds write up to position ~3 (s_max + 1) of every slot
            for b in range(self.B):
                self.t_cache.mgr.ensure(b, min(self.t_cache.max_len, 3 * (self.cfg.s_max + 2)))
            self.t_cache.upload()
        for g in self.groups:
            for s in s_values:
                # every catch-up width a round at this s can need: s+1, or up to
                # s_prev+1 <= s_max+1 after the selector lowered s
                for qc in range(s + 1, self.cfg.s_max + 2):
                    if ("draft", g.gid, s, qc) in self.graphs:
                        continue
                    B = g.B
                    lens = np.full(B, 2 * qc + 1, np.int64)
                    mh = g.meta_h.numpy()
                    mh[:] = 0
                    o, _ = g.meta_off["w"]
                    mh[o: o + 2 * self.K] = np.ones(self.K, np.float64).view(np.int32)
                    def put(name, v):
                        o, _ = g.meta_off[name]
                        v = np.ascontiguousarray(v, dtype=np.int32).reshape(-1)
                        mh[o: o + v.size] = v

                    steps = np.stack([lens + j - 1 for j in range(1, self.cfg.s_max + 1)])
                    for name, v in (("ctx_len", lens), ("c_start", lens - qc), ("v_start", lens - 1),
                                    ("c_head", np.arange(B) * qc + qc - 1), ("step_start", steps)):
                        put(name, v)
                    self._put_grouped_meta(g, put, lens - qc, np.arange(B) * qc + qc - 1, steps, None, qc)
                    with torch.cuda.stream(self.draft_stream):
                        g.meta.copy_(g.meta_h, non_blocking=True)
                    self._launch_draft(g, s, qc)  # eager run, then capture (_replay)
                    if ("verify", g.gid, s) not in self.graphs:
                        self._launch_verify(g, s)
                    g.ev_res.synchronize()
                    torch.cuda.synchronize(self.dev)
        torch.cuda.synchronize(self.dev)

    # ------------------------------------------------------------- host side
    def _upload(self, g: _Group, s: int) -> int:
        """Pack the group's round inputs into its pinned buffer; one H2D copy
        on the draft stream.  Returns Qc (catch-up rows)."""
        B = g.B
        lens = np.array([len(c) for c in g.ctx] + [1] * (B - len(g.ctx)), np.int64)
        act = g.active()
        need = [lens[b] - g.ssm_cached[k][b] for k in range(self.K) for b in act]
        # catch-up width s+1 (the most a drafter can lag when s did not shrink):
        # one draft graph per s.  Rows an SSM has already cached are recomputed
        # and rewritten with identical K/V (the forward is batch invariant), so
        # this only costs a slightly wider first step.  After the selector
        # lowered s a drafter can lag by up to s_prev+1: a wider graph then.
        qc = max(s + 1, int(max(need)) if need else 1)
        start = np.maximum(lens - qc, 0)
        c_tok = np.zeros((B, qc), np.int32)
        for b, c in enumerate(g.ctx):
            seg = c[start[b]: start[b] + qc]
            c_tok[b, : len(seg)] = seg
        c_head = np.arange(B) * qc + (lens - 1 - start)
        rem = np.zeros(B, np.int32)
        for b in act:
            rem[b] = g.requests[b].remaining
        last = np.array([c[-1] for c in g.ctx] + [0] * (B - len(g.ctx)), np.int32)
        steps = np.stack([lens + j - 1 for j in range(1, self.cfg.s_max + 1)])
        mh = g.meta_h.numpy()

        def put(name, v):
            o, _ = g.meta_off[name]
            v = np.ascontiguousarray(v, dtype=np.int32).reshape(-1)
            mh[o: o + v.size] = v

        w = np.array([self.weights.weights[k] for k in range(self.K)], np.float64)  # snapshot
        put("w", w.view(np.int32))
        if self.sampling:
            # draft_sequence draws s uniforms per (request, drafter) per round; the
            # verifier's uniforms are peeked (<= s + 1) and the stream advanced by
            # the device's n_draws after the round (verification.peek_uniforms)
            smax = self.cfg.s_max
            ud = np.zeros((self.K, B, smax), np.float64)
            uv = np.zeros((B, s + 1), np.float64)
            for b in act:
                rid = g.requests[b].id
                for k in range(self.K):
                    ud[k, b, :s] = self._draft_rngs[(rid, k)].random(s)
                uv[b] = peek_uniforms(self._verify_rngs[rid], s + 1)
            put("u_draft", ud.view(np.int32))
            put("u_verify", uv.view(np.int32))
        put("ctx_len", lens)
        put("c_start", start)
        put("c_head", c_head)
        put("v_start", lens - 1)
        put("last", last)
        put("remaining", rem)
        put("step_start", steps)
        put("c_tok", c_tok)
        self._put_grouped_meta(g, put, start, c_head, steps, c_tok, qc)
        with torch.cuda.stream(self.draft_stream):
            g.meta.copy_(g.meta_h, non_blocking=True)
        self.h2d_bytes += g.meta_h.numel() * 4
        if self.paged:  # the verify writes positions len(ctx)-1 .. len(ctx)-1+s
            for b in act:
                self.t_cache.mgr.ensure(g.slot0 + b, len(g.ctx[b]) + s)
            self.h2d_bytes += self.t_cache.upload(slice(g.slot0, g.slot0 + B), stream=self.draft_stream)
        return qc

    def _start_draft(self, g: _Group) -> bool:
        """Take the group's unfinished requests as a draft batch (s = the
        selector's current s, weights snapshot) and launch its drafting."""
        act = g.active()
        if not act:
            return False
        s = self.selector.current_s
        g.prev_states = [g.requests[b].state for b in act]
        for b in act:
            g.requests[b].advance(RequestState.DRAFTING)
        qc = self._upload(g, s)
        self._launch_draft(g, s, qc)
        g.pending = (s, qc, act, time.perf_counter())
        return True

    def _discard_draft(self, g: _Group) -> None:
        """Drop a group's drafted-but-unverified round (decode stopped by
        max_rounds while it was in flight): its requests go back to the state
        they had before the draft, so the next decode() re-drafts them.  The
        drafters' KV written by the discarded round lies past their cached
        lengths (rollback arithmetic) and is simply overwritten later."""
        if g.pending is None:
            return
        g.ev_d1.synchronize()
        for b, st in zip(g.pending[2], g.prev_states):
            g.requests[b].state = st
        g.pending = None

    def _finish_verify(self, g: _Group, rnd: int) -> RoundStats:
        """Host bookkeeping of a verified group (reference semantics)."""
        s, qc, active, t_start = g.pending
        g.pending = None
        g.ev_res.synchronize()
        self.d2h_bytes += g.res_h.numel() * 4
        rh = g.res_h.numpy()

        def get(name, n=None):
            o, m = g.res_off[name]
            return rh[o: o + (m if n is None else n)]

        B = g.B
        n_acc = get("n_acc")
        n_emit = get("n_emit")
        emitted = get("emitted", B * (s + 1)).reshape(B, s + 1)
        voted = get("voted")
        drafts = get("drafts", B * self.K * s).reshape(B, self.K, s)
        t_verify = g.ev_v0.elapsed_time(g.ev_v1)
        t_draft = g.ev_d0.elapsed_time(g.ev_d1)
        if self.sampling:  # advance each verify stream by the uniforms the device used
            nd = get("n_draws")
            for b in active:
                self._verify_rngs[g.requests[b].id].random(int(nd[b]))
        # selector input (MonitorSample.t_llm): the verify's device time, as the
        # reference (aggspec/engine.py:322); "round" adds the draft time (the
        # sequential schedule's round period); sim_cost: the reference's
        # simulated clock t_llm(len(batch), s) (aggspec/engine.py:359)
        if self.sim_cost is not None:
            t_sel = float(self.sim_cost.t_llm(len(active), s))
        else:
            t_sel = t_verify + (t_draft if self.selector_time == "round" else 0.0)
        if self.sync_time is not None:
            t_sel = float(self.sync_time(t_sel))
        t0 = self._run_t0
        ts = (t0.elapsed_time(g.ev_d0), t0.elapsed_time(g.ev_d1), t0.elapsed_time(g.ev_v0),
              t0.elapsed_time(g.ev_v1)) if t0 is not None else (None,) * 4
        out = commit_round(g.requests, g.ctx, g.ssm_cached, active, s, n_acc, n_emit, emitted, voted, drafts,
                           self.weights, self.selector, self.cfg, t_sel, rnd, self.adaptive,
                           finish_time=ts[3] if ts[3] is not None else time.perf_counter())  # device ms
        if self.paged:  # free blocks holding only rejected tokens' KV (or all, when finished)
            for b in active:
                if g.requests[b].state == RequestState.FINISHED:
                    self.t_cache.mgr.release(g.slot0 + b)
                else:
                    self.t_cache.mgr.truncate(g.slot0 + b, len(g.ctx[b]))
        accs, ems, vts, vl, decision = out.accepted, out.emitted, out.voted, out.vl, out.decision
        trace = None
        if self.record:
            trace = dict(active=active, drafts=drafts.copy(), weights_used=g.w_dev.cpu().numpy(),
                         path=get("path", B * s).reshape(B, s).copy(), voted=voted.copy(),
                         n_acc=n_acc.copy(), n_emit=n_emit.copy(), emitted=emitted.copy(),
                         tgt=get("tgt", B * (s + 1)).reshape(B, s + 1).copy(),
                         remaining=g.remaining.cpu().numpy())
        return RoundStats(s=s, qc=qc, t_verify_ms=t_verify, t_draft_ms=t_draft, trace=trace,
                          t_round_ms=(time.perf_counter() - t_start) * 1e3, accepted=accs,
                          emitted=ems, voted=vts, vl=vl, decision=decision.value, group=g.gid,
                          s_next=self.selector.current_s, weights=dict(self.weights.weights),
                          round_index=rnd, request_ids=tuple(g.requests[b].id for b in active),
                          pool_depth=sum(1 for x in self.groups if x.pending is not None),
                          draft_start=ts[0], draft_end=ts[1], verify_start=ts[2], verify_end=ts[3])

    def run(self, requests: list[Request], max_rounds: int | None = None) -> RunResult:
        """Generate until every request finishes (reference semantics)."""
        self.prefill(requests)
        return self.decode(max_rounds)

    def decode(self, max_rounds: int | None = None, reset_controllers: bool = False) -> RunResult:
        """Run rounds until the prefilled requests finish.  The drafter weights
        and the speculation-length selector persist across calls (a serving
        engine keeps adapting over its request stream); the first call or
        reset_controllers=True starts them from the config (s_init, initial
        weights), as the reference engine does per run."""
        cfg = self.cfg
        if reset_controllers or getattr(self, "selector", None) is None:
            self.weights = WeightTable.from_config(list(range(self.K)), cfg)
            self.selector = SelectorState.from_config(cfg)
        res = RunResult(outputs={})
        t0 = time.perf_counter()
        rnd = 0
        # device clock origin of this decode (trace timestamps, request finish times)
        self._run_t0 = torch.cuda.Event(enable_timing=True)
        self._run_t0.record(self.draft_stream)
        for r in self.requests:
            r.arrival_time = 0.0
        if not self.pipelined:
            g = self.groups[0]
            while (max_rounds is None or rnd < max_rounds) and self._start_draft(g):
                self._launch_verify(g, g.pending[0])
                res.rounds.append(self._finish_verify(g, rnd))
                rnd += 1
        else:
            # phase: verify `cur` on the verify stream while drafting `nxt` on the
            # draft stream (the drafter runs only while the pool holds < 1 batch)
            cur, nxt = self.groups
            self._start_draft(cur)
            while max_rounds is None or rnd < max_rounds:
                if cur.pending is None:  # nothing to verify here: try the other group
                    if nxt.pending is None and not self._start_draft(nxt):
                        if not self._start_draft(cur):
                            break
                        continue
                    cur, nxt = nxt, cur
                    continue
                self._launch_verify(cur, cur.pending[0])
                if nxt.pending is None:
                    self._start_draft(nxt)
                res.rounds.append(self._finish_verify(cur, rnd))
                rnd += 1
                cur, nxt = nxt, cur
            for g in self.groups:  # stopped by max_rounds with a draft in flight
                self._discard_draft(g)
        torch.cuda.synchronize(self.dev)
        res.wall_s = time.perf_counter() - t0
        res.outputs = {r.id: list(r.generated) for r in self.requests}
        res.tokens = sum(len(r.generated) for r in self.requests)
        return res

    # ----------------------------------------------------- greedy reference
    def greedy_teacher(self, requests: list[Request], n_new: int) -> dict:
        """Plain (non-speculative) greedy decoding with the target: one
        forward of one row per request per token.  Used for fidelity injection
        and as the lossless check (speculative output must equal it)."""
        B = self.B
        cache = self.t_cache
        ctx = [list(r.prompt) for r in requests]
        P = max(len(c) for c in ctx) - 1
        toks = np.zeros((B, max(P, 1)), np.int32)
        for b, c in enumerate(ctx):
            toks[b, : len(c) - 1] = c[:-1]
        zero = torch.zeros(B, dtype=I32, device=self.dev)
        empty = torch.zeros(0, dtype=I32, device=self.dev)
        dummy = torch.empty(0, self.Vt, device=self.dev)
        if self.paged:
            for b in range(B):
                cache.mgr.release(b)
            for b in range(B):
                cache.mgr.ensure(b, (len(ctx[b]) if b < len(ctx) else 1) + n_new + 1)
            cache.upload()
        tt = torch.from_numpy(toks).to(self.dev)
        for c0 in range(0, P, self.PREFILL_CHUNK):
            self.target.forward(tt[:, c0: c0 + self.PREFILL_CHUNK].contiguous(),
                                torch.full((B,), c0, dtype=I32, device=self.dev), self.slot, cache, dummy,
                                head_rows=empty, prefill=True)
        out = {r.id: [] for r in requests}
        lens = np.array([len(c) for c in ctx] + [1] * (B - len(ctx)))
        cur = np.array([c[-1] for c in ctx] + [0] * (B - len(ctx)), np.int32)
        logits = torch.empty(B, self.Vt, device=self.dev)
        am = torch.zeros(B, dtype=I32, device=self.dev)
        ws = torch.zeros(B, dtype=torch.int64, device=self.dev)
        for t in range(n_new):
            self.target.forward(torch.from_numpy(cur[:, None].copy()).to(self.dev),
                                torch.from_numpy((lens - 1).astype(np.int32)).to(self.dev),
                                self.slot, cache, logits)
            if self.tp:
                self.target.argmax(logits, am)
            else:
                _native.call("ms_argmax_rows", logits.data_ptr(), 0, B, self.V, self.V, am.data_ptr(),
                             ws.data_ptr(), _dev.stream_ptr())
            nxt = am.cpu().numpy()
            for b, r in enumerate(requests):
                out[r.id].append(int(nxt[b]))
            cur = nxt.astype(np.int32)
            lens = lens + 1
        return out
