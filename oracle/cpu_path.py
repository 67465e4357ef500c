"""The reference's CPU path, for bench.py's reference arm — TEST / BASELINE
INFRASTRUCTURE ONLY (see oracle/__init__.py: only tests/, smoke() and the
bench's cpu_baseline / --impl reference legs may use this module).

What is timed is the UNMODIFIED reference engine — aggspec.run_sequential /
run_pipelined (aggspec/engine.py:619-671; imported from baseline/_ref, the
pip install of /root/reference/pkg, or from the reference tree when it is
present) with its own draft_sequence, merge / select_majority, verify,
update_weights and selector — driving fp32 CPU transformer ModelOracles
(aggspec/oracles.py:19-26) of the bench's model shapes.

The oracles:

* `PrefixCachedOracle` — next_dist(context) of an fp32 decoder (explicit
  norms, no bf16 rounding: the fp32 verification-mode contract of
  oracle/llama_ref.py / opt_ref.py with exact=True) behind the protocol.  The
  protocol is one call per context (the reference recomputes each draft and
  verify position from the full context, aggspec/oracles.py:135-153,
  aggspec/engine.py:294-296); a full forward of a 70B model over a ~190-token
  context is ~27 TFLOP, so the adapter keeps a small longest-common-prefix KV
  cache (as GPUOracle does on the device) and each call computes only the
  positions its context adds.  It is greedy: the point mass on the first-index
  argmax of the logits.
* `FidelityDrafter` — the bench's fidelity injection (DESIGN.md §6,
  csrc/spec.cu draft_commit_kernel) restated: the drafter's forward is
  computed in full, then with probability f_k — the same counter hash of
  (seed, request key, k, absolute position) — its token is replaced by the
  target's greedy continuation at that position.  So the CPU arm sees the
  same acceptance process as the GPU arm.

`shared_layers=True` builds one decoder layer of random weights and runs it
n_layers times: every layer's matmuls, attention and KV cache are computed
(the FLOPs and bytes per token of the full model; each layer's 3.4 GB of fp32
weights still streams from DRAM), without 275 GB of fp32 weights in host
memory.  Nothing is scaled or extrapolated: the reported time is the wall
clock of complete reference-engine runs.
"""
from __future__ import annotations

import math
import os
import sys
import time
import zlib

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def import_reference():
    """The reference package: baseline/_ref (installed by build(), travels to
    the GPU box) or the read-only tree in the dev container."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "aggspec")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import aggspec  # noqa: F401
            import aggspec.engine
            return sys.modules["aggspec"], p
    raise ImportError("reference package not found (baseline/_ref or /root/reference)")


# ------------------------------------------------------------ fp32 decoder
class DecoderF32:
    """Incremental fp32 forward (KV cache) of the OPT / Llama-2 decoders of
    paper_2402_15678_b200/weights.py, exact fp32 (explicit norms)."""

    def __init__(self, w: dict, cfg, shared_layers: bool = False):
        self.cfg = cfg
        self.f = {k: v.float().contiguous() for k, v in w.items()}
        self.L = cfg.n_layers
        self.shared = shared_layers
        if cfg.family == "llama":
            from .llama_ref import rope_table, split_gate_up
            self.table = rope_table(cfg.max_pos, cfg.head_dim, cfg.rope_theta)
            self.gu = {}
            for i in range(1 if shared_layers else self.L):
                g, u = split_gate_up(self.f[f"l{i}.w_gu"], cfg.ffn)
                self.gu[i] = (g.contiguous(), u.contiguous())

    def _p(self, i: int) -> str:
        return "l0." if self.shared else f"l{i}."

    def new_cache(self, cap: int):
        c = self.cfg
        shape = (self.L, cap, c.n_kv_heads, c.head_dim)
        return [torch.empty(shape), torch.empty(shape)]

    def extend(self, kv, n: int, tokens: list[int]) -> torch.Tensor:
        """Positions n .. n+T-1 (cache holds 0..n-1); writes their K/V into kv;
        returns the fp32 logits of the last position [V]."""
        c, f = self.cfg, self.f
        T = len(tokens)
        tok = torch.as_tensor(tokens, dtype=torch.long)
        H, Hkv, D = c.n_heads, c.n_kv_heads, c.head_dim
        G = H // Hkv
        scale = 1.0 / math.sqrt(D)
        N = n + T
        mask = torch.ones(T, N, dtype=torch.bool).triu(n + 1)  # query t sees keys <= n + t
        pos = torch.arange(n, N)
        if c.family == "llama":
            x = f["tok_emb"][tok]
            cs = self.table[pos]
            cos, sin = cs[..., 0][:, None, :], cs[..., 1][:, None, :]

            def rope(z):
                a, b = z[..., : D // 2], z[..., D // 2:]
                return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)

            def rms(z, g):
                return z * torch.rsqrt((z * z).mean(-1, keepdim=True) + c.eps) * g
            for i in range(self.L):
                p = self._p(i)
                qkv = rms(x, f[p + "attn_norm"]) @ f[p + "w_qkv"].T
                q = rope(qkv[:, : H * D].view(T, H, D))
                kv[0][i, n:N] = rope(qkv[:, H * D: (H + Hkv) * D].view(T, Hkv, D))
                kv[1][i, n:N] = qkv[:, (H + Hkv) * D:].view(T, Hkv, D)
                a = self._attend(q, kv[0][i, :N], kv[1][i, :N], G, scale, mask)
                x = a @ f[p + "w_o"].T + x
                h = rms(x, f[p + "mlp_norm"])
                wg, wu = self.gu[0 if self.shared else i]
                gt = h @ wg.T
                x = (gt / (1.0 + torch.exp(-gt)) * (h @ wu.T)) @ f[p + "w_down"].T + x
            return (rms(x[-1:], f["norm_f"]) @ f["lm_head"].T)[0]
        x = f["tok_emb"][tok] + f["pos_emb"][pos + c.pos_offset]

        def ln(z, g, b):
            m = z.mean(-1, keepdim=True)
            return (z - m) * torch.rsqrt(((z - m) ** 2).mean(-1, keepdim=True) + c.eps) * g + b
        for i in range(self.L):
            p = self._p(i)
            qkv = ln(x, f[p + "ln1_g"], f[p + "ln1_b"]) @ f[p + "w_qkv"].T + f[p + "b_qkv"]
            q, k, v = qkv.split(c.d, dim=-1)
            kv[0][i, n:N] = k.view(T, H, D)
            kv[1][i, n:N] = v.view(T, H, D)
            a = self._attend(q.view(T, H, D), kv[0][i, :N], kv[1][i, :N], 1, scale, mask)
            x = a @ f[p + "w_o"].T + f[p + "b_o"] + x
            h = ln(x, f[p + "ln2_g"], f[p + "ln2_b"])
            x = torch.relu(h @ f[p + "w_fc1"].T + f[p + "b_fc1"]) @ f[p + "w_fc2"].T + f[p + "b_fc2"] + x
        return (ln(x[-1:], f["lnf_g"], f["lnf_b"]) @ f["tok_emb"].T)[0]

    @staticmethod
    def _attend(q, k, v, G, scale, mask):
        T, H, D = q.shape
        if G > 1:
            k = k.repeat_interleave(G, dim=1)
            v = v.repeat_interleave(G, dim=1)
        sc = (q.transpose(0, 1) @ k.permute(1, 2, 0)) * scale  # [H, T, N]
        sc = sc.masked_fill(mask, float("-inf"))
        return (torch.softmax(sc, dim=-1) @ v.transpose(0, 1)).transpose(0, 1).reshape(T, H * D)


# -------------------------------------------------------------- ModelOracles
class _Entry:
    __slots__ = ("tokens", "kv", "logits", "pinned", "used")

    def __init__(self, tokens, kv, logits, pinned=False):
        self.tokens, self.kv, self.logits, self.pinned, self.used = tokens, kv, logits, pinned, 0


class PrefixCachedOracle:
    """ModelOracle (aggspec/oracles.py:19-26) over DecoderF32, greedy, with a
    small longest-common-prefix KV cache (module docstring)."""

    def __init__(self, model: DecoderF32, prob_dist, context_cap: int = 4096, capacity: int = 6,
                 cache_len: int = 512):
        self.model, self.P = model, prob_dist
        self.vocab_size = model.cfg.vocab
        self.context_cap = context_cap
        self.capacity, self.cache_len = capacity, cache_len
        self.entries: list[_Entry] = []
        self.calls = self.positions = 0
        self._tick = 0

    def _lcp(self, a, b) -> int:
        n = min(len(a), len(b))
        i = 0
        while i < n and a[i] == b[i]:
            i += 1
        return i

    def logits(self, context) -> torch.Tensor:
        ctx = list(context)
        self.calls += 1
        self._tick += 1
        best, lcp = None, 0
        for e in self.entries:
            m = self._lcp(e.tokens, ctx)
            if m > lcp:
                best, lcp = e, m
        if best is not None and lcp == len(ctx) == len(best.tokens):
            best.used = self._tick
            return best.logits
        n = min(lcp, len(ctx) - 1)  # compute at least the last position
        if best is not None and not best.pinned and n == len(best.tokens):
            e = best  # ctx extends this entry: grow it in place
        else:
            kv = self.model.new_cache(max(self.cache_len, len(ctx) + 16))
            if best is not None and n > 0:
                kv[0][:, :n] = best.kv[0][:, :n]
                kv[1][:, :n] = best.kv[1][:, :n]
            else:
                n = 0
            e = _Entry(ctx[:n], kv, None)
            self._insert(e)
        if len(ctx) > e.kv[0].shape[1]:
            raise ValueError("context longer than the oracle's cache")
        e.logits = self.model.extend(e.kv, n, ctx[n:])
        self.positions += len(ctx) - n
        e.tokens = ctx
        e.used = self._tick
        return e.logits

    def _insert(self, e):
        free = [x for x in self.entries if not x.pinned]
        if len(free) >= self.capacity:
            self.entries.remove(min(free, key=lambda x: x.used))
        self.entries.append(e)

    def pin(self, context) -> None:
        """Prefill `context` (untimed setup) and keep it as a root entry."""
        self.logits(context)
        e = next(x for x in self.entries if x.tokens == list(context))
        e.pinned = True

    def reset(self) -> None:
        """Drop every unpinned entry (each timed step starts from the prefilled prompts)."""
        self.entries = [e for e in self.entries if e.pinned]

    def next_dist(self, context):
        if len(context) > self.context_cap:
            raise ValueError("context exceeds context_cap")
        p = np.zeros(self.vocab_size)
        p[int(torch.argmax(self.logits(context)))] = 1.0
        return self.P(p)


def _splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def request_key(rid: str) -> int:
    """engine.py: zlib.crc32(request id) & 0x7FFFFFFF."""
    return zlib.crc32(str(rid).encode()) & 0x7FFFFFFF


def inject_u(seed: int, key: int, k: int, p: int) -> float:
    """csrc/spec.cu draft_commit_kernel's uniform (fp32)."""
    h = _splitmix64(seed ^ _splitmix64(((key << 40) ^ (k << 32) ^ p) & ((1 << 64) - 1)))
    return float(np.float32(h >> 40) * np.float32(1.0 / 16777216.0))


class FidelityDrafter:
    """Drafter k with the bench's fidelity injection (module docstring)."""

    def __init__(self, base: PrefixCachedOracle, k: int, fidelity: float, requests, teacher: dict,
                 seed: int = 0):
        self.base, self.k, self.f, self.seed = base, k, float(fidelity), seed
        self.vocab_size, self.context_cap = base.vocab_size, base.context_cap
        self.req = [(list(r.prompt), request_key(r.id), teacher.get(r.id, [])) for r in requests]

    def next_dist(self, context):
        tok = int(torch.argmax(self.base.logits(context)))  # the drafter's forward, always computed
        p = len(context)
        for prompt, key, seq in self.req:
            if list(context[: len(prompt)]) == prompt:
                i = p - len(prompt)
                if 0 <= i < len(seq) and inject_u(self.seed, key, self.k, p) < np.float32(self.f):
                    tok = int(seq[i])
                break
        d = np.zeros(self.vocab_size)
        d[tok] = 1.0
        return self.base.P(d)


# ------------------------------------------------------------ timed runs
def reference_run(target_name: str, ssm_name: str, fidelity, n_requests: int, prompt_len: int,
                  new_tokens: int, schedule: str, steps: int, warmup: int, threads: int | None = None,
                  shared_layers: bool | None = None, s_init: int = 4, adaptive: bool = True,
                  log=None) -> dict:
    """Time `steps` complete runs (after `warmup`) of the reference engine over
    `n_requests` bench requests (req-000.., the bench's prompts) generating
    `new_tokens` each.  Prompt prefill, weights and the fidelity teacher are
    untimed setup (the GPU arm's `value` also starts from prefilled caches)."""
    aggspec, ref_path = import_reference()
    from aggspec.core import EngineConfig, ProbDist, Request, seeded_rng
    from aggspec.oracles import CostModel

    from paper_2402_15678_b200.weights import CONFIGS, LlamaWeights, OPTWeights  # torch-only, no libminions

    n_thr = threads or len(os.sched_getaffinity(0))
    torch.set_num_threads(n_thr)
    tcfg, scfg = CONFIGS[target_name], CONFIGS[ssm_name]
    if shared_layers is None:
        shared_layers = tcfg.n_layers * tcfg.d * tcfg.d > 4e9  # > ~16 GB of fp32 weights: share one layer
    t0 = time.perf_counter()
    W = LlamaWeights if tcfg.family == "llama" else OPTWeights
    import dataclasses
    wt = W.random(dataclasses.replace(tcfg, n_layers=1) if shared_layers else tcfg, 0, device="cpu")
    target = PrefixCachedOracle(DecoderF32(wt.t, tcfg, shared_layers=shared_layers), ProbDist,
                                cache_len=prompt_len + new_tokens + 32)
    del wt
    K = len(fidelity)
    Ws = LlamaWeights if scfg.family == "llama" else OPTWeights
    bases = [PrefixCachedOracle(DecoderF32(Ws.random(scfg, k + 1, device="cpu").t, scfg), ProbDist,
                                cache_len=prompt_len + new_tokens + 32) for k in range(K)]
    t_weights = time.perf_counter() - t0

    rng = seeded_rng(0, "workload")  # bench.make_requests (aggspec/bench.py:177-186)
    prompts = [[int(t) for t in rng.integers(0, tcfg.vocab, size=prompt_len)] for _ in range(n_requests)]
    ids = [f"req-{i:03d}" for i in range(n_requests)]
    t0 = time.perf_counter()
    for p in prompts:
        target.pin(p)
        for b in bases:
            b.pin(p)
    t_prefill = time.perf_counter() - t0
    # fidelity teacher: the target's greedy continuation (untimed, as on the GPU arm)
    t0 = time.perf_counter()
    teacher = {}
    for rid, p in zip(ids, prompts):
        ctx = list(p)
        for _ in range(new_tokens):
            ctx.append(int(torch.argmax(target.logits(ctx))))
        teacher[rid] = ctx[len(p):]
    t_teacher = time.perf_counter() - t0
    target.reset()

    def fresh():
        return [Request(id=i, prompt=list(p), max_new_tokens=new_tokens) for i, p in zip(ids, prompts)]

    drafters = [FidelityDrafter(b, k, fidelity[k], fresh(), teacher) for k, b in enumerate(bases)]
    cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=n_requests, b_ssm=n_requests, s_init=s_init, s_min=1,
                       s_max=12, initial_weights=(1.0,) * K, seed=0)
    cost = CostModel(c0=2.5, c1=0.1, d0=56.5, d1=0.75, d2=0.25)
    runner = aggspec.engine.run_pipelined if schedule == "pipelined" else aggspec.engine.run_sequential
    times, toks, acc, lossless = [], [], [], True
    calls = {"target": 0, "drafters": 0}
    for it in range(warmup + steps):
        target.reset()
        for b in bases:
            b.reset()
        c0 = target.calls, sum(b.calls for b in bases)
        reqs = fresh()
        t0 = time.perf_counter()
        metrics, trace = runner(reqs, drafters, target, cost, cfg, adaptive=adaptive, clock="simulated")
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
            toks.append(sum(len(r.generated) for r in reqs))
            acc += [a for e in trace if e.kind == "verify" for a in e.accepted]
            lossless &= all(list(r.generated) == teacher[r.id] for r in reqs)
            calls["target"] += target.calls - c0[0]
            calls["drafters"] += sum(b.calls for b in bases) - c0[1]
        if log:
            log(f"reference step {it}: {dt:.2f}s, {sum(len(r.generated) for r in reqs)} tokens")
    return {"value": sum(toks) / sum(times), "unit": "tokens/s", "cores": n_thr, "kind": "reference",
            "tokens": sum(toks), "seconds": sum(times), "step_s": times,
            "mean_accepted_length": float(np.mean(acc)) if acc else 0.0, "lossless_vs_greedy": lossless,
            "oracle_calls_per_step": {k: v / max(steps, 1) for k, v in calls.items()},
            "setup_s": {"weights": round(t_weights, 1), "prefill": round(t_prefill, 1),
                        "teacher": round(t_teacher, 1)},
            "shared_layers": shared_layers, "reference_src": ref_path,
            "sample": (f"{n_requests} request(s) x {new_tokens} new tokens of the bench workload "
                       f"(prompts req-000.. {prompt_len} tokens), {schedule} aggspec engine "
                       f"(baseline/_ref, unmodified) over fp32 CPU ModelOracles: {target_name}"
                       f"{' (one random layer run ' + str(tcfg.n_layers) + 'x: full per-token FLOPs/bytes)' if shared_layers else ''}"
                       f" + {K}x {ssm_name} with fidelity {list(fidelity)}, prefix-KV-cached next_dist; "
                       f"{steps} complete runs timed (wall clock, no scaling), prompt prefill untimed")}
