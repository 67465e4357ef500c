"""Benchmark of the speculate-vote-verify hot path (BASELINE.json metric:
output tokens/s + mean accepted length).

Workload at N=1: the configuration BASELINE.json's metric is quoted on —
Llama-2-70B target + 3 x Llama-160M drafters — which fits one B200 (137.4 GB
of bf16 weights in 180 GB): bf16, verify batch 16, pipelined SSM decode / LLM
verify as cfg3 specifies (two request groups of 16: the drafters draft one
while the verifier verifies the other), adaptive speculation length (s_init
4, s in [1, 12]), greedy, 128-token synthetic prompts, 128 new tokens per
request.  --schedule sequential runs one group of 16.  `--target opt-13b --ssm opt-125m` runs configs[1] (cfg2).
Random-init weights (no checkpoints offline); because random-init drafters
never agree with the target, drafts use fidelity injection
(engine.py / DESIGN.md): with probability f_k SSM k's drafted token is
replaced by the target's greedy continuation — every kernel still runs in
full and the output stays exactly the target's greedy decode.

One step = one generation batch: decode of 16 requests x 128 new tokens (x2
groups pipelined), from prefilled KV caches, the speculation-length selector and
the drafter weights starting from the config (--controllers fresh, default: the
reference engine's per-run semantics; warm = they persist across steps, both
reported) (prompt prefill is outside the hot path) to
the last request finishing.  `value` = generated tokens / device time of the
decode (CUDA events, weights 137 GB >> L2 so no flush is needed).  `e2e` =
the same metric through the public API (SpecEngine.run) from host prompt
lists, H2D of prompts + per-round metadata and D2H of per-round results
inside the timed region, prompt prefill included.

--impl reference: the reference's own CPU path, timed on the host cores —
the UNMODIFIED reference engine (aggspec run_pipelined / run_sequential from
baseline/_ref) driving fp32 CPU ModelOracles of the same model shapes, with
the same fidelity injection (oracle/cpu_path.py).  A step is a bounded sample
of the workload: --ref-requests request(s) of the bench's prompt set
generating --ref-new-tokens tokens each, timed end to end by wall clock; no
scaling or extrapolation.  The GPU arm's `cpu_baseline` is one such step.

Multi-GPU (torchrun, N>1), --parallelism tp (default): the verifier is
tensor parallel over the N ranks (Megatron split; the sums over ranks are
libminions' fixed-order reductions over CUDA-IPC peer memory), the drafters
are replicated, every rank serves the same global batch of 16 (strong
scaling); value = tokens / max-over-ranks time.  --parallelism replicas: every
rank runs the single-GPU workload on its own batch (weak scaling, no
data-path collective).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "output tokens/sec, Llama-2-70B + 3x160M SSMs, 1-8 B200; mean accepted length"


def workload(args) -> str:
    sched = ("pipelined SSM decode / LLM verify (2 groups)" if args.schedule == "pipelined"
             else "sequential draft / verify")
    k = len(args.fidelity.split(",")) if args.fidelity else 3
    if args.target == "llama-2-70b":
        return (f"cfg3: Llama-2-70B target + {k}x {args.ssm} SSMs, bf16, verify batch {args.batch}, {sched}, "
                f"adaptive s")
    if args.preset == "cfg1":
        return (f"cfg1: tiny OPT-style target (4L d256) + {k}x tiny 1L SSMs, batch {args.batch}, s={args.fixed_s}, "
                f"greedy, {args.new_tokens} new tokens, no fidelity injection")
    if args.preset == "cfg5":
        return (f"cfg5 on one GPU: Llama-2-13B target + {k}x {args.ssm} SSMs, {args.prompt_len}-token prompts, "
                f"bf16, verify batch {args.batch}, {sched}, adaptive s (KV-cache-bound verify)")
    return (f"{args.target} target + {k}x {args.ssm} SSMs, bf16, verify batch {args.batch}, {sched}, adaptive s")


def data_note(args) -> str:
    return "synthetic prompts, random-init weights" + (", fidelity-injected drafts" if args.fidelity else "")


def bench_config(args, ws: int, tp: bool) -> dict:
    """The workload description both arms print (same dict: same_config)."""
    from paper_2402_15678_b200.weights import CONFIGS  # torch-only (no libminions)
    tcfg = CONFIGS[args.target]
    fid = [float(x) for x in args.fidelity.split(",")] if args.fidelity else None
    K = len(fid) if fid else 3
    n_req = args.batch * (2 if args.schedule == "pipelined" else 1)
    return {"workload": workload(args), "target": args.target, "ssms": [args.ssm] * K,
            "global_batch": n_req * (1 if tp else ws), "schedule": args.schedule,
            "prompt_len": args.prompt_len,
            "new_tokens": args.new_tokens, "s_init": args.fixed_s or 4,
            "s_range": [args.fixed_s] * 2 if args.fixed_s else [1, 12], "greedy": True,
            "fidelity": fid,
            "parallelism": (f"tp{ws}" if tp else "replicas") if ws > 1 else "single-gpu",
            "l2": (f"inputs larger than L2 ({2 * tcfg.matmul_params() / 1e9:.1f} GB of weights "
                   "streamed per verify)"),
            "controllers": ("selector + drafter weights reset to the config at every step (as the reference "
                            "engine starts each run, aggspec/engine.py:209-210)" if args.controllers == "fresh" else
                            "selector + drafter weights persist across batches (adapted in warm-up)"),
            "kv_cache": f"paged, {args.kv_block_size}-token blocks" if args.kv_block_size else "contiguous",
            "sm_partition": (f"drafters on a {args.draft_sms}-SM green context, verifier on the rest"
                             if args.draft_sms and args.schedule == "pipelined" else "shared")}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--target", default="llama-2-70b")
    ap.add_argument("--ssm", default="llama-160m")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt-len", type=int, default=128)
    ap.add_argument("--new-tokens", type=int, default=128)
    ap.add_argument("--fidelity", default="0.9,0.85,0.8",
                    help="one per drafter (the drafter count is the number of values)")
    ap.add_argument("--preset", default="", choices=["", "cfg1", "cfg2", "cfg5"],
                    help="cfg1: the reference's own CPU-runnable case (tiny OPT 4L d256 + 3x 1L, B=4, s=4, "
                         "64 new tokens, no fidelity injection; the reference arm runs it in full); "
                         "cfg2: OPT-13B + 3x OPT-125M, sequential; cfg5: Llama-2-13B + 5 drafters, 4K prompts "
                         "(verify batch 16 x 2 pipelined groups on one GPU: B=64 needs ~218 GB of KV)")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-requests", type=int, default=0,
                    help="reference arm / cpu_baseline sample: requests per step (0: 1, cfg1: all)")
    ap.add_argument("--ref-new-tokens", type=int, default=0,
                    help="reference arm / cpu_baseline sample: new tokens per request per step "
                         "(0: 4, cfg1: all)")
    ap.add_argument("--controllers", default="fresh", choices=["fresh", "warm"],
                    help="fresh: the selector and drafter weights restart from the config every step (the reference "
                         "engine's per-run semantics); warm: they persist across steps")
    ap.add_argument("--fresh-steps", type=int, default=-1,
                    help="extra timed steps with the selector and drafter weights reset per step "
                         "(the reference's per-run semantics); -1 = min(steps, 3), 0 = skip")
    ap.add_argument("--fixed-s", type=int, default=0, help="disable the adaptive selector, use this s")
    ap.add_argument("--kv-block-size", type=int, default=0,
                    help="> 0: the verifier's KV cache is paged with this block size (paged.PagedKVCache)")
    ap.add_argument("--parallelism", default="tp", choices=["tp", "replicas"],
                    help="N>1: tensor-parallel verifier over the ranks (default, SURVEY §8e) or one full "
                         "replica per GPU serving its own batch")
    ap.add_argument("--draft-sms", type=int, default=0,
                    help="pipelined: SMs of the drafters' green context (the verifier gets the rest); 0 = shared")
    ap.add_argument("--schedule", default="pipelined", choices=["sequential", "pipelined"],
                    help="pipelined (cfg3, default): two request groups of --batch each (verify batch "
                         "--batch, 2x requests in flight), verify of one overlapping drafting of the "
                         "other (aggspec/engine.py:494-576); sequential: one group, draft then verify")
    a = ap.parse_args()
    if a.preset == "cfg1":
        a.target, a.ssm, a.schedule, a.batch = "tiny-target", "tiny-ssm", "sequential", 4
        a.prompt_len, a.new_tokens, a.fixed_s, a.fidelity = 8, 64, 4, ""
    elif a.preset == "cfg2":
        a.target, a.ssm, a.schedule = "opt-13b", "opt-125m", "sequential"
    elif a.preset == "cfg5":
        a.target, a.ssm, a.prompt_len = "llama-2-13b", "llama-160m", 4096
        a.fidelity = "0.9,0.85,0.8,0.75,0.7"
    full = a.preset == "cfg1"
    a.ref_requests = a.ref_requests or (a.batch if full else 1)
    a.ref_new_tokens = a.ref_new_tokens or (a.new_tokens if full else 4)
    return a


# --------------------------------------------------------------------------- dist
def dist_init():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        # MS_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo plumbing — a
        # functional test of the multi-process path on a one-GPU box (NCCL
        # refuses two ranks on one GPU); never a performance configuration
        if os.environ.get("MS_BENCH_SHARE_GPU", "0") == "1":
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, ws, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    from paper_2402_15678_b200.dist import max_over_ranks as mx
    return mx(x, device="cuda") if ws > 1 else x


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                row = [c.strip() for c in out.split(",")] if out else []
                if len(row) == 6:
                    self.rows.append(row)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        import statistics
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# -------------------------------------------------------------------- workload
def make_requests(n, prompt_len, new_tokens, vocab, seed=0):
    """make_requests semantics of aggspec/bench.py:177-186: ids req-%03d,
    prompt tokens uniform in [0, V) from seeded_rng(seed, "workload")."""
    from paper_2402_15678_b200.core import Request, seeded_rng
    rng = seeded_rng(seed, "workload")
    return [Request(f"req-{i:03d}", [int(t) for t in rng.integers(0, vocab, size=prompt_len)], new_tokens)
            for i in range(n)]


def fresh(reqs):
    from paper_2402_15678_b200.core import Request
    return [Request(r.id, list(r.prompt), r.max_new_tokens) for r in reqs]


def roofline_verify(engine, rounds, peaks):
    """Dominant unit: the verify forward (4 ms_linear GEMMs per layer + LM
    head + attention), timed per round with CUDA events on its stream.
    Algorithmic bytes per round = 2 * matmul params (bf16 weights) + KV read
    (B * ctx * kv_bytes_per_token) + KV write (B * (s+1) * kv_bytes_per_token)."""
    c = engine.target.cfg
    P2 = 2 * c.matmul_params()
    kvb = c.kv_bytes_per_token()
    vb = engine.groups[0].B  # rows of one verify (one group's slots)
    tot_bytes = tot_t = 0.0
    for r in rounds:
        ctx = r.ctx_mean
        nb = len(r.accepted) if r.accepted else vb
        b = P2 + nb * ctx * kvb + nb * (r.s + 1) * kvb
        tot_bytes += b
        tot_t += r.t_verify_ms * 1e-3
    ach = tot_bytes / tot_t / 1e9
    # measured copy bandwidth (MEASURED_PEAKS.json, driver-written) or the
    # fallback of B200_PROFILING.md (6.65 TB/s) when the file is absent
    peak = peaks.get("hbm_gbs")
    src = "measured"
    if not peak:
        peak, src = 6650.0, "fallback"
    traffic, tnote = None, None
    try:  # ncu --metrics dram__bytes_{read,write}.sum of one verify forward (profiles/)
        with open(os.path.join(ROOT, "profiles", "r1n_verify_traffic.json")) as fh:
            tr = json.load(fh)
        if tr["model"] == c.name.split("/")[0] and vb == tr["B"] and not getattr(engine, "tp", False):
            traffic = tr["dram_bytes"]
            tnote = (f"ncu DRAM bytes of one verify forward at Q={tr['Q']}, ctx={tr['ctx']} "
                     f"(algorithmic {tr['algorithmic_bytes']} B: {tr['dram_bytes'] / tr['algorithmic_bytes']:.3f}x)")
    except (OSError, KeyError, ValueError):
        pass
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4), "peak_source": src, "traffic": traffic, "traffic_note": tnote,
            "kernel": "verify forward (ms_linear x4/layer + attention + LM head), per round",
            "bytes_per_launch": round(tot_bytes / max(len(rounds), 1)),
            "mean_ms": round(tot_t * 1e3 / max(len(rounds), 1), 3)}


def run_ours(args, rank, ws):
    import numpy as np
    import torch

    from paper_2402_15678_b200 import _native
    from paper_2402_15678_b200.core import EngineConfig
    from paper_2402_15678_b200.engine import SpecEngine
    from paper_2402_15678_b200.models import config, random_weights

    tcfg, scfg = config(args.target), config(args.ssm)
    fid = [float(x) for x in args.fidelity.split(",")] if args.fidelity else None
    K = len(fid) if fid else 3
    cfg = EngineConfig(vocab_size=tcfg.vocab, b_llm=args.batch, b_ssm=args.batch,
                       s_init=args.fixed_s or 4, s_min=1, s_max=12, initial_weights=(1.0,) * K, seed=0)
    max_len = args.prompt_len + args.new_tokens + cfg.s_max + 4
    pipelined = args.schedule == "pipelined"
    n_req = args.batch * (2 if pipelined else 1)
    tp = ws > 1 and args.parallelism == "tp"
    target = None
    sync = None
    if tp:
        # the verifier tensor-parallel over the ranks (Megatron split,
        # sums over ranks by the peer-memory kernels of csrc/tp.cu), drafters
        # replicated on every rank; one global batch -> strong scaling
        import torch.distributed as tdist
        from paper_2402_15678_b200.tp import LlamaTPModel, TPComm, random_shard
        max_rows = max(n_req * (cfg.s_max + 1), n_req * max_len)
        err = None
        try:
            comm = TPComm.from_process_group(max_rows, tcfg.d)
        except Exception as e:  # e.g. no CUDA IPC / peer access between the GPUs
            err = f"{type(e).__name__}: {e}"
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device="cuda")
        tdist.all_reduce(ok, op=tdist.ReduceOp.MIN)  # every rank fails together
        if int(ok.item()) != 1:
            # never a silent fallback to replicas: --parallelism tp was asked for
            raise RuntimeError(f"tensor-parallel setup failed ({err or 'on a peer rank'}); "
                               "rerun with --parallelism replicas for independent replicas")
        target = LlamaTPModel(random_shard(tcfg, rank, ws, 0), comm, max_rows=max_rows)
        from paper_2402_15678_b200.dist import sync_time_fn
        sync = sync_time_fn("cuda")
    if target is None:
        target = random_weights(tcfg, 0, device="cuda")
    drafters = [random_weights(scfg, k + 1, device="cuda") for k in range(K)]
    eng = SpecEngine(target, drafters, cfg, slots=n_req, max_len=max_len,
                     use_graphs=not args.no_graphs, fidelity=fid, pipelined=pipelined,
                     adaptive=not args.fixed_s, sync_time=sync, kv_block_size=args.kv_block_size,
                     draft_sms=args.draft_sms if pipelined else 0)
    if tp:  # every rank serves the same global batch
        reqs = make_requests(n_req, args.prompt_len, args.new_tokens, tcfg.vocab)
    else:
        # weak scaling: the global request list is n_req per rank; each rank serves
        # its own contiguous slice (requests are independent — no data-path collective)
        from paper_2402_15678_b200.dist import shard_requests
        reqs = shard_requests(make_requests(n_req * ws, args.prompt_len, args.new_tokens, tcfg.vocab), rank, ws)
    eng.capture_graphs()  # every s, before timing (and before prefill)
    teacher = eng.greedy_teacher(fresh(reqs), args.new_tokens) if fid else None

    def one_step(timed_events=True):
        rs = fresh(reqs)
        eng.prefill(rs)
        if teacher is not None:
            eng.set_teacher(teacher)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        n0 = eng.kernel_launches
        e0.record()
        res = eng.decode(reset_controllers=args.controllers == "fresh")
        e1.record()
        torch.cuda.synchronize()
        return res, e0.elapsed_time(e1) * 1e-3, eng.kernel_launches - n0

    for _ in range(args.warmup):
        one_step()
    barrier(ws)
    torch.cuda.synchronize()
    results, t_total, launches = [], 0.0, 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            res, t, nl = one_step()
            results.append(res)
            t_total += t
            launches += nl
    torch.cuda.synchronize()
    barrier(ws)
    lossless = all(r.outputs == teacher for r in results) if teacher else None
    tokens = sum(r.tokens for r in results)
    t_max = max_over_ranks(t_total, ws)
    value = tokens * (1 if tp else ws) / t_max
    rounds = [rd for r in results for rd in r.rounds]
    # mean context per round for the KV term of the roofline
    for r in results:
        ctx = args.prompt_len
        for rd in r.rounds:
            rd.ctx_mean = ctx
            ctx += rd.vl
    acc = [a for rd in rounds for a in rd.accepted]
    emt = [e for rd in rounds for e in rd.emitted]

    # ---- e2e through the public API from host buffers (prefill included)
    barrier(ws)
    torch.cuda.synchronize()
    h0, d0 = eng.h2d_bytes, eng.d2h_bytes
    t0 = time.perf_counter()
    e2e_tokens = 0
    for _ in range(args.steps):
        rs = fresh(reqs)
        eng.prefill(rs)
        if teacher is not None:
            eng.set_teacher(teacher)
            eng.h2d_bytes += eng.teacher.numel() * 4
        res = eng.decode(reset_controllers=args.controllers == "fresh")
        e2e_tokens += res.tokens
    torch.cuda.synchronize()
    t_e2e = max_over_ranks(time.perf_counter() - t0, ws)
    e2e = {"value": round(e2e_tokens * (1 if tp else ws) / t_e2e, 2), "unit": "tokens/s",
           "h2d_bytes_per_step": int((eng.h2d_bytes - h0) / args.steps),
           "d2h_bytes_per_step": int((eng.d2h_bytes - d0) / args.steps),
           "includes": "prompt H2D + prefill + decode + per-round H2D/D2H"}

    # ---- the other controller mode beside the headline one (fresh: selector
    # + drafter weights reset every step, as the reference starts both from the
    # config per run, aggspec/engine.py:209-210; warm: they persist)
    other = "warm" if args.controllers == "fresh" else "fresh"
    n_fresh = min(args.steps, 3) if args.fresh_steps < 0 else args.fresh_steps
    fresh_out = None
    if n_fresh > 0:
        barrier(ws)
        f_tok, f_t, f_acc = 0, 0.0, []
        for _ in range(n_fresh):
            rs = fresh(reqs)
            eng.prefill(rs)
            if teacher is not None:
                eng.set_teacher(teacher)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            res = eng.decode(reset_controllers=other == "fresh")
            e1.record()
            torch.cuda.synchronize()
            f_t += e0.elapsed_time(e1) * 1e-3
            f_tok += res.tokens
            f_acc += [a for rd in res.rounds for a in rd.accepted]
        f_t = max_over_ranks(f_t, ws)
        fresh_out = {"value": round(f_tok * (1 if tp else ws) / f_t, 2), "unit": "tokens/s", "steps": n_fresh,
                     "mean_accepted_length": round(float(np.mean(f_acc)), 4) if f_acc else 0.0,
                     "note": ("selector and drafter weights reset to the config at every step" if other == "fresh"
                              else "selector and drafter weights persist across steps")}

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except Exception:
        pass
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_max / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if tp else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": data_note(args),
        "config": bench_config(args, ws, tp),
        "mean_accepted_length": round(float(np.mean(acc)), 4) if acc else 0.0,
        "mean_emitted_per_round": round(float(np.mean(emt)), 4) if emt else 0.0,
        "rounds_per_step": round(len(rounds) / args.steps, 2),
        "s_trajectory_tail": [rd.s for rd in results[-1].rounds[-8:]],
        "s_hist": {int(k): int(v) for k, v in zip(*np.unique([rd.s for rd in rounds], return_counts=True))},
        "draft_ms_mean": round(float(np.mean([rd.t_draft_ms for rd in rounds])), 3),
        "lossless_vs_greedy": lossless,
        "verify_ms_mean": round(float(np.mean([rd.t_verify_ms for rd in rounds])), 3),
        "round_ms_mean": round(float(np.mean([rd.t_round_ms for rd in rounds])), 3),
        "roofline": roofline_verify(eng, rounds, peaks),
        "e2e": e2e,
        f"{other}_controllers": fresh_out,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "libminions": _native.LIB_PATH,
    }
    return out


# ---------------------------------------------------------------- CPU baseline
def cpu_reference(args, steps: int, warmup: int) -> dict:
    """The reference's CPU path on a bounded sample of this workload
    (oracle/cpu_path.py): complete runs of the unmodified reference engine
    over fp32 CPU ModelOracles, wall clock, all host threads.  Never scaled.
    Prompts of more than 1,024 tokens (cfg5) are not sampled: their CPU
    prefill alone is minutes per request."""
    if args.prompt_len > 1024:
        return {"value": None, "unit": "tokens/s", "cores": len(os.sched_getaffinity(0)), "kind": "reference",
                "sample": f"n/a: {args.prompt_len}-token prompts do not prefill on the CPU in a bounded sample"}
    from oracle.cpu_path import reference_run
    fid = [float(x) for x in args.fidelity.split(",")] if args.fidelity else [0.0, 0.0, 0.0]
    r = reference_run(args.target, args.ssm, fid, args.ref_requests, args.prompt_len, args.ref_new_tokens,
                      args.schedule, steps, warmup, s_init=args.fixed_s or 4, adaptive=not args.fixed_s,
                      log=lambda m: print(m, file=sys.stderr, flush=True))
    return r


def main():
    args = parse()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        cb = cpu_reference(args, args.steps, args.warmup)
        v = round(cb["value"], 6) if cb["value"] is not None else None
        line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                "scaling": "strong" if ws > 1 and args.parallelism == "tp" else "weak", "vs_baseline": None,
                "dtype": "f32", "data": data_note(args),
                "impl": "reference",
                "config": bench_config(args, ws, ws > 1 and args.parallelism == "tp"),
                "mean_accepted_length": round(cb.get("mean_accepted_length", 0.0), 4),
                "lossless_vs_greedy": cb.get("lossless_vs_greedy"),
                "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cb["cores"], "kind": cb["kind"],
                                 "sample": cb["sample"]},
                "reference_detail": {k: cb[k] for k in ("step_s", "setup_s", "oracle_calls_per_step",
                                                        "shared_layers", "reference_src") if k in cb},
                "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    rank, ws, local = dist_init()
    out = run_ours(args, rank, ws)
    if rank == 0:
        if not args.no_cpu_baseline and ws == 1:
            cb = cpu_reference(args, steps=1, warmup=0)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            if cb["value"] is not None:
                out["cpu_baseline"]["value"] = round(cb["value"], 6)
                out["cpu_baseline"]["mean_accepted_length"] = round(cb["mean_accepted_length"], 4)
        print(json.dumps(out))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
