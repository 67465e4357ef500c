"""N>1 plumbing on CPU with gloo, world_size 2: request sharding covers every
request exactly once; the timing/token reductions bench.py uses are
max/sum over ranks; barrier works."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_15678_b200 import dist as D
        from paper_2402_15678_b200.core import Request
        reqs = [Request(f"req-{i:03d}", [1, 2, 3], 8) for i in range(33)]
        mine = D.shard_requests(reqs, rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, [r.id for r in mine])
        D.barrier()
        mx = D.max_over_ranks(float(rank + 1) * 1.5)
        sm = D.sum_over_ranks(float(len(mine)))
        q.put((rank, ids, mx, sm, D.world()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharding_and_reductions():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ids, mx, sm, w in out:
        flat = [i for part in ids for i in part]
        assert sorted(flat) == [f"req-{i:03d}" for i in range(33)]  # each request exactly once
        assert abs(len(ids[0]) - len(ids[1])) <= 1
        assert mx == 3.0 and sm == 33.0
        assert w == (rank, world, rank)


def test_single_process_reductions_are_identity():
    from paper_2402_15678_b200 import dist as D
    assert D.max_over_ranks(2.5) == 2.5 and D.sum_over_ranks(4.0) == 4.0
    assert D.shard_requests(list(range(5)), 0, 1) == [0, 1, 2, 3, 4]


def _tp_host_worker(rank, world, port, q, synced):
    """One rank of the tensor-parallel engine's host path: identical device
    results on every rank (the TP forward is bitwise identical across ranks),
    rank-dependent local verify times, selector time through sync_time."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        from paper_2402_15678_b200 import dist as D
        from paper_2402_15678_b200.core import EngineConfig, Request, RequestState
        from paper_2402_15678_b200.rounds import commit_round
        from paper_2402_15678_b200.selector import SelectorState
        from paper_2402_15678_b200.voting import WeightTable
        K, B = 3, 8
        cfg = EngineConfig(vocab_size=100, b_llm=B, b_ssm=B, s_init=4, s_min=1, s_max=12,
                           initial_weights=(1.0,) * K, seed=0)
        reqs = [Request(f"req-{i:03d}", [1, 2, 3], 300) for i in range(B)]
        ctx = [list(r.prompt) for r in reqs]
        cached = [[len(c) - 1 for c in ctx] for _ in range(K)]
        weights, sel = WeightTable.from_config(list(range(K)), cfg), SelectorState.from_config(cfg)
        sync = D.sync_time_fn("cpu") if synced else (lambda ms: ms)
        dev = np.random.default_rng(7)           # "device results": identical on every rank
        local = np.random.default_rng(100 + rank)  # per-rank timing noise
        log = []
        for rnd in range(60):
            act = [b for b, r in enumerate(reqs) if r.state != RequestState.FINISHED]
            if not act:
                break
            s = sel.current_s
            for b in act:
                reqs[b].advance(RequestState.DRAFTING)
            drafts = dev.integers(0, 4, size=(B, K, s)).astype(np.int32)
            voted = dev.integers(0, K, size=B).astype(np.int32)
            n_acc = dev.integers(0, s + 1, size=B).astype(np.int32)
            emitted = np.zeros((B, s + 1), np.int32)
            n_emit = np.zeros(B, np.int32)
            for b in act:
                emitted[b, : n_acc[b]] = drafts[b, voted[b], : n_acc[b]]
                emitted[b, n_acc[b]] = 5
                n_emit[b] = min(n_acc[b] + 1, reqs[b].remaining)
            # rank-dependent cost curve: the two ranks' local times rank s differently
            t_local = 20.0 + (1.5 if rank == 0 else -1.0) * s + local.normal(0, 2.0)
            t_sel = sync(t_local)
            out = commit_round(reqs, ctx, cached, act, s, n_acc, n_emit, emitted, voted, drafts, weights, sel,
                               cfg, t_sel, rnd, adaptive=True)
            log.append((s, out.decision.value, out.s_next, round(out.vl, 9),
                        tuple(round(weights.weights[k], 12) for k in range(K))))
        q.put((rank, log, [list(r.generated) for r in reqs], [c[:] for c in cached]))
    finally:
        dist.destroy_process_group()


def _run_tp_host(synced):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_host_worker, args=(r, world, port, q, synced)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_tp_engine_host_path_identical_decisions_over_gloo():
    """The TP engine's host logic (rounds.commit_round + sync_time, what every
    rank of SpecEngine runs after reading identical device results) makes the
    same decisions on both ranks; without sync_time the local clocks drive the
    selectors apart — the synchronisation is what keeps the ranks in step."""
    (_, log0, gen0, c0), (_, log1, gen1, c1) = _run_tp_host(True)
    assert log0 == log1 and gen0 == gen1 and c0 == c1
    assert len({e[0] for e in log0}) > 1  # the selector did move s
    (_, u0, _, _), (_, u1, _, _) = _run_tp_host(False)
    assert [e[0] for e in u0] != [e[0] for e in u1]
