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
