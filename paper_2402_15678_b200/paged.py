"""Paged KV cache (the vLLM-style block manager extended
with per-token slot deletion for rejected speculative tokens).

The reference keeps no KV cache at all (ModelOracle.next_dist recomputes from
the full context, aggspec/oracles.py:19-26); its "rollback" is implicit in
request.generated (aggspec/engine.py:300-315).  On the device the verifier's
KV must follow that: a round writes K/V for s+1 speculative positions, only
n_acc+1 of them survive.

Layout: per layer a block pool [n_blocks, Hkv, block_size, D] bf16 for K and
for V, and one block table [slots, max_blocks] int32 shared by all layers
(csrc/attention.cu, csrc/model.cu: position t of a slot lives in block
table[slot][t // bs], row t % bs).  The kernels' arithmetic is the same as
with the contiguous cache — only K/V row addresses change (tested bitwise).

BlockManager (host): before a round `ensure(slot, n)` grows a sequence to
cover positions [0, n) (the verify writes up to len(ctx) + s); after the
accept `truncate(slot, valid)` returns every block that lies entirely past the
accepted length to the free list — the KV of rejected tokens; `release(slot)`
frees a finished request.  The pool can be smaller than slots x max_len
(over-subscription for variable-length serving): ensure() raises when empty.
"""
from __future__ import annotations

import numpy as np
import torch

BF16 = torch.bfloat16


class KVPoolExhausted(RuntimeError):
    pass


class BlockManager:
    def __init__(self, n_blocks: int, slots: int, max_blocks: int, block_size: int):
        self.n_blocks, self.slots, self.max_blocks, self.bs = n_blocks, slots, max_blocks, block_size
        self.free = list(range(n_blocks - 1, -1, -1))  # pop() hands out low ids first
        self.owned: list[list[int]] = [[] for _ in range(slots)]
        # unassigned entries point at a scratch block (pool index n_blocks, never
        # handed out): the fixed-shape verify graph still writes K/V rows for
        # finished / padding slots, and those writes must not land in a live block
        self.scratch = n_blocks
        self.table = torch.full((slots, max_blocks), n_blocks, dtype=torch.int32,
                                pin_memory=torch.cuda.is_available())
        self.dirty = True

    def blocks_for(self, n_tokens: int) -> int:
        return (n_tokens + self.bs - 1) // self.bs

    def ensure(self, slot: int, n_tokens: int) -> None:
        need = self.blocks_for(n_tokens)
        if need > self.max_blocks:
            raise ValueError(f"{n_tokens} positions exceed max_blocks * block_size")
        own = self.owned[slot]
        while len(own) < need:
            if not self.free:
                raise KVPoolExhausted(f"KV block pool of {self.n_blocks} blocks exhausted")
            b = self.free.pop()
            self.table[slot, len(own)] = b
            own.append(b)
            self.dirty = True

    def truncate(self, slot: int, n_tokens: int) -> int:
        """Free the blocks past position n_tokens; returns how many."""
        keep = self.blocks_for(n_tokens)
        own = self.owned[slot]
        n = 0
        while len(own) > keep:
            self.free.append(own.pop())
            self.table[slot, len(own)] = self.scratch
            n += 1
        if n:
            self.dirty = True
        return n

    def release(self, slot: int) -> int:
        return self.truncate(slot, 0)

    def used(self) -> int:
        return self.n_blocks - len(self.free)


class PagedKVCache:
    """Per-layer K/V block pools + one block table; drop-in for opt.KVCache
    (models pass cache.page to the attention kernel)."""

    def __init__(self, cfg, slots: int, max_len: int, block_size: int = 16, n_blocks: int | None = None,
                 device="cuda"):
        self.slots, self.bs = slots, block_size
        self.max_blocks = (max_len + block_size - 1) // block_size
        self.max_len = self.max_blocks * block_size
        self.n_blocks = n_blocks if n_blocks is not None else slots * self.max_blocks
        shape = (self.n_blocks + 1, cfg.n_kv_heads, block_size, cfg.head_dim)  # + the scratch block
        self.k = [torch.zeros(shape, dtype=BF16, device=device) for _ in range(cfg.n_layers)]
        self.v = [torch.zeros(shape, dtype=BF16, device=device) for _ in range(cfg.n_layers)]
        self.table = torch.full((slots, self.max_blocks), self.n_blocks, dtype=torch.int32, device=device)
        self.page = (self.table, block_size)
        self.mgr = BlockManager(self.n_blocks, slots, self.max_blocks, block_size)

    def nbytes(self) -> int:
        return sum(t.numel() * 2 for t in self.k + self.v)

    def upload(self, rows: slice | None = None, stream=None) -> int:
        """Copy the host block table (or rows of it) to the device, stream-ordered."""
        if not self.mgr.dirty and rows is None:
            return 0
        src = self.mgr.table if rows is None else self.mgr.table[rows]
        dst = self.table if rows is None else self.table[rows]
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            dst.copy_(src, non_blocking=True)
        if rows is None:
            self.mgr.dirty = False
        return src.numel() * 4
