"""Weighted-majority drafting (mirrors aggspec/voting.py) on the K4 vote kernel.

Reference API kept verbatim: `WeightTable`, `SpeculationTree`, `MajorityOutput`,
`merge`, `select_majority`, `record_acr`, `update_weights`, plus the errors
`LengthMismatch` / `UnknownSSM`.  The trie of the reference (voting.py:83-111)
is never materialised: `merge` validates and packs the drafts into the device
layout and `select_majority` runs `ms_vote` (csrc/vote.cu) on it.  The batched
engine path calls `vote_batch` directly on [B, K, S] device tensors.

`record_acr` / `update_weights` stay on the host in fp64 with the reference's
exact arithmetic (voting.py:142-170): they run once per verify batch on K
scalars, and their result is the fp64 weight vector the next vote kernel reads.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Hashable, Mapping, Sequence

import numpy as np
import torch

from . import _dev
from . import _native
from .core import AggSpecError, EngineConfig, LengthMismatch, ProbDist, UnknownSSM

__all__ = ["LengthMismatch", "UnknownSSM", "WeightTable", "SpeculationTree", "MajorityOutput",
           "merge", "select_majority", "record_acr", "update_weights", "vote_batch",
           "drafter_ranks"]


@dataclass
class WeightTable:
    """Per-drafter fp64 weights plus the ACRs logged since the last update
    (aggspec/voting.py:36-61)."""

    weights: dict[Hashable, float]
    acr_log: dict[Hashable, list[float]] = field(default_factory=dict)
    w_floor: float = 1e-3
    w_cap: float = 1e3

    def __post_init__(self):
        if any(w <= 0 for w in self.weights.values()):
            raise ValueError("all weights must be > 0")
        for sid in self.weights:
            self.acr_log.setdefault(sid, [])

    @classmethod
    def from_config(cls, ssm_ids: Sequence[Hashable], cfg: EngineConfig) -> "WeightTable":
        if len(cfg.initial_weights) != len(ssm_ids):
            raise ValueError(f"initial_weights has {len(cfg.initial_weights)} entries "
                             f"for {len(ssm_ids)} drafters")
        return cls(weights=dict(zip(ssm_ids, cfg.initial_weights)))

    def snapshot(self) -> dict[Hashable, float]:
        return dict(self.weights)


@dataclass
class SpeculationTree:
    """Packed drafts awaiting the vote: the device form of the reference's trie.

    `ids` are the drafter ids in draft order, `tokens` [K, S] int32 and
    `weights` [K] fp64 the per-draft weights looked up at merge time.
    """

    ids: list
    tokens: np.ndarray
    weights: np.ndarray
    depth: int


@dataclass
class MajorityOutput:
    """Voted draft queued for verification (aggspec/voting.py:64-76)."""

    tokens: list[int]
    dists: list[ProbDist] | None
    voted_ssm: Hashable
    request_id: Any = None

    @property
    def s_used(self) -> int:
        return len(self.tokens)


def _weights_of(weights) -> Mapping[Hashable, float]:
    return weights.weights if isinstance(weights, WeightTable) else weights


def drafter_ranks(ids: Sequence[Hashable]) -> np.ndarray:
    """rank[k] = position of ids[k] in sorted(ids): the kernel's stand-in for
    `min(node.contributors)` (aggspec/voting.py:132)."""
    order = sorted(range(len(ids)), key=lambda k: ids[k])
    rank = np.empty(len(ids), np.int32)
    rank[order] = np.arange(len(ids), dtype=np.int32)
    return rank


def merge(drafts: Sequence[tuple[Hashable, Sequence[int]]], weights) -> SpeculationTree:
    """Validate and pack equal-length drafts (same errors as aggspec/voting.py:83-111)."""
    if not drafts:
        raise ValueError("at least one draft is required")
    w = _weights_of(weights)
    depth = len(drafts[0][1])
    if depth < 1:
        raise LengthMismatch("draft sequences must be non-empty")
    ids, rows, ws = [], [], []
    for sid, seq in drafts:
        if len(seq) != depth:
            raise LengthMismatch(f"draft for {sid!r} has length {len(seq)}, expected {depth}")
        if sid not in w:
            raise UnknownSSM(f"no weight for drafter {sid!r}")
        ids.append(sid)
        rows.append([int(t) for t in seq])
        ws.append(float(w[sid]))
    return SpeculationTree(ids=ids, tokens=np.asarray(rows, np.int32),
                           weights=np.asarray(ws, np.float64), depth=depth)


def vote_batch(tokens: torch.Tensor, weights: torch.Tensor, rank: torch.Tensor | None = None,
               *, path: torch.Tensor | None = None, voted: torch.Tensor | None = None,
               stream: torch.cuda.Stream | None = None):
    """Batched K4: tokens [B, K, S] int32, weights [K] fp64 (draft order),
    rank [K] int32 or None → (path [B, S] int32, voted draft index [B] int32)."""
    dev = _dev.require_cuda()
    if tokens.dim() != 3:
        raise ValueError("tokens must be [B, K, S]")
    B, K, S = tokens.shape
    if path is None:
        path = torch.empty((B, S), dtype=torch.int32, device=dev)
    if voted is None:
        voted = torch.empty((B,), dtype=torch.int32, device=dev)
    if weights.numel() != K or (rank is not None and rank.numel() != K):
        raise LengthMismatch(f"expected {K} weights/ranks")
    _native.call("ms_vote", _dev.ptr(tokens, torch.int32, "tokens"),
                 _dev.ptr(weights, torch.float64, "weights"),
                 _dev.ptr(rank, torch.int32, "rank"), B, K, S,
                 _dev.ptr(path, torch.int32, "path"), _dev.ptr(voted, torch.int32, "voted"),
                 _dev.stream_ptr(stream))
    return path, voted


def select_majority(tree: SpeculationTree,
                    drafts: Mapping[Hashable, tuple[Sequence[int], Sequence[ProbDist]]] | None = None,
                    request_id: Any = None) -> MajorityOutput:
    """Majority path + voted drafter (aggspec/voting.py:114-139) via ms_vote."""
    dev = _dev.require_cuda()
    tok = torch.from_numpy(tree.tokens).to(dev).reshape(1, *tree.tokens.shape)
    w = torch.from_numpy(tree.weights).to(dev)
    rank = torch.from_numpy(drafter_ranks(tree.ids)).to(dev)
    path, voted = vote_batch(tok, w, rank)
    p = path[0].tolist()
    vsid = tree.ids[int(voted[0])]
    dists = None
    if drafts is not None:
        toks, cand = drafts[vsid]
        if list(toks) != p:
            raise AggSpecError("voted drafter's sequence does not match the selected path")
        dists = list(cand)
    return MajorityOutput(tokens=p, dists=dists, voted_ssm=vsid, request_id=request_id)


def record_acr(weights: WeightTable, voted_ssm: Hashable, rate: float) -> WeightTable:
    """Log one verification's acceptance rate (aggspec/voting.py:142-149)."""
    if voted_ssm not in weights.weights:
        raise UnknownSSM(f"unknown drafter {voted_ssm!r}")
    if not (0.0 <= rate <= 1.0):
        raise ValueError("acceptance rate must be in [0, 1]")
    weights.acr_log[voted_ssm].append(rate)
    return weights


def update_weights(weights: WeightTable, cfg: EngineConfig) -> WeightTable:
    """Reward/punish once per verify batch, clamp, clear the log
    (aggspec/voting.py:152-170; fp64, sequential mean)."""
    for sid, rates in weights.acr_log.items():
        if not rates:
            continue
        acr = sum(rates) / len(rates)
        w = weights.weights[sid]
        if acr >= cfg.reward_threshold:
            w *= cfg.reward_factor
        elif acr <= cfg.punish_threshold:
            w *= cfg.punish_factor
        weights.weights[sid] = min(max(w, weights.w_floor), weights.w_cap)
        rates.clear()
    return weights
