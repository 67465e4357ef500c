"""Tensor-parallel Llama verifier: Megatron split over t ranks
with the sums over ranks done by libminions' fixed-order two-shot reduction
over peer memory (csrc/tp.cu) instead of an NCCL allreduce, so the TP forward
is deterministic, identical on every rank and batch invariant.

Per layer on rank r (H/t query heads, Hkv/t KV heads, F/t MLP columns):

  h    = RMSNorm(x)                         (fused with the wait of the previous sum)
  qkv  = h · W_qkv[r]ᵀ                      column-parallel (q | k | v rows of the rank's heads)
  a    = attention(qkv, KV cache of the rank's KV heads)
  P_r  = a · W_o[:, r]ᵀ (+ x on rank 0)     row-parallel, fp32 partial in the rank's symmetric buffer
  x    = Σ_j P_j (rank order)               signal / reduce-gather / signal
  h    = RMSNorm(x) ; f = silu(h·W_g[r]ᵀ) ⊙ (h·W_u[r]ᵀ) ; P_r = f · W_down[:, r]ᵀ (+ x on rank 0) ; x = Σ_j P_j
LM head vocab-parallel: logits [R, V/t] -> per-rank (value, index) argmax ->
cross-rank first-index argmax (every rank gets the target argmax; no logits
are gathered).

Two ways to build a group:
  TPComm.local_group(t, ...)   all ranks in one process (one GPU, one stream
                               per rank) — the single-GPU test of the protocol
  TPComm.from_process_group()  one process per GPU: symmetric buffers are
                               cudaMalloc'd, exchanged as CUDA IPC handles over
                               torch.distributed, opened on every peer
"""
from __future__ import annotations

import ctypes

import torch

from . import _dev, _native
from . import kernels as K
from .llama import LlamaConfig, LlamaModel, LlamaWeights

BF16 = torch.bfloat16
I64 = torch.int64


class _Region:
    """One rank's symmetric region: flags [3][64] int32 | argmax [R] u64 |
    partial P [R, d] fp32 | residual stream x [R, d] bf16.  Owned as a torch
    tensor (local group) or cudaMalloc'd + IPC-exported (process group)."""

    FLAG_BYTES = 4096

    def __init__(self, max_rows: int, d: int):
        self.max_rows, self.d = max_rows, d
        self.off_am = self.FLAG_BYTES
        self.off_p = self.off_am + ((max_rows * 8 + 255) // 256) * 256
        self.off_x = self.off_p + ((max_rows * d * 4 + 255) // 256) * 256
        self.nbytes = self.off_x + max_rows * d * 2

    def ptrs(self, base: int) -> dict:
        return {"flags": base, "am": base + self.off_am, "p": base + self.off_p, "x": base + self.off_x}


class TPComm:
    """Rank r's view of the group: local buffers as torch tensors, device arrays
    of every rank's buffer pointers, per-flag-set epoch counters."""

    def __init__(self, rank: int, t: int, max_rows: int, d: int, device, local_buf: torch.Tensor,
                 bases: list[int], owner=None, early: bool = False):
        self.rank, self.t, self.max_rows, self.d = rank, t, max_rows, d
        # PDL release before the peer wait: only when every rank has its own GPU
        self.early = int(early)
        self.device = torch.device(device)
        self.reg = _Region(max_rows, d)
        self._buf = local_buf  # uint8 [nbytes] aliasing this rank's region
        self._owner = owner
        off = self.reg
        self.flags = local_buf[: off.FLAG_BYTES].view(torch.int32)  # [3 * 64 + ...]
        self.am = local_buf[off.off_am: off.off_am + max_rows * 8].view(torch.int64)
        self.p = local_buf[off.off_p: off.off_p + max_rows * d * 4].view(torch.float32).view(max_rows, d)
        self.x = local_buf[off.off_x: off.off_x + max_rows * d * 2].view(BF16).view(max_rows, d)
        ps = [off.ptrs(b) for b in bases]
        dev = self.device
        # flag set k of rank j lives at flags_j + k * 64 ints
        self.peer_flags = [torch.tensor([p["flags"] + k * 256 for p in ps], dtype=I64, device=dev) for k in range(3)]
        self.peer_p = torch.tensor([p["p"] for p in ps], dtype=I64, device=dev)
        self.peer_x = torch.tensor([p["x"] for p in ps], dtype=I64, device=dev)
        self.peer_am = torch.tensor([p["am"] for p in ps], dtype=I64, device=dev)
        self.epoch = torch.zeros(3, dtype=torch.int32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        _native.check(_native.lib.ms_preload(), "ms_preload")  # no lazy loads under spin-waits

    # ------------------------------------------------------------ construction
    @classmethod
    def local_group(cls, t: int, max_rows: int, d: int, device="cuda") -> list["TPComm"]:
        """All t ranks in this process on one device (protocol test)."""
        reg = _Region(max_rows, d)
        bufs = [torch.zeros(reg.nbytes, dtype=torch.uint8, device=device) for _ in range(t)]
        bases = [b.data_ptr() for b in bufs]
        return [cls(r, t, max_rows, d, device, bufs[r], bases) for r in range(t)]

    @classmethod
    def from_process_group(cls, max_rows: int, d: int, group=None) -> "TPComm":
        """One process per GPU: cudaMalloc + IPC export, all-gather of the
        handles over torch.distributed, IPC open of every peer's region."""
        import torch.distributed as dist
        rank, t = dist.get_rank(group), dist.get_world_size(group)
        dev = _dev.require_cuda()
        reg = _Region(max_rows, d)
        hsz = int(_native.lib.ms_ipc_handle_size())
        handle = (ctypes.c_char * hsz)()
        ptr = ctypes.c_void_p()
        _native.check(_native.lib.ms_ipc_alloc(reg.nbytes, ctypes.byref(ptr), handle), "ms_ipc_alloc")
        handles = [None] * t
        dist.all_gather_object(handles, bytes(handle), group=group)
        bases = []
        for j, hb in enumerate(handles):
            if j == rank:
                bases.append(ptr.value)
                continue
            pj = ctypes.c_void_p()
            _native.check(_native.lib.ms_ipc_open(hb, ctypes.byref(pj)), "ms_ipc_open")
            bases.append(pj.value)
        local = _DeviceBytes(ptr.value, reg.nbytes, dev).tensor
        return cls(rank, t, max_rows, d, dev, local, bases, owner=(ptr.value, bases), early=True)

    # ----------------------------------------------------------------- kernels
    def signal(self, k: int, stream=None) -> None:
        _native.call("ms_tp_signal", self.peer_flags[k].data_ptr(), self.rank, self.t,
                     self.epoch[k:k + 1].data_ptr(), _dev.stream_ptr(stream))

    def reduce_gather(self, R: int, stream=None) -> None:
        _native.call("ms_tp_reduce_gather", self.peer_p.data_ptr(), self.d, self.peer_x.data_ptr(), self.d,
                     self.flags[0:64].data_ptr(), self.epoch[0:1].data_ptr(), self.rank, self.t, R, self.d,
                     self.err.data_ptr(), self.early, _dev.stream_ptr(stream))

    def rmsnorm_wait(self, R: int, gamma: torch.Tensor, eps: float, out: torch.Tensor, stream=None) -> None:
        _native.call("ms_rmsnorm_wait", self.x.data_ptr(), self.d, _dev.ptr(gamma, BF16), eps, R, self.d,
                     out.data_ptr(), out.stride(0), self.flags[64:128].data_ptr(), self.epoch[1:2].data_ptr(),
                     self.t, self.err.data_ptr(), self.early, _dev.stream_ptr(stream))

    def linear_scatter(self, x: torch.Tensor, w: torch.Tensor, residual: torch.Tensor | None, stream=None) -> None:
        """Row-parallel GEMM with the reduce-scatter fused into its epilogue:
        fp32 partials pushed into the owning ranks' receive slots (the P
        regions, viewed [t][max_rows][d/t])."""
        M, Kd = x.shape
        _native.call("ms_linear_tp_scatter", x.data_ptr(), x.stride(0), w.data_ptr(),
                     None if residual is None else residual.data_ptr(), 0 if residual is None else residual.stride(0),
                     M, self.d, Kd, self.peer_p.data_ptr(), self.rank, self.t, self.max_rows,
                     _dev.stream_ptr(stream))

    def reduce_recv(self, R: int, stream=None) -> None:
        _native.call("ms_tp_reduce_recv_gather", self.p.data_ptr(), self.max_rows, self.d // self.t,
                     self.peer_x.data_ptr(), self.d, self.flags[0:64].data_ptr(), self.epoch[0:1].data_ptr(),
                     self.rank, self.t, R, self.err.data_ptr(), self.early, _dev.stream_ptr(stream))

    def scatter_allreduce_norm(self, R: int, gamma: torch.Tensor, eps: float, out: torch.Tensor, stream=None) -> None:
        """After linear_scatter: x[:R] = sum of the received slots, then out = RMSNorm(x) * gamma."""
        self.signal(0, stream)
        self.reduce_recv(R, stream)
        self.signal(1, stream)
        self.rmsnorm_wait(R, gamma, eps, out, stream)

    def allreduce_norm(self, R: int, gamma: torch.Tensor, eps: float, out: torch.Tensor, stream=None) -> None:
        """x[:R] = sum over ranks of P[:R] (rank order), then out = RMSNorm(x) * gamma."""
        self.signal(0, stream)
        self.reduce_gather(R, stream)
        self.signal(1, stream)
        self.rmsnorm_wait(R, gamma, eps, out, stream)

    def argmax(self, logits: torch.Tensor, v0: int, out: torch.Tensor, stream=None) -> None:
        """Cross-rank first-index argmax of vocab-parallel logits [R, V/t]."""
        R, Vr = logits.shape
        _native.call("ms_tp_argmax_local", logits.data_ptr(), logits.stride(0), R, Vr, v0, self.am.data_ptr(),
                     _dev.stream_ptr(stream))
        self.signal(2, stream)
        _native.call("ms_tp_argmax_combine", self.peer_am.data_ptr(), self.t, R, self.flags[128:192].data_ptr(),
                     self.epoch[2:3].data_ptr(), _dev.ptr(out, torch.int32), self.err.data_ptr(), self.early,
                     _dev.stream_ptr(stream))

    def check(self) -> None:
        if int(self.err.item()) != 0:
            raise RuntimeError("tensor-parallel peer wait timed out (a rank stopped making progress)")


class _DeviceBytes:
    """uint8 torch tensor over cudaMalloc'd memory (freed by the library at exit)."""

    def __init__(self, ptr: int, nbytes: int, device):
        class _CAI:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
        self.tensor = torch.as_tensor(_CAI(), device=device)


# --------------------------------------------------------------------- weights
def shard_llama(w: LlamaWeights, rank: int, t: int) -> LlamaWeights:
    """Rank r's Megatron shard of full Llama weights (the layouts of llama.py)."""
    c = w.cfg
    check_tp(c, t)
    D, H, Hkv, F, V = c.head_dim, c.n_heads, c.n_kv_heads, c.ffn, c.vocab
    hq, hk, f, v = H // t, Hkv // t, F // t, V // t
    out = {"tok_emb": w["tok_emb"], "norm_f": w["norm_f"],
           "lm_head": w["lm_head"][rank * v:(rank + 1) * v].contiguous()}
    for i in range(c.n_layers):
        p = f"l{i}."
        qkv = w[p + "w_qkv"]
        q = qkv[rank * hq * D:(rank + 1) * hq * D]
        k = qkv[H * D + rank * hk * D: H * D + (rank + 1) * hk * D]
        vv = qkv[(H + Hkv) * D + rank * hk * D: (H + Hkv) * D + (rank + 1) * hk * D]
        out[p + "w_qkv"] = torch.cat([q, k, vv]).contiguous()
        out[p + "w_o"] = w[p + "w_o"][:, rank * hq * D:(rank + 1) * hq * D].contiguous()
        # the gate/up interleave is in 64-row blocks and F/t is a multiple of 64:
        # the rank's rows are one contiguous range
        out[p + "w_gu"] = w[p + "w_gu"][rank * 2 * f:(rank + 1) * 2 * f].contiguous()
        out[p + "w_down"] = w[p + "w_down"][:, rank * f:(rank + 1) * f].contiguous()
        out[p + "attn_norm"] = w[p + "attn_norm"]
        out[p + "mlp_norm"] = w[p + "mlp_norm"]
    return LlamaWeights(shard_config(c, t), out)


def check_tp(c: LlamaConfig, t: int) -> None:
    if c.n_heads % t or c.n_kv_heads % t or (c.ffn // t) % 64 or c.ffn % t or c.vocab % t or c.d % (4 * t):
        raise ValueError(f"{c.name} does not split over {t} ranks (heads, KV heads, ffn/64, vocab, d)")


def shard_config(c: LlamaConfig, t: int) -> LlamaConfig:
    import dataclasses
    return dataclasses.replace(c, name=f"{c.name}/tp{t}", n_heads=c.n_heads // t, n_kv_heads=c.n_kv_heads // t,
                               ffn=c.ffn // t, vocab=c.vocab // t, d=c.d, hd=c.head_dim)


def random_shard(c: LlamaConfig, rank: int, t: int, seed: int, device="cuda", std: float = 0.02) -> LlamaWeights:
    """Rank r's shard of a random-init model generated shard-locally (70B never
    exists whole on one GPU); the replicated tensors come from the same seed on
    every rank."""
    check_tp(c, t)
    sc = shard_config(c, t)
    local = LlamaWeights.random(sc, seed * 1000 + 1 + rank, device=device, std=std)
    shared = LlamaWeights.random(dataclasses_replace_layers(c, 0), seed, device=device, std=std)
    local.t["tok_emb"] = shared["tok_emb"]
    local.t["norm_f"] = shared["norm_f"]
    return local


def dataclasses_replace_layers(c: LlamaConfig, n: int) -> LlamaConfig:
    import dataclasses
    return dataclasses.replace(c, n_layers=n)


# ----------------------------------------------------------------------- model
class LlamaTPModel(LlamaModel):
    """Rank r of a tensor-parallel Llama.  The shard's config holds the rank's
    head / ffn / vocab counts; the residual stream x is the group's symmetric
    buffer (peers write their reduced column slices into it)."""

    def __init__(self, shard: LlamaWeights, comm: TPComm, max_rows: int, device="cuda", fused: bool = True):
        if max_rows > comm.max_rows:
            raise ValueError("max_rows exceeds the symmetric buffers")
        super().__init__(shard, max_rows=max_rows, device=device, fuse_norm=False)
        self.comm = comm
        self.tp = comm.t
        self.x = comm.x  # residual stream = symmetric buffer
        self.v0 = comm.rank * shard.cfg.vocab
        # fused (default): GEMM -> reduce-scatter by peer stores from the O /
        # down epilogues; False: GEMM to a local partial + two-shot pull reduction
        self.fused = bool(fused)

    def forward(self, tokens, start, slot, cache, logits, head_rows=None, stream=None, prefill: bool = False):
        """Rank-local vocab slice of the logits ([R', V/t] fp32).  prefill: the
        same tensor-parallel GEMMs (ms_linear; the row-parallel epilogues scatter)."""
        c, w, cm = self.cfg, self.w, self.comm
        B, Q = tokens.shape
        R = B * Q
        if R > self.max_rows:
            raise ValueError(f"{R} rows exceed max_rows={self.max_rows}")
        x, h, qkv, at, ff = self.x[:R], self.h[:R], self.qkv[:R], self.attn[:R], self.ff[:R]
        P = cm.p[:R]
        r0 = cm.rank == 0
        K.embed(tokens, start, Q, w["tok_emb"], None, 0, out=x, stream=stream)
        K.rmsnorm(x, w["l0.attn_norm"], c.eps, out=h, stream=stream)
        for i in range(c.n_layers):
            p = f"l{i}."
            K.linear(h, w[p + "w_qkv"], out=qkv, stream=stream)
            K.attention(qkv, B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], self.scale,
                        out=at, stream=stream, n_kv_heads=c.n_kv_heads, rope=self.rope,
                        page=getattr(cache, "page", None))
            nxt = w[f"l{i + 1}.attn_norm"] if i + 1 < c.n_layers else w["norm_f"]
            if self.fused:
                cm.linear_scatter(at, w[p + "w_o"], x if r0 else None, stream)
                cm.scatter_allreduce_norm(R, w[p + "mlp_norm"], c.eps, h, stream)
                K.linear(h, w[p + "w_gu"], act=2, out=ff, stream=stream)
                cm.linear_scatter(ff, w[p + "w_down"], x if r0 else None, stream)
                cm.scatter_allreduce_norm(R, nxt, c.eps, h, stream)
                continue
            K.linear(at, w[p + "w_o"], residual=x if r0 else None, out=P, out_f32=True, stream=stream)
            cm.allreduce_norm(R, w[p + "mlp_norm"], c.eps, h, stream)
            K.linear(h, w[p + "w_gu"], act=2, out=ff, stream=stream)
            K.linear(ff, w[p + "w_down"], residual=x if r0 else None, out=P, out_f32=True, stream=stream)
            cm.allreduce_norm(R, nxt, c.eps, h, stream)
        if head_rows is None:
            hf = h
        else:
            hf = self.h[R:R + head_rows.numel()] if R + head_rows.numel() <= self.max_rows else None
            if hf is None:
                raise ValueError("head_rows do not fit the activation buffer")
            K.rmsnorm(x, w["norm_f"], c.eps, out=hf, rows=head_rows, stream=stream)
        K.linear(hf, w["lm_head"], out=logits, out_f32=True, stream=stream)
        return logits

    def argmax(self, logits: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
        """Global first-index argmax of the full-vocab logits row (all ranks)."""
        self.comm.argmax(logits, self.v0, out, stream)
        return out
