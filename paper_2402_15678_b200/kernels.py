"""Python wrappers of the model-forward kernels (csrc/gemm.cu, csrc/model.cu).

Each wrapper checks shapes/dtypes, then calls the C-ABI with raw pointers on
the current (or given) CUDA stream.  Nothing here allocates on the hot path
when `out=` buffers are passed, so launches can be captured in CUDA graphs.
"""
from __future__ import annotations

import ctypes

import torch

from . import _dev
from . import _native

BF16 = torch.bfloat16


def linear_splits(N: int, K: int) -> int:
    return int(_native.lib.ms_linear_splits(N, K))


# drafter decode projections (<= 64 token rows) up to this reduction length run
# on ms_gemv (4 K-splitting warps up to K = 1024, 8 beyond); the verifier never
# uses it
GEMV_MAX_K = 4096


def linear(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None,
           residual: torch.Tensor | None = None, act: int = 0, out: torch.Tensor | None = None,
           out_f32: bool = False, splits: int = 0, stream=None) -> torch.Tensor:
    """out = act(x @ w.T + bias) + residual on tcgen05 (ms_linear, cluster
    split-K).  act=2: gated SiLU over a 64-row interleaved gate/up weight, out
    [M, N/2]."""
    if x.dim() != 2 or w.dim() != 2 or x.dtype != BF16 or w.dtype != BF16:
        raise ValueError("x [M, K] and w [N, K] must be 2-D bf16")
    M, K = x.shape
    N = w.shape[0]
    if w.shape[1] != K or x.stride(1) != 1 or not w.is_contiguous():
        raise ValueError("shape/stride mismatch")
    No = N // 2 if act == 2 else N
    if out is None:
        out = torch.empty((M, No), dtype=torch.float32 if out_f32 else BF16, device=x.device)
    if out.stride(1) != 1 or out.shape != (M, No):
        raise ValueError(f"out must be [M, {No}] with unit column stride")
    if residual is not None and (residual.shape != (M, N) or residual.stride(1) != 1):
        raise ValueError("residual must be [M, N]")
    _native.call("ms_linear", x.data_ptr(), x.stride(0), w.data_ptr(),
                 None if bias is None else _dev.ptr(bias, BF16, "bias"),
                 None if residual is None else residual.data_ptr(),
                 0 if residual is None else residual.stride(0),
                 out.data_ptr(), out.stride(0), int(out.dtype == torch.float32), M, N, K, act,
                 splits, _dev.stream_ptr(stream))
    return out


def linear_wide(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None,
                residual: torch.Tensor | None = None, act: int = 0, out: torch.Tensor | None = None,
                out_f32: bool = False, stream=None) -> torch.Tensor:
    """Prefill GEMM on tcgen05 CTA pairs (ms_linear_wide): same contract as
    linear(); full-K accumulation (not M-invariant like linear's split-K)."""
    if x.dim() != 2 or w.dim() != 2 or x.dtype != BF16 or w.dtype != BF16:
        raise ValueError("x [M, K] and w [N, K] must be 2-D bf16")
    M, K = x.shape
    N = w.shape[0]
    if w.shape[1] != K or x.stride(1) != 1 or not w.is_contiguous():
        raise ValueError("shape/stride mismatch")
    No = N // 2 if act == 2 else N
    if out is None:
        out = torch.empty((M, No), dtype=torch.float32 if out_f32 else BF16, device=x.device)
    if out.stride(1) != 1 or out.shape != (M, No):
        raise ValueError(f"out must be [M, {No}] with unit column stride")
    if residual is not None and (residual.shape != (M, N) or residual.stride(1) != 1):
        raise ValueError("residual must be [M, N]")
    _native.call("ms_linear_wide", x.data_ptr(), x.stride(0), w.data_ptr(),
                 None if bias is None else _dev.ptr(bias, BF16, "bias"),
                 None if residual is None else residual.data_ptr(),
                 0 if residual is None else residual.stride(0),
                 out.data_ptr(), out.stride(0), int(out.dtype == torch.float32), M, N, K, act,
                 _dev.stream_ptr(stream))
    return out


def gated_silu(gu: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """out [M, N/2] bf16 = silu(gate) * up of an fp32 gate/up GEMM output gu
    [M, N] over the 64-row interleaved weight (ms_gated_silu: the act=2
    epilogue of ms_linear, for prefill GEMMs run on cuBLAS)."""
    M, N = gu.shape
    if gu.dtype != torch.float32 or gu.stride(1) != 1 or out.dtype != BF16 or out.shape != (M, N // 2) \
            or out.stride(1) != 1:
        raise ValueError("gu [M, N] fp32 and out [M, N/2] bf16 with unit column stride")
    _native.call("ms_gated_silu", gu.data_ptr(), gu.stride(0), M, N, out.data_ptr(), out.stride(0),
                 _dev.stream_ptr(stream))
    return out


def linear_rms(x: torch.Tensor, w: torch.Tensor, *, residual: torch.Tensor | None = None, act: int = 0,
               out: torch.Tensor, out_f32: bool = False, rms_in: torch.Tensor | None = None, eps: float = 1e-5,
               rms_out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """ms_linear with the RMSNorm folded across GEMMs: rms_in [rows, n_parts]
    fp32 partial sums of squares (from the producer) -> scale by rstd; rms_out
    [rows, N / 128] fp32 -> this (residual-writing, split-K) GEMM emits them."""
    M, K = x.shape
    N = w.shape[0]
    if x.dtype != BF16 or w.dtype != BF16 or w.shape[1] != K or not w.is_contiguous():
        raise ValueError("x [M, K] and w [N, K] must be bf16")
    ref = rms_in if rms_in is not None else rms_out
    if ref is None or ref.dtype != torch.float32 or not ref.is_contiguous():
        raise ValueError("rms partial buffers must be contiguous fp32 [parts, ld]")
    _native.call("ms_linear_rms", x.data_ptr(), x.stride(0), w.data_ptr(), None,
                 None if residual is None else residual.data_ptr(), 0 if residual is None else residual.stride(0),
                 out.data_ptr(), out.stride(0), int(out.dtype == torch.float32), M, N, K, act, 0,
                 None if rms_in is None else rms_in.data_ptr(), 0 if rms_in is None else rms_in.shape[1], eps,
                 None if rms_out is None else rms_out.data_ptr(), ref.stride(0), _dev.stream_ptr(stream))
    return out


def gemv(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None,
         residual: torch.Tensor | None = None, act: int = 0, out: torch.Tensor | None = None,
         out_f32: bool = False, stream=None, rms_eps: float | None = None) -> torch.Tensor:
    """out = act(x @ w.T + bias) + residual for M <= 64 rows (ms_gemv, low latency).
    rms_eps: x's RMSNorm folded in (gain pre-folded into w; no bias)."""
    M, K = x.shape
    N = w.shape[0]
    if x.dtype != BF16 or w.dtype != BF16 or w.shape[1] != K or x.stride(1) != 1 or not w.is_contiguous():
        raise ValueError("x [M, K] and w [N, K] must be bf16 with unit column stride")
    if rms_eps is not None:
        if bias is not None:
            raise ValueError("the folded-RMSNorm gemv takes no bias")
        return gemv_grouped(x, w.view(1, N, K), 1, residual=residual, act=act, out=out, out_f32=out_f32,
                            stream=stream, rms_eps=rms_eps)
    if out is None:
        out = torch.empty((M, N // 2 if act == 2 else N), dtype=torch.float32 if out_f32 else BF16,
                          device=x.device)
    _native.call("ms_gemv", x.data_ptr(), x.stride(0), w.data_ptr(),
                 None if bias is None else _dev.ptr(bias, BF16, "bias"),
                 None if residual is None else residual.data_ptr(),
                 0 if residual is None else residual.stride(0), out.data_ptr(), out.stride(0),
                 int(out.dtype == torch.float32), M, N, K, act, _dev.stream_ptr(stream))
    return out


def embed(tok: torch.Tensor, start: torch.Tensor, Q: int, tok_emb: torch.Tensor,
          pos_emb: torch.Tensor | None, pos_offset: int = 2, out: torch.Tensor | None = None,
          stream=None) -> torch.Tensor:
    """Rows r = b*Q + i (tok [B, Q] flattened) at positions start[b] + i."""
    R = tok.numel()
    d = tok_emb.shape[1]
    out = out if out is not None else torch.empty((R, d), dtype=BF16, device=tok.device)
    _native.call("ms_embed", _dev.ptr(tok, torch.int32, "tok"), _dev.ptr(start, torch.int32, "start"), Q,
                 _dev.ptr(tok_emb, BF16), _dev.ptr(pos_emb, BF16), pos_offset, R, d,
                 _dev.ptr(out, BF16), _dev.stream_ptr(stream))
    return out


def layernorm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-5,
              out: torch.Tensor | None = None, rows: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
    """LayerNorm of x's rows (or of x[rows] when a row-index tensor is given)."""
    d = x.shape[1]
    R = x.shape[0] if rows is None else rows.numel()
    out = out if out is not None else torch.empty((R, d), dtype=BF16, device=x.device)
    _native.call("ms_layernorm", x.data_ptr(), x.stride(0), _dev.ptr(rows, torch.int32, "rows"),
                 _dev.ptr(gamma, BF16),
                 _dev.ptr(beta, BF16), eps, R, d, out.data_ptr(), out.stride(0),
                 _dev.stream_ptr(stream))
    return out


def rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float = 1e-5, out: torch.Tensor | None = None,
            rows: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """RMSNorm of x's rows (or of x[rows]) — Llama's pre-norm."""
    d = x.shape[1]
    R = x.shape[0] if rows is None else rows.numel()
    out = out if out is not None else torch.empty((R, d), dtype=BF16, device=x.device)
    _native.call("ms_rmsnorm", x.data_ptr(), x.stride(0), _dev.ptr(rows, torch.int32, "rows"),
                 _dev.ptr(gamma, BF16), eps, R, d, out.data_ptr(), out.stride(0), _dev.stream_ptr(stream))
    return out


def rope_table(max_pos: int, head_dim: int, theta: float = 10000.0, device="cuda") -> torch.Tensor:
    """(cos, sin) of p * theta^(-2i/D), i < D/2, as fp32 [max_pos, D/2, 2]
    (computed in fp64 on the host, rounded once)."""
    import numpy as np
    inv = theta ** (-np.arange(0, head_dim, 2, dtype=np.float64) / head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    t = np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)
    return torch.from_numpy(t).to(device)


def kv_append(qkv: torch.Tensor, B: int, Q: int, H: int, D: int, slot: torch.Tensor,
              start: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, stream=None) -> None:
    T = k_cache.shape[2]
    _native.call("ms_kv_append", qkv.data_ptr(), qkv.stride(0), B, Q, H, D,
                 _dev.ptr(slot, torch.int32), _dev.ptr(start, torch.int32), T,
                 _dev.ptr(k_cache, BF16), _dev.ptr(v_cache, BF16), _dev.stream_ptr(stream))


class AttnWorkspace:
    """Split-KV scratch of ms_attention (chunk partials + per-(request, head)
    counters), sized for a model's (B, Q, H, D, T) envelope."""

    def __init__(self, B: int, Q: int, H: int, D: int, T: int, device, n_kv_heads: int | None = None):
        b = ctypes.c_int64()
        c = ctypes.c_int()
        Hkv = H if n_kv_heads is None else n_kv_heads
        _native.check(_native.lib.ms_attention_workspace_gqa(B, Q, H, Hkv, D, T, ctypes.byref(b), ctypes.byref(c)),
                      "ms_attention_workspace_gqa")
        self.ws = torch.empty((b.value + 3) // 4, dtype=torch.float32, device=device)
        self.counters = torch.zeros(c.value, dtype=torch.int32, device=device)


# grouped-query decode / verify attention (head dim 128, <= 16 positions) on
# the tcgen05 kernels (csrc/attention_tc.cu) instead of the warp-MMA row
# kernel: one pass for caches of <= TC_SHORT_KEYS positions (contiguous or
# paged with 16..128-row blocks), online softmax over 128-key chunks for
# longer contiguous caches — faster than the row kernel at every measured
# length (ctx 190 Q = 7: 9.1 vs 12.7 us per 70B layer; 4K Q = 5: 90 vs 117).
# "auto" (default): tcgen05 for grouped-query heads wherever the shape allows;
# True: also multi-head (G = 1) shapes — correct (tests), but slower there
# than the row kernel at every measured length (Llama-2-13B heads, B = 16:
# 44.6 vs 26.9 us at ctx 190, 437 vs 271 at 4K; profiles/
# r2_attn_tc_mha_ab.jsonl: one query row per head leaves the 128-row MMA
# tile nearly empty while the row kernel's 640 CTAs stream 4.9 TB/s);
# False: the row kernel.  Chosen by shape and cache length, never by Q alone.
TC_ATTENTION: bool | str = "auto"
# prompt-prefill calls (more than 16 positions or 128 flattened rows, head
# dim 128 or 64, contiguous or paged caches, GQA and multi-head alike):
# append, then the online kernel in 128-row query tiles
TC_PREFILL = True
# head dims routed to the tiles by default.  The kernel also takes 64 (tested
# against the fp32 restatement), but the small head-dim-64 models (drafters,
# OPT-125M, the tiny cfg1 models) keep the row kernel, whose P.V carries P as
# bf16 hi + lo: on the tiny cfg1 target the bf16-P tiles cut the free-running
# agreement with the fp32 reference from >= 24 to 9 of 48 tokens
# (tests/test_engine_gpu.py), while the drafters' 4K prefill would gain
# 21.6 -> 5.5 ms per layer (profiles/r2_prefill_attn_ab.jsonl)
PREFILL_TILE_DIMS = (128,)
# ... except long caches (chosen by the cache length, never by Q or the
# chunking): the drafters' 4K-prompt prefill (cfg5) takes the D = 64 tiles
PREFILL_TILE_D64_MIN_T = 1024
TC_SHORT_KEYS = 384


def attention(qkv: torch.Tensor, B: int, Q: int, H: int, D: int, slot: torch.Tensor,
              start: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, scale: float,
              out: torch.Tensor | None = None, append: bool = True, ws: AttnWorkspace | None = None,
              stream=None, n_kv_heads: int | None = None, rope: torch.Tensor | None = None,
              page=None, prefill: bool | None = None) -> torch.Tensor:
    """Causal KV-cache attention of Q rows per request (K/V append fused when
    append; split-KV over fixed 128-key chunks when a workspace is given).
    n_kv_heads < H: grouped-query attention (qkv = [q H*D | k Hkv*D | v Hkv*D],
    caches [slots, Hkv, T, D]); rope: the fp32 (cos, sin) table of rope_table."""
    # page: (block_table [slots, max_blocks] int32, block_size) of a paged cache
    # (k_cache / v_cache are then block pools [n_blocks, Hkv, bs, D])
    T = k_cache.shape[2] if page is None else page[0].shape[1] * page[1]
    Hkv = H if n_kv_heads is None else n_kv_heads
    if k_cache.shape[1] != Hkv:
        raise ValueError("cache heads != n_kv_heads")
    if rope is not None and (rope.dtype != torch.float32 or rope.shape[0] < T or rope.shape[1] * 2 != D):
        raise ValueError("rope table must be fp32 [>= T, D/2, 2]")
    out = out if out is not None else torch.empty((B * Q, H * D), dtype=BF16, device=qkv.device)
    use_tc = TC_ATTENTION in (True, "auto")
    # prefill: the model's prompt-prefill calls (every chunk size takes the
    # tiles, so a prompt's rows do not depend on the chunking); None: by shape
    tiles = prefill if prefill is not None else (Q > 16 or Q * (H // Hkv) > 128)
    tile_d = D in PREFILL_TILE_DIMS or (D == 64 and T >= PREFILL_TILE_D64_MIN_T)
    if (use_tc and TC_PREFILL and tiles and tile_d and ws is None
            and (page is None or (page[1] % 16 == 0 and 128 % page[1] == 0))
            and k_cache.is_contiguous() and v_cache.is_contiguous()):
        # prompt prefill: the call's K / V rows appended first, then query
        # tiles of the online tcgen05 kernel (128 rows each) read them back
        # (contiguous or paged alike, so the two stay bitwise equal)
        tab = None if page is None else _dev.ptr(page[0], torch.int32, "block_table")
        if append:
            _native.call("ms_kv_append_paged", qkv.data_ptr(), qkv.stride(0), B, Q, H, Hkv, D,
                         _dev.ptr(slot, torch.int32), _dev.ptr(start, torch.int32), T, _dev.ptr(k_cache, BF16),
                         _dev.ptr(v_cache, BF16), None if rope is None else rope.data_ptr(), tab,
                         0 if page is None else page[0].shape[1], 0 if page is None else page[1],
                         _dev.stream_ptr(stream))
        _native.call("ms_attention_tc", qkv.data_ptr(), qkv.stride(0), B, Q, H, Hkv, D,
                     _dev.ptr(slot, torch.int32), _dev.ptr(start, torch.int32), T, k_cache.shape[0],
                     _dev.ptr(k_cache, BF16), _dev.ptr(v_cache, BF16), None if rope is None else rope.data_ptr(),
                     scale, 0, out.data_ptr(), out.stride(0), tab, 0 if page is None else page[0].shape[1],
                     0 if page is None else page[1], _dev.stream_ptr(stream))
        return out
    if page is not None:  # paged pools: the one-pass kernel, 16..128-row blocks
        use_tc = use_tc and T <= TC_SHORT_KEYS and page[1] % 16 == 0 and 128 % page[1] == 0
    if (use_tc and (Hkv < H or TC_ATTENTION is True) and D == 128 and ws is None and Q <= 16
            and Q * (H // Hkv) <= 128 and k_cache.is_contiguous() and v_cache.is_contiguous()):
        _native.call("ms_attention_tc", qkv.data_ptr(), qkv.stride(0), B, Q, H, Hkv, D,
                     _dev.ptr(slot, torch.int32), _dev.ptr(start, torch.int32), T, k_cache.shape[0],
                     _dev.ptr(k_cache, BF16), _dev.ptr(v_cache, BF16), None if rope is None else rope.data_ptr(),
                     scale, int(append), out.data_ptr(), out.stride(0),
                     None if page is None else _dev.ptr(page[0], torch.int32, "block_table"),
                     0 if page is None else page[0].shape[1], 0 if page is None else page[1],
                     _dev.stream_ptr(stream))
        return out
    _native.call("ms_attention_paged", qkv.data_ptr(), qkv.stride(0), B, Q, H, Hkv, D,
                 _dev.ptr(slot, torch.int32), _dev.ptr(start, torch.int32), T,
                 _dev.ptr(k_cache, BF16), _dev.ptr(v_cache, BF16),
                 None if rope is None else rope.data_ptr(), scale, int(append),
                 out.data_ptr(), out.stride(0),
                 None if ws is None else ws.ws.data_ptr(), 0 if ws is None else ws.ws.numel() * 4,
                 None if ws is None else ws.counters.data_ptr(), 0 if ws is None else ws.counters.numel(),
                 None if page is None else _dev.ptr(page[0], torch.int32, "block_table"),
                 0 if page is None else page[0].shape[1], 0 if page is None else page[1],
                 _dev.stream_ptr(stream))
    return out


# ------------------------------------------------------------ grouped drafters
def linear_grouped(x: torch.Tensor, w: torch.Tensor, G: int, residual: torch.Tensor | None = None, act: int = 0,
                   out: torch.Tensor | None = None, out_f32: bool = False, stream=None) -> torch.Tensor:
    """G row groups in one launch: x [G*M, K], w [G*N, K] (stacked), out [G*M, N']."""
    GM, K = x.shape
    N = w.shape[0] // G
    M = GM // G
    if GM % G or w.shape[0] % G or w.shape[1] != K or x.dtype != BF16 or w.dtype != BF16 or not w.is_contiguous():
        raise ValueError("x [G*M, K], w [G*N, K] bf16")
    No = N // 2 if act == 2 else N
    if out is None:
        out = torch.empty((GM, No), dtype=torch.float32 if out_f32 else BF16, device=x.device)
    _native.call("ms_linear_grouped", x.data_ptr(), x.stride(0), w.data_ptr(), None,
                 None if residual is None else residual.data_ptr(), 0 if residual is None else residual.stride(0),
                 out.data_ptr(), out.stride(0), int(out.dtype == torch.float32), M, N, K, act, 0, G,
                 _dev.stream_ptr(stream))
    return out


def gemv_grouped(x: torch.Tensor, w: torch.Tensor, G: int, residual: torch.Tensor | None = None, act: int = 0,
                 out: torch.Tensor | None = None, out_f32: bool = False, stream=None,
                 rms_eps: float | None = None) -> torch.Tensor:
    """ms_gemv over G row groups: x [G*M, K] (M <= 64), w [G, N, K] stacked.
    rms_eps: each x row's RMSNorm folded in (ms_gemv_rms_grouped; the gain
    must already be folded into w)."""
    GM, K = x.shape
    M = GM // G
    N = w.shape[-2]
    if out is None:
        out = torch.empty((GM, N // 2 if act == 2 else N), dtype=torch.float32 if out_f32 else BF16,
                          device=x.device)
    res = (None if residual is None else residual.data_ptr(), 0 if residual is None else residual.stride(0))
    if rms_eps is not None:
        _native.call("ms_gemv_rms_grouped", x.data_ptr(), x.stride(0), w.data_ptr(), N * K, *res,
                     out.data_ptr(), out.stride(0), int(out.dtype == torch.float32), M, N, K, act, G,
                     float(rms_eps), _dev.stream_ptr(stream))
        return out
    _native.call("ms_gemv_grouped", x.data_ptr(), x.stride(0), w.data_ptr(), N * K, None, *res,
                 out.data_ptr(), out.stride(0), int(out.dtype == torch.float32), M, N, K, act, G,
                 _dev.stream_ptr(stream))
    return out


def embed_grouped(tok: torch.Tensor, start: torch.Tensor, Q: int, tok_emb: torch.Tensor, rpg: int,
                  out: torch.Tensor, stream=None) -> torch.Tensor:
    """tok_emb [G, V, d] stacked; row r uses table r // rpg."""
    R = tok.numel()
    G, V, d = tok_emb.shape
    _native.call("ms_embed_grouped", _dev.ptr(tok, torch.int32, "tok"), _dev.ptr(start, torch.int32, "start"), Q,
                 _dev.ptr(tok_emb, BF16), V * d, rpg, None, 0, R, d, _dev.ptr(out, BF16), _dev.stream_ptr(stream))
    return out


def rmsnorm_grouped(x: torch.Tensor, gamma: torch.Tensor, rpg: int, eps: float, out: torch.Tensor,
                    rows: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """gamma [G, d] stacked; output row r uses gain r // rpg."""
    d = x.shape[1]
    R = x.shape[0] if rows is None else rows.numel()
    _native.call("ms_rmsnorm_grouped", x.data_ptr(), x.stride(0), _dev.ptr(rows, torch.int32, "rows"),
                 _dev.ptr(gamma, BF16), d, rpg, eps, R, d, out.data_ptr(), out.stride(0), _dev.stream_ptr(stream))
    return out
