"""Llama-2-style decoder (pre-RMSNorm, rotary positions, grouped-query
attention, SwiGLU MLP, untied LM head) on the libminions kernels — the model
family BASELINE.json's headline metric names: Llama-2-70B as the verifier and
Llama-160M drafters (cfg3), Llama-2-13B (cfg5).

As for opt.py, the reference has no model: this is the compute behind
ModelOracle.next_dist (aggspec/oracles.py:19-26), called per draft position by
draft_sequence (aggspec/oracles.py:135-153) and for the s+1 verify positions by
_do_verify_batch (aggspec/engine.py:294-296), batched over requests and
positions against a KV cache.

Memory layout (HBM):
  weights    bf16 [out, in]; w_qkv [(H + 2 Hkv) D, d] (q | k | v rows);
             w_gu [2F, d] = gate and up rows interleaved in 64-row blocks
             (rows 128t..128t+63 = gate 64t.., rows 128t+64.. = up 64t..), so
             the SwiGLU product is the epilogue of one GEMM (ms_linear act=2)
  rope       fp32 (cos, sin) table [max_pos, D/2, 2]
  KV cache   per layer K and V [slots, Hkv, T, D] bf16, K stored rotated
  activations x [B*Q, d] bf16 residual stream, updated in place by the
             O-proj / down-proj epilogues (residual add fused)
"""
from __future__ import annotations

import math

import torch

from . import kernels as K
from .weights import KVCache, LlamaConfig, LlamaWeights, gate_up_rows  # noqa: F401
from .weights import LLAMA_CONFIGS as CONFIGS  # noqa: F401

BF16 = torch.bfloat16


class LlamaModel:
    """Batched forward over the kernels with static activation buffers (CUDA
    graph capturable), same interface as opt.OPTModel.

    Prompt prefill (forward(..., prefill=True) from the engine's prompt
    chunks) is compute-bound: its layer GEMMs run on
    ms_linear_wide (tcgen05 CTA pairs, csrc/gemm_pair.cu) whatever the chunk's
    row count (full-K accumulation in k order: a row's result does not depend
    on the chunking, tests/test_paged_gpu.py).  Every decode / verify / drafter GEMM is ms_linear or
    ms_gemv whatever its row count — their per-row results never depend on
    how many rows share a launch (the lossless property); the prefill path is
    chosen by the caller, never by the row count, and the greedy teacher and
    the speculative run prefill with identical calls."""


    def __init__(self, w: LlamaWeights, max_rows: int, device="cuda", small_gemm: bool = False,
                 fuse_norm: bool | None = None, split_kv: str | bool = False):
        """small_gemm: projections of <= 64 token rows with K <= K.GEMV_MAX_K use the
        low-latency ms_gemv (drafters' decode steps); the verifier keeps the
        tcgen05 path everywhere, so its numerics never depend on the row count.

        fuse_norm (default on for the verifier; False disables): RMSNorm folded
        across GEMMs — the gains are folded into w_qkv / w_gu / lm_head
        (LlamaWeights.fold_norms, in place), the O / down GEMMs emit per-row
        sums of squares and the QKV / gate-up / LM-head GEMMs scale by rstd:
        no RMSNorm kernel and no normalised activation between layers (one
        explicit norm before layer 0).  Numerics: out = rstd * (x . (g * W)^T)
        in fp32, one rounding (oracle/llama_ref.forward(fused_norm=True))."""
        self.w, self.cfg = w, w.cfg
        self.small_gemm = small_gemm
        c = self.cfg
        if fuse_norm is None:
            # on by default: interleaved graph A/B of
            # the 70B verify forward (tools/ab_fuse_norm.py, same weights and
            # process) 27.02 vs 27.84 ms at Q = 5, 29.90 vs 30.85 at Q = 7,
            # 33.09 vs 33.62 at Q = 9, 36.89 vs 36.97 at Q = 11.  (An earlier
            # whole-bench A/B read it as a loss, but the adaptive selector's
            # s trajectory differs run to run, so bench lines cannot resolve
            # a ~2% forward change.)
            fuse_norm = not small_gemm
        o_split = K.linear_splits(c.d, c.n_heads * c.head_dim)
        d_split = K.linear_splits(c.d, c.ffn)
        self.fuse_norm = bool(fuse_norm) and o_split > 1 and d_split > 1  # producers need split-K
        if self.fuse_norm or small_gemm:
            # drafters (small_gemm): decode steps fold each RMSNorm into the
            # QKV / gate-up ms_gemv (rstd from x inside the kernel, gain in the
            # weight) — two fewer launches per layer; catch-up / prefill rows
            # keep an explicit norm (unit gains after the fold)
            w.fold_norms()
        self.n_parts = (c.d + 127) // 128
        self.rms_a = torch.zeros((max_rows, self.n_parts), dtype=torch.float32, device=device) if self.fuse_norm else None
        self.rms_b = torch.zeros((max_rows, self.n_parts), dtype=torch.float32, device=device) if self.fuse_norm else None
        self.device = torch.device(device)
        self.max_rows = max_rows
        self.x = torch.empty((max_rows, c.d), dtype=BF16, device=device)
        self.h = torch.empty((max_rows, c.d), dtype=BF16, device=device)
        self.qkv = torch.empty((max_rows, c.qkv_out), dtype=BF16, device=device)
        self.attn = torch.empty((max_rows, c.n_heads * c.head_dim), dtype=BF16, device=device)
        self.ff = torch.empty((max_rows, c.ffn), dtype=BF16, device=device)
        self.scale = 1.0 / math.sqrt(c.head_dim)
        self.rope = K.rope_table(c.max_pos, c.head_dim, c.rope_theta, device=device)
        self.ws = None
        # split over the cache length (chunks fixed by the cache length, <= 8,
        # merged in chunk order) for decode / verify calls (Q <= 16), never for
        # prefill chunks (large per-shape scratch; the prefill path is shared
        # by the greedy teacher and the speculative run, so losslessness
        # holds).  Opt-in: split_kv="auto" (caches >= 1024 positions) or True
        # (every decode / verify call).  Measured no gain on either kernel: MHA
        # (cfg5 on one GPU) verify 31.7 vs 29.4 ms; GQA row kernel (70B heads,
        # tools/attn_ab.py with AB_WS=1) 151 vs 116 us at a 4K cache, Q = 5, and
        # slower at every shorter cache — each extra CTA repeats the query
        # staging, the first DRAM latency and a 50 KB record.
        self.split_kv = split_kv in (True, "auto")
        self.split_kv_min_len = 0 if split_kv is True else 1024
        self._aws: dict = {}

    def _attn_ws(self, B: int, Q: int, T: int):
        """Split-KV scratch per (B, Q, T) call shape (allocated on the first,
        eager call of a shape — never inside a CUDA-graph capture)."""
        if not self.split_kv or T < self.split_kv_min_len or Q > 16:
            return None
        key = (B, Q, T)
        if key not in self._aws:
            c = self.cfg
            self._aws[key] = K.AttnWorkspace(B, Q, c.n_heads, c.head_dim, T, self.device, n_kv_heads=c.n_kv_heads)
        return self._aws[key]

    def forward(self, tokens: torch.Tensor, start: torch.Tensor, slot: torch.Tensor, cache: KVCache,
                logits: torch.Tensor, head_rows: torch.Tensor | None = None, stream=None,
                prefill: bool = False) -> torch.Tensor:
        """Run Q positions for B requests (contract of OPTModel.forward)."""
        c, w = self.cfg, self.w
        B, Q = tokens.shape
        R = B * Q
        if R > self.max_rows:
            raise ValueError(f"{R} rows exceed max_rows={self.max_rows}")
        if cache.max_len > c.max_pos:
            raise ValueError("KV cache longer than the RoPE table")
        x, h, qkv, at, ff = self.x[:R], self.h[:R], self.qkv[:R], self.attn[:R], self.ff[:R]
        K.embed(tokens, start, Q, w["tok_emb"], None, 0, out=x, stream=stream)
        small = self.small_gemm and R <= 64
        if self.fuse_norm and not prefill:
            return self._forward_fused(tokens, start, slot, cache, logits, head_rows, stream)

        def lin(xx, wname, **kw):
            if prefill:
                return _prefill_linear(xx, w[wname], stream=stream, **kw)
            if small and xx.shape[1] <= K.GEMV_MAX_K:
                return K.gemv(xx, w[wname], stream=stream, **kw)
            return K.linear(xx, w[wname], stream=stream, **kw)

        # decode steps of a drafter: RMSNorm folded into the QKV / gate-up gemv
        fold = small and not prefill and c.d <= K.GEMV_MAX_K
        for i in range(c.n_layers):
            p = f"l{i}."
            if fold:
                K.gemv(x, w[p + "w_qkv"], out=qkv, stream=stream, rms_eps=c.eps)
            else:
                K.rmsnorm(x, w[p + "attn_norm"], c.eps, out=h, stream=stream)
                lin(h, p + "w_qkv", out=qkv)
            K.attention(qkv, B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], self.scale,
                        out=at, stream=stream, n_kv_heads=c.n_kv_heads, rope=self.rope,
                        page=getattr(cache, "page", None), ws=self._attn_ws(B, Q, cache.max_len), prefill=prefill)
            lin(at, p + "w_o", residual=x, out=x)
            if fold:
                K.gemv(x, w[p + "w_gu"], act=2, out=ff, stream=stream, rms_eps=c.eps)
            else:
                K.rmsnorm(x, w[p + "mlp_norm"], c.eps, out=h, stream=stream)
                lin(h, p + "w_gu", act=2, out=ff)
            lin(ff, p + "w_down", residual=x, out=x)
        Rh = R if head_rows is None else head_rows.numel()
        hf = self.h[:Rh]
        K.rmsnorm(x, w["norm_f"], c.eps, out=hf, rows=head_rows, stream=stream)
        K.linear(hf, w["lm_head"], out=logits, out_f32=True, stream=stream)
        return logits

    def _forward_fused(self, tokens, start, slot, cache, logits, head_rows, stream):
        """Layers with the RMSNorms folded across GEMMs (see __init__); x is
        already embedded."""
        c, w = self.cfg, self.w
        B, Q = tokens.shape
        R = B * Q
        x, h, qkv, at, ff = self.x[:R], self.h[:R], self.qkv[:R], self.attn[:R], self.ff[:R]
        ra, rb = self.rms_a, self.rms_b
        for i in range(c.n_layers):
            p = f"l{i}."
            if i == 0:  # the embedding has no producer GEMM: one explicit norm (gain folded: ones)
                K.rmsnorm(x, w[p + "attn_norm"], c.eps, out=h, stream=stream)
                K.linear(h, w[p + "w_qkv"], out=qkv, stream=stream)
            else:
                K.linear_rms(x, w[p + "w_qkv"], out=qkv, rms_in=rb, eps=c.eps, stream=stream)
            K.attention(qkv, B, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], self.scale,
                        out=at, stream=stream, n_kv_heads=c.n_kv_heads, rope=self.rope,
                        page=getattr(cache, "page", None), ws=self._attn_ws(B, Q, cache.max_len))
            K.linear_rms(at, w[p + "w_o"], residual=x, out=x, rms_out=ra, stream=stream)
            K.linear_rms(x, w[p + "w_gu"], act=2, out=ff, rms_in=ra, eps=c.eps, stream=stream)
            K.linear_rms(ff, w[p + "w_down"], residual=x, out=x, rms_out=rb, stream=stream)
        if head_rows is None:
            K.linear_rms(x, w["lm_head"], out=logits, out_f32=True, rms_in=rb, eps=c.eps, stream=stream)
        elif head_rows.numel() > 0:
            hf = self.h[: head_rows.numel()]
            K.rmsnorm(x, w["norm_f"], c.eps, out=hf, rows=head_rows, stream=stream)
            K.linear(hf, w["lm_head"], out=logits, out_f32=True, stream=stream)
        return logits


def _prefill_linear(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, residual=None, act: int = 0,
                    stream=None) -> torch.Tensor:
    """Prefill GEMM on tcgen05 CTA pairs (ms_linear_wide): out = x @ w^T
    (+ residual, in place when out is residual) or, act=2, the gated SiLU of
    the 64-row interleaved gate/up weight (fused epilogue)."""
    return K.linear_wide(x, w, residual=residual, act=act, out=out, stream=stream)


class GroupedLlamaModel:
    """The K drafters of a round (one Llama architecture, K weight sets) as ONE
    forward: drafter k is row group k — its weights stacked at index k, its KV
    cache slots k*S + s of one cache with K*S slots — so every op of a decode
    step is a single launch for all drafters (ms_*_grouped) instead of K
    launches on K streams.  Replaces the per-drafter draft_sequence loop of
    _do_draft_batch (aggspec/engine.py:262-276).

    forward(tokens [K*B, Q], start [K*B], slot [K*B], cache, logits [K*Bh, V],
    head_rows [K*Bh] | None): rows of group k are k*B*Q .. (k+1)*B*Q - 1; the
    head rows must be group-major (Bh per group)."""

    def __init__(self, ws: list[LlamaWeights], max_rows: int, device="cuda"):
        c = ws[0].cfg
        if any(w.cfg != c for w in ws):
            raise ValueError("grouped drafters must share one architecture")
        self.cfg, self.G = c, len(ws)
        self.device = torch.device(device)
        self.t = {k: torch.stack([w[k] for w in ws]).contiguous() for k in ws[0].t}
        # RMSNorm gains folded into the stacked projections (the callers'
        # weights are untouched): bf16(w * g), the same rounding as
        # LlamaWeights.fold_norms, so a grouped forward stays bitwise equal to
        # K separate small_gemm LlamaModels
        t = self.t
        pairs = [(f"l{i}.attn_norm", f"l{i}.w_qkv") for i in range(c.n_layers)]
        pairs += [(f"l{i}.mlp_norm", f"l{i}.w_gu") for i in range(c.n_layers)] + [("norm_f", "lm_head")]
        for gname, wname in pairs:
            if not bool(torch.all(t[gname] == 1)):
                t[wname].mul_(t[gname].to(t[wname].dtype)[:, None, :])
            t[gname] = torch.ones_like(t[gname])
        G = self.G
        # set by the engine while it launches this model's steps in the
        # co-resident mode (ms_set_coresident): the LM head then runs on ms_gemv
        self.coresident = False
        self.max_rows = max_rows  # per group
        R = G * max_rows
        self.x = torch.empty((R, c.d), dtype=BF16, device=device)
        self.h = torch.empty((R, c.d), dtype=BF16, device=device)
        self.qkv = torch.empty((R, c.qkv_out), dtype=BF16, device=device)
        self.attn = torch.empty((R, c.n_heads * c.head_dim), dtype=BF16, device=device)
        self.ff = torch.empty((R, c.ffn), dtype=BF16, device=device)
        self.scale = 1.0 / math.sqrt(c.head_dim)
        self.rope = K.rope_table(c.max_pos, c.head_dim, c.rope_theta, device=device)

    def forward(self, tokens, start, slot, cache, logits, head_rows=None, stream=None, prefill: bool = False):
        c, t, G = self.cfg, self.t, self.G
        GB, Q = tokens.shape
        B = GB // G
        M = B * Q  # rows per group
        R = G * M
        if M > self.max_rows:
            raise ValueError(f"{M} rows per group exceed max_rows={self.max_rows}")
        x, h, qkv, at, ff = self.x[:R], self.h[:R], self.qkv[:R], self.attn[:R], self.ff[:R]
        K.embed_grouped(tokens, start, Q, t["tok_emb"], M, out=x, stream=stream)

        def lin(xx, name, **kw):
            wt = t[name]  # [G, N, K]
            if prefill:  # prompt prefill: per-group ms_linear_wide
                out, res = kw["out"], kw.get("residual")
                for g in range(G):
                    sl = slice(g * M, (g + 1) * M)
                    _prefill_linear(xx[sl], wt[g], out=out[sl], residual=None if res is None else res[sl],
                                    act=kw.get("act", 0), stream=stream)
                return out
            if M <= 64 and wt.shape[2] <= K.GEMV_MAX_K:
                return K.gemv_grouped(xx, wt, G, stream=stream, **kw)
            return K.linear_grouped(xx, wt.view(-1, wt.shape[2]), G, stream=stream, **kw)

        # decode steps (<= 64 rows per drafter): RMSNorm folded into the QKV /
        # gate-up gemv; catch-up and prefill rows: explicit norm (unit gains)
        fold = not prefill and M <= 64 and c.d <= K.GEMV_MAX_K
        for i in range(c.n_layers):
            p = f"l{i}."
            if fold:
                K.gemv_grouped(x, t[p + "w_qkv"], G, out=qkv, stream=stream, rms_eps=c.eps)
            else:
                K.rmsnorm_grouped(x, t[p + "attn_norm"], M, c.eps, out=h, stream=stream)
                lin(h, p + "w_qkv", out=qkv)
            K.attention(qkv, GB, Q, c.n_heads, c.head_dim, slot, start, cache.k[i], cache.v[i], self.scale,
                        out=at, stream=stream, n_kv_heads=c.n_kv_heads, rope=self.rope,
                        page=getattr(cache, "page", None), prefill=prefill)
            lin(at, p + "w_o", residual=x, out=x)
            if fold:
                K.gemv_grouped(x, t[p + "w_gu"], G, act=2, out=ff, stream=stream, rms_eps=c.eps)
            else:
                K.rmsnorm_grouped(x, t[p + "mlp_norm"], M, c.eps, out=h, stream=stream)
                lin(h, p + "w_gu", act=2, out=ff)
            lin(ff, p + "w_down", residual=x, out=x)
        Rh = R if head_rows is None else head_rows.numel()
        if Rh == 0:
            return logits
        if fold and head_rows is None and self.coresident:
            # co-resident decode step: the LM head as a folded-norm gemv too
            # (the tcgen05 GEMM's shared-memory rings cannot sit beside the
            # verifier's GEMM CTAs)
            K.gemv_grouped(x, t["lm_head"], G, out=logits, out_f32=True, stream=stream, rms_eps=c.eps)
            return logits
        hf = self.h[:Rh]
        K.rmsnorm_grouped(x, t["norm_f"], Rh // G, c.eps, out=hf, rows=head_rows, stream=stream)
        head = t["lm_head"]
        K.linear_grouped(hf, head.view(-1, head.shape[2]), G, out=logits, out_f32=True, stream=stream)
        return logits
