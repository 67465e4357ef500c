"""The tcgen05 grouped-query attention (csrc/attention_tc.cu, ms_attention_tc)
against the fp32 restatement (oracle/llama_ref rope + softmax), the K/V append
it fuses, multi-chunk contexts (online softmax across 128-key chunks), and
batch invariance (a request's rows do not depend on Q or on the other
requests)."""
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
BF = torch.bfloat16
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import llama_ref  # noqa: E402
from test_llama_gpu import _ref_attention  # noqa: E402


def _run(qkv, B, Q, H, Hkv, D, start, kc, vc, table):
    from paper_2402_15678_b200 import kernels as Kn
    old, old_dims = Kn.TC_ATTENTION, Kn.PREFILL_TILE_DIMS
    Kn.TC_ATTENTION, Kn.PREFILL_TILE_DIMS = True, (64, 128)
    try:
        return Kn.attention(qkv.cuda(), B, Q, H, D, torch.arange(B, dtype=torch.int32).cuda(), start.cuda(), kc, vc,
                            D ** -0.5, n_kv_heads=Hkv, rope=None if table is None else table.cuda())
    finally:
        Kn.TC_ATTENTION, Kn.PREFILL_TILE_DIMS = old, old_dims


@pytest.mark.parametrize("H,Hkv,Q,T,rope", [(64, 8, 5, 320, True), (64, 8, 16, 320, True), (64, 8, 1, 320, True),
                                            (64, 8, 7, 272, True), (64, 8, 3, 384, True), (64, 8, 5, 100, True),
                                            (16, 2, 7, 640, False), (64, 8, 7, 4300, True),
                                            (40, 40, 5, 320, True), (40, 40, 7, 4300, True), (40, 40, 1, 600, True)])
def test_tc_attention_vs_reference(H, Hkv, Q, T, rope):
    D = 128
    B = 3
    g = torch.Generator().manual_seed(H + Q + T)
    kc = torch.randn(B, Hkv, T, D, generator=g).to(BF)
    vc = torch.randn(B, Hkv, T, D, generator=g).to(BF)
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, generator=g).to(BF)
    starts = [0, min(127, T // 2), T - Q - 1] if T < 1000 else [0, 1500, T - Q - 1]
    start = torch.tensor(starts, dtype=torch.int32)
    table = llama_ref.rope_table(T + 4, D, 10000.0) if rope else None
    kcd, vcd = kc.cuda(), vc.cuda()
    got = _run(qkv, B, Q, H, Hkv, D, start, kcd, vcd, table).cpu().float()
    want = _ref_attention(qkv, kc, vc, start, B, Q, H, Hkv, D, table)
    torch.testing.assert_close(got, want, rtol=2e-2, atol=2e-2)
    for b in range(B):  # the appended (rotated) K and V rows
        p0 = int(start[b])
        kn = qkv.float().view(B, Q, -1)[b, :, H * D: (H + Hkv) * D].view(Q, Hkv, D)
        vn = qkv.float().view(B, Q, -1)[b, :, (H + Hkv) * D:].view(Q, Hkv, D)
        if table is not None:
            kn = llama_ref.rope(kn, torch.arange(p0, p0 + Q), table)
        torch.testing.assert_close(kcd[b, :, p0:p0 + Q].cpu().float().transpose(0, 1), kn, rtol=1e-2, atol=1e-2)
        torch.testing.assert_close(vcd[b, :, p0:p0 + Q].cpu().float().transpose(0, 1), vn, rtol=0, atol=0)


@pytest.mark.parametrize("T", [272, 400, 1500])
def test_tc_attention_batch_invariant(T):
    """Row (request b, position i) equals the same row computed with Q = i + 1
    (a shorter verify of the same prefix) and with the request alone — for the
    one-pass short-cache kernel (T <= 384) and the online-softmax one."""
    H, Hkv, D, Q = 64, 8, 128, 9
    B = 2
    g = torch.Generator().manual_seed(5)
    kc = torch.randn(B, Hkv, T, D, generator=g).to(BF)
    vc = torch.randn(B, Hkv, T, D, generator=g).to(BF)
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, generator=g).to(BF)
    # request 0's rows cross a 128-key chunk; at T = 1500 request 1 sees full
    # chunks (the online kernel's mask-free path) and a partial last one
    start = torch.tensor([122, 250 if T < 1000 else 1400], dtype=torch.int32)
    table = llama_ref.rope_table(T + 4, D, 10000.0)
    full = _run(qkv, B, Q, H, Hkv, D, start, kc.cuda(), vc.cuda(), table).cpu()
    q3 = qkv.view(B, Q, -1)[:, :4].reshape(B * 4, -1).contiguous()
    part = _run(q3, B, 4, H, Hkv, D, start, kc.cuda(), vc.cuda(), table).cpu()
    assert torch.equal(full.view(B, Q, -1)[:, :4], part.view(B, 4, -1))
    one = _run(qkv.view(B, Q, -1)[1].contiguous(), 1, Q, H, Hkv, D, start[1:], kc[1:].contiguous().cuda(),
               vc[1:].contiguous().cuda(), table).cpu()
    assert torch.equal(one, full.view(B, Q, -1)[1])


@pytest.mark.parametrize("H,Hkv,Q,T,starts,D", [(64, 8, 100, 300, [0, 60], 128), (40, 40, 300, 700, [0, 350], 128),
                                                (16, 2, 200, 1100, [0, 800], 128), (40, 40, 130, 4300, [4000, 0], 128),
                                                (12, 12, 300, 700, [0, 350], 64), (12, 12, 130, 1500, [1300, 7], 64)])
def test_tc_attention_prefill_tiles_vs_reference(H, Hkv, Q, T, starts, D):
    """Prompt-prefill calls (Q > 16 or Q * G > 128): the K / V rows appended,
    then 128-row query tiles of the online kernel — against the fp32
    restatement, GQA and multi-head, head dim 128 and 64 (the drafters),
    tiles crossing 128-key chunks."""
    B = len(starts)
    g = torch.Generator().manual_seed(H + Q + T)
    kc = torch.randn(B, Hkv, T, D, generator=g).to(BF)
    vc = torch.randn(B, Hkv, T, D, generator=g).to(BF)
    qkv = torch.randn(B * Q, (H + 2 * Hkv) * D, generator=g).to(BF)
    start = torch.tensor(starts, dtype=torch.int32)
    table = llama_ref.rope_table(T + 4, D, 10000.0)
    kcd, vcd = kc.cuda(), vc.cuda()
    got = _run(qkv, B, Q, H, Hkv, D, start, kcd, vcd, table).cpu().float()
    want = _ref_attention(qkv, kc, vc, start, B, Q, H, Hkv, D, table)
    torch.testing.assert_close(got, want, rtol=2e-2, atol=2e-2)
    for b in range(B):
        p0 = int(start[b])
        vn = qkv.float().view(B, Q, -1)[b, :, (H + Hkv) * D:].view(Q, Hkv, D)
        torch.testing.assert_close(vcd[b, :, p0:p0 + Q].cpu().float().transpose(0, 1), vn, rtol=0, atol=0)


def test_tc_attention_prefill_chunked_equals_whole():
    """A prompt prefilled in two calls gives bitwise the rows of one call
    (a row's arithmetic depends only on its position and keys)."""
    H, Hkv, D, T, P = 40, 40, 128, 640, 500
    g = torch.Generator().manual_seed(7)
    qkv = torch.randn(P, (H + 2 * Hkv) * D, generator=g).to(BF)
    table = llama_ref.rope_table(T + 4, D, 10000.0)
    z = torch.zeros(1, Hkv, T, D, dtype=BF)
    kc1, vc1 = z.clone().cuda(), z.clone().cuda()
    whole = _run(qkv, 1, P, H, Hkv, D, torch.tensor([0], dtype=torch.int32), kc1, vc1, table).cpu()
    kc2, vc2 = z.clone().cuda(), z.clone().cuda()
    a = _run(qkv[:300].contiguous(), 1, 300, H, Hkv, D, torch.tensor([0], dtype=torch.int32), kc2, vc2, table).cpu()
    b = _run(qkv[300:].contiguous(), 1, 200, H, Hkv, D, torch.tensor([300], dtype=torch.int32), kc2, vc2, table).cpu()
    assert torch.equal(torch.cat([a, b]), whole)
    assert torch.equal(kc1, kc2) and torch.equal(vc1, vc2)
