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
    old = Kn.TC_ATTENTION
    Kn.TC_ATTENTION = True
    try:
        return Kn.attention(qkv.cuda(), B, Q, H, D, torch.arange(B, dtype=torch.int32).cuda(), start.cuda(), kc, vc,
                            D ** -0.5, n_kv_heads=Hkv, rope=None if table is None else table.cuda())
    finally:
        Kn.TC_ATTENTION = old


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
