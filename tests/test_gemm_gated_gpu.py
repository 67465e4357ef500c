"""The persistent gated schedule (csrc/gemm_gated.cuh) for one-split gated
GEMMs wider than two CTAs per SM (the 70B gate/up): bitwise equal to the
one-tile-per-CTA path (ms_set_gated_persistent(0)) for every token-tile width
it takes, with and without the folded-RMSNorm scaling, and against a float64
reference."""
import pytest
import torch

pytestmark = pytest.mark.gpu
BF = torch.bfloat16


@pytest.fixture(scope="module")
def gu():
    g = torch.Generator().manual_seed(11)
    F, K = 28672, 8192
    w = (torch.randn(2 * F, K, generator=g) * 0.02).to(BF).cuda()
    x = torch.randn(160, K, generator=g).to(BF).cuda()
    return x, w, F, K


def _both(fn):
    from paper_2402_15678_b200 import _native
    old = _native.lib.ms_set_gated_persistent(0)
    try:
        base = fn()
    finally:
        _native.lib.ms_set_gated_persistent(1)
    pers = fn()
    _native.lib.ms_set_gated_persistent(old)
    return base, pers


@pytest.mark.parametrize("M", [1, 16, 33, 80, 112, 128, 160])
def test_persistent_gated_bitwise_equal(gu, M):
    from paper_2402_15678_b200 import kernels as Kn
    x, w, F, K = gu
    base, pers = _both(lambda: Kn.linear(x[:M], w, act=2))
    assert torch.equal(base, pers)
    if M in (1, 112):
        y = x[:M].double().cpu() @ w.double().cpu().T
        t = y.view(M, -1, 2, 64)
        g_, u_ = t[:, :, 0].reshape(M, F), t[:, :, 1].reshape(M, F)
        torch.testing.assert_close(pers.cpu().float(), (g_ * torch.sigmoid(g_) * u_).float(), rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("M", [16, 112])
def test_persistent_gated_folded_norm_bitwise_equal(gu, M):
    from paper_2402_15678_b200 import kernels as Kn
    x, w, F, K = gu
    parts = (x[:M].float().view(M, K // 128, 128) ** 2).sum(-1).contiguous()

    def run():
        out = torch.empty(M, F, dtype=BF, device="cuda")
        Kn.linear_rms(x[:M], w, act=2, out=out, rms_in=parts, eps=1e-5)
        return out
    base, pers = _both(run)
    assert torch.equal(base, pers)
