"""ms_linear_wide (csrc/gemm_pair.cu): the prefill GEMM on tcgen05 CTA pairs
(cta_group::2, persistent, double-buffered TMEM).  Checked against the fp32
torch product of the same bf16 operands, on every epilogue (bias / ReLU /
residual in place / gated SiLU / fp32 out) and on ragged M, N, K tails;
deterministic (bitwise equal on a second run)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(x, w, b, r, act, f32):
    y = x.float() @ w.float().t()
    if b is not None:
        y = y + b.float()
    if act == 1:
        y = torch.relu(y)
    if act == 2:
        F = w.shape[0] // 2
        j = torch.arange(F, device=w.device)
        gate = (j // 64) * 128 + j % 64
        g, u = y[:, gate], y[:, gate + 64]
        y = g / (1 + torch.exp(-g)) * u
    if r is not None:
        y = y + r.float()
    return y if f32 else y.to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(256, 1024, 512), (1000, 3072, 768), (37, 640, 256), (2048, 8192, 1024),
                                   (300, 1000, 200), (512, 57344 // 16, 8192), (129, 768, 3072)])
def test_wide_linear_vs_torch(M, N, K):
    from paper_2402_15678_b200 import kernels as Kn
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device="cuda") * 0.03).to(torch.bfloat16)
    b = torch.randn(N, generator=g, device="cuda").to(torch.bfloat16)
    r = torch.randn(M, N, generator=g, device="cuda").to(torch.bfloat16)
    tol = dict(rtol=1.6e-2, atol=2e-2)
    # fp32 out, no epilogue
    got = Kn.linear_wide(x, w, out_f32=True)
    torch.testing.assert_close(got, _ref(x, w, None, None, 0, True), rtol=1e-4, atol=3e-5 * K ** 0.5)
    assert torch.equal(got, Kn.linear_wide(x, w, out_f32=True))  # deterministic
    # bias + relu, bf16
    torch.testing.assert_close(Kn.linear_wide(x, w, b, act=1).float(), _ref(x, w, b, None, 1, False).float(), **tol)
    # residual in place (out is residual), bf16
    rr = r.clone()
    Kn.linear_wide(x, w, residual=rr, out=rr)
    torch.testing.assert_close(rr.float(), _ref(x, w, None, r, 0, False).float(), **tol)
    # gated SiLU (N % 128 == 0)
    if N % 128 == 0:
        torch.testing.assert_close(Kn.linear_wide(x, w, act=2).float(), _ref(x, w, None, None, 2, False).float(),
                                   **tol)


def test_wide_matches_cluster_path_one_split():
    """Same k order as ms_linear's one-split cluster path (a k-block of 64 as
    four K=16 MMAs, fp32 accumulation in TMEM)."""
    from paper_2402_15678_b200 import kernels as Kn
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(512, 2048, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(4096, 2048, generator=g, device="cuda") * 0.03).to(torch.bfloat16)
    a = Kn.linear_wide(x, w, out_f32=True)
    c = Kn.linear(x, w, out_f32=True, splits=1)
    assert (a - c).abs().max().item() <= 1e-5 * a.abs().max().item()
