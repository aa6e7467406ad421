"""GPT MLP GEMMs with the bias / GELU work in the cuBLASLt epilogue
(csrc/mlp_lt.cpp, krt_mlp_fc1_gelu / krt_mlp_fc2_dgelu) vs torch fp32 on the
same bf16 operands: f1 = x w1^T + b1, g = gelu_tanh(f1); df1 = (dy w2) *
gelu_tanh'(f1).  Tolerances: bf16 rounding of the
outputs (2^-8 relative) on top of fp32 accumulation-order differences:
1e-2 of each tensor's max for the forward, 2e-2 for the backward (gelu'
evaluated on the bf16 f1 by two different implementations); repeat calls
bitwise equal."""
import pytest
import torch
import torch.nn.functional as F

from paper_2008_11421_b200 import lnfused

pytestmark = pytest.mark.gpu


def rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(torch.bfloat16)


def rel(a, b):
    return float((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6))


@pytest.mark.parametrize("T,H", [(256, 128), (1024, 256), (2048, 1920), (384, 3072)])
def test_fc1_gelu_and_fc2_dgelu(T, H):
    N = 4 * H
    x, w1, b1 = rand((T, H), 1), rand((N, H), 2, H ** -0.5), rand((N,), 3, 0.1)
    f1_out = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
    f1, g = lnfused.mlp_fc1_gelu(x, w1, b1, f1_out=f1_out)
    assert f1.data_ptr() == f1_out.data_ptr()
    ref_f1 = x.float() @ w1.float().t() + b1.float()
    assert rel(f1, ref_f1) < 1e-2
    assert rel(g, F.gelu(ref_f1, approximate="tanh")) < 1e-2
    # backward: dy [T, H], w2 [H, N]
    dy, w2 = rand((T, H), 4), rand((H, N), 5, N ** -0.5)
    df1 = lnfused.mlp_fc2_dgelu(dy, w2, f1)
    fr = f1.float().requires_grad_(True)
    gr = F.gelu(fr, approximate="tanh")
    (gr * (dy.float() @ w2.float())).sum().backward()
    ref_df1 = fr.grad
    assert rel(df1, ref_df1) < 2e-2
    # deterministic
    f1b, gb = lnfused.mlp_fc1_gelu(x, w1, b1)
    assert torch.equal(f1b, f1) and torch.equal(gb, g)
    assert torch.equal(lnfused.mlp_fc2_dgelu(dy, w2, f1), df1)


@pytest.mark.parametrize("T,H", [(256, 128), (2048, 1920)])
def test_fc2_residual(T, H):
    K = 4 * H
    g, w2, b2, x2 = rand((T, K), 6), rand((H, K), 7, K ** -0.5), rand((H,), 8, 0.1), rand((T, H), 9)
    y = lnfused.mlp_fc2_residual(g, w2, b2, x2)
    ref = x2.float() + g.float() @ w2.float().t() + b2.float()
    assert rel(y, ref) < 1e-2
    out = torch.empty_like(x2)
    assert torch.equal(lnfused.mlp_fc2_residual(g, w2, b2, x2, out=out), y)


@pytest.mark.parametrize("M,N,K", [(2048, 768, 256), (1024, 1920, 7680), (4096, 4256, 1064)])
def test_linear_wgrad_bgrad(M, N, K):
    """dW = dy^T x and db = dy.sum(0) from one cuBLASLt GEMM (BGRADB epilogue)
    vs fp32 torch on the same bf16 operands."""
    from paper_2008_11421_b200 import lnfused
    g = torch.Generator(device="cuda").manual_seed(9)
    dy = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    gw = torch.full((N, K), float("nan"), device="cuda")
    gb = torch.full((N,), float("nan"), device="cuda")
    assert lnfused.linear_wgrad_bgrad(dy, x, gw, gb)
    torch.testing.assert_close(gw, dy.float().t() @ x.float(), rtol=1e-3, atol=1e-2)
    torch.testing.assert_close(gb, dy.float().sum(0), rtol=1e-4, atol=1e-3)
