"""GPT-layer kernels (csrc/ln_kernels.cu) vs torch: LayerNorm with the fused
residual add (bf16 outputs at bf16 resolution, statistics at fp32-reduction
tolerance) and GELU backward with fused bias-gradient column sums."""
import pytest
import torch
import torch.nn.functional as F

from paper_2008_11421_b200 import lnfused

pytestmark = pytest.mark.gpu
BF16_TOL = dict(rtol=1.6e-2, atol=1.6e-2)


def rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("T,H", [(64, 1920), (7, 4256), (33, 64), (1, 8)])
@pytest.mark.parametrize("res", [False, True])
def test_ln_fwd(T, H, res):
    x, r = rand((T, H), 1, 2.0), rand((T, H), 2)
    g, b = rand((H,), 3, 0.2) + 1, rand((H,), 4, 0.1)
    m, s = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
    x2 = torch.empty_like(x)
    h = lnfused.ln_fwd(x, g, b, 1e-5, m, s, residual=r if res else None, x2_out=x2 if res else None)
    src = (x.float() + r.float()).to(torch.bfloat16) if res else x
    if res:
        assert torch.equal(x2, src)
    ref, rm, rr = torch.ops.aten.native_layer_norm(src.float(), [H], g.float(), b.float(), 1e-5)
    torch.testing.assert_close(h.float(), ref, **BF16_TOL)
    torch.testing.assert_close(m, rm.view(-1), rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(s, rr.view(-1), rtol=1e-3, atol=1e-3)
    h2 = lnfused.ln_fwd(x, g, b, 1e-5, torch.empty_like(m), torch.empty_like(s),
                        residual=r if res else None, x2_out=torch.empty_like(x) if res else None)
    assert torch.equal(h, h2)   # deterministic: the backward recompute is bitwise the forward


@pytest.mark.parametrize("T,N", [(300, 7680), (5, 64), (257, 2056)])
def test_gelu_bwd_colsum(T, N):
    f, dy = rand((T, N), 5, 2.0), rand((T, N), 6)
    cs = torch.empty(N, device="cuda")
    dx = lnfused.gelu_bwd_colsum(dy, f, cs)
    ref = torch.ops.aten.gelu_backward(dy, f, approximate="tanh")
    torch.testing.assert_close(dx.float(), ref.float(), **BF16_TOL)
    torch.testing.assert_close(cs, dx.float().sum(0), rtol=1e-4, atol=1e-3)
    cs2 = torch.empty_like(cs)
    assert torch.equal(lnfused.gelu_bwd_colsum(dy, f, cs2), dx) and torch.equal(cs2, cs)
