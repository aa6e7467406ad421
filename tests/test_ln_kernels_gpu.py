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


@pytest.mark.parametrize("T,H", [(64, 1920), (7, 4256), (33, 64), (1, 8), (64, 3072), (300, 4256), (10000, 3072)])
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


@pytest.mark.parametrize("T,H", [(1000, 1920), (257, 3072), (9, 4256), (33, 64), (600, 1024), (5000, 3072), (3001, 4256)])
@pytest.mark.parametrize("add", [False, True])
def test_ln_bwd(T, H, add):
    """One-pass LayerNorm backward vs fp32 autograd of layer_norm on the same
    bf16 input: dx (+ the residual gradient) at bf16 resolution, dgamma and
    dbeta (fp32, fixed-order sums) at fp32-reduction tolerance; bitwise
    repeatable."""
    x, dy, a = rand((T, H), 11, 2.0), rand((T, H), 12), rand((T, H), 13)
    g, b = rand((H,), 14, 0.2) + 1, rand((H,), 15, 0.1)
    m, s = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
    lnfused.ln_fwd(x, g, b, 1e-5, m, s)
    dg, db = torch.empty(H, device="cuda"), torch.empty(H, device="cuda")
    dx = lnfused.ln_bwd(dy, x, g, m, s, dg, db, addend=a if add else None)
    xf = x.float().requires_grad_(True)
    gf = g.float().requires_grad_(True)
    bf = b.float().requires_grad_(True)
    F.layer_norm(xf, [H], gf, bf, 1e-5).backward(dy.float())
    ref = xf.grad + (a.float() if add else 0)
    torch.testing.assert_close(dx.float(), ref, **BF16_TOL)
    torch.testing.assert_close(dg, gf.grad, rtol=2e-3, atol=2e-3)
    torch.testing.assert_close(db, bf.grad, rtol=1e-4, atol=1e-3)
    dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
    dx2 = lnfused.ln_bwd(dy, x, g, m, s, dg2, db2, addend=a if add else None)
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2) and torch.equal(db, db2)


@pytest.mark.parametrize("T,V", [(37, 128), (300, 51200), (5, 4104), (9, 65536), (2000, 51200)])
def test_lm_xent(T, V):
    """Fused next-token cross-entropy vs fp32 torch on the same bf16 logits:
    per-row losses at fp32 tolerance, dlogits at bf16 resolution; bitwise
    repeatable; lm_loss's fused branch equals the kernel's."""
    from paper_2008_11421_b200.units import lm_loss
    z = rand((T, V), 21, 4.0)
    g = torch.Generator(device="cuda").manual_seed(22)
    y = torch.randint(0, V, (T,), device="cuda", generator=g)
    y[0] = V - 1
    scale = 1.0 / T
    rl, dl = lnfused.lm_xent(z, y, scale)
    zf = z.float().requires_grad_(True)
    ref = F.cross_entropy(zf, y, reduction="none")
    ref.sum().mul(scale).backward()
    torch.testing.assert_close(rl, ref.detach(), rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(dl.float(), zf.grad, rtol=1.6e-2, atol=1e-6 * scale + 1e-8)
    rl2, dl2 = lnfused.lm_xent(z, y, scale)
    assert torch.equal(rl, rl2) and torch.equal(dl, dl2)
    loss, dl3 = lm_loss(z, y)
    assert torch.equal(dl3, dl)
    torch.testing.assert_close(loss, ref.detach().mean(), rtol=1e-5, atol=1e-6)
