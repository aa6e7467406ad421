"""Fused NHWC batch-norm kernels (csrc/bn_kernels.cu) vs a torch fp32
reference on the same bf16 inputs.  Tolerances: statistics and parameter
gradients are fp32 reductions (rtol 1e-4 / 1e-3); bf16 outputs are compared
at bf16 resolution (one ulp = 2^-8 relative)."""
import pytest
import torch
import torch.nn.functional as F

from paper_2008_11421_b200 import bnfused

pytestmark = pytest.mark.gpu
BF16_TOL = dict(rtol=1.6e-2, atol=1.6e-2)


def rand(n, c, h, w, scale=1.0, shift=0.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    t = torch.randn(n, c, h, w, device="cuda", generator=g) * scale + shift
    return t.to(torch.bfloat16).contiguous(memory_format=torch.channels_last)


def params(c, seed=1):
    g = torch.Generator(device="cuda").manual_seed(seed)
    gamma = (1 + 0.2 * torch.randn(c, device="cuda", generator=g)).to(torch.bfloat16)
    beta = (0.1 * torch.randn(c, device="cuda", generator=g)).to(torch.bfloat16)
    return gamma, beta


def ref_stats(x):
    xf = x.float()
    mean = xf.mean(dim=(0, 2, 3))
    var = xf.var(dim=(0, 2, 3), unbiased=False)
    return mean, torch.rsqrt(var + bnfused.EPS)


@pytest.mark.parametrize("shape", [(64, 64, 28, 28), (16, 256, 14, 14), (8, 2048, 7, 7), (3, 128, 5, 7)])
def test_stats_and_apply(shape):
    n, c, h, w = shape
    x = rand(*shape, scale=2.0, shift=0.5)
    g, b = params(c)
    m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    bnfused.stats(x, m, i)
    rm, ri = ref_stats(x)
    torch.testing.assert_close(m, rm, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(i, ri, rtol=1e-4, atol=1e-5)
    pre = ((x.float() - rm[None, :, None, None]) * ri[None, :, None, None] * g.float()[None, :, None, None]
           + b.float()[None, :, None, None])
    y = bnfused.apply(x, m, i, g, b, relu=True)
    torch.testing.assert_close(y.float(), F.relu(pre), **BF16_TOL)
    # residual forms: identity and bn'(res)
    r = rand(*shape, seed=5)
    y1 = bnfused.apply(x, m, i, g, b, relu=True, res=r)
    torch.testing.assert_close(y1.float(), F.relu(pre + r.float()), **BF16_TOL)
    y2 = bnfused.apply(x, m, i, g, b, relu=False, res=x, rstats=(m, i), rg=g, rb=b)
    torch.testing.assert_close(y2.float(), 2 * pre, **BF16_TOL)


def bn_ref_fwd(x, g, b):
    return F.batch_norm(x, None, None, g, b, training=True, momentum=0.0, eps=bnfused.EPS)


@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("shape", [(32, 64, 28, 28), (16, 512, 7, 7), (4, 2048, 7, 7)])
def test_backward_matches_autograd(shape, relu):
    n, c, h, w = shape
    x = rand(*shape, scale=1.5, shift=0.2, seed=2)
    dy = rand(*shape, seed=3)
    g, b = params(c, seed=4)
    m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    bnfused.stats(x, m, i)
    dg, db = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    dx = bnfused.backward(dy, x, m, i, g, b, relu=relu, dgamma=dg, dbeta=db)
    xr = x.float().requires_grad_(True)
    gr = g.float().requires_grad_(True)
    br = b.float().requires_grad_(True)
    out = bn_ref_fwd(xr, gr, br)
    if relu:
        out = F.relu(out)
    out.backward(dy.float())
    torch.testing.assert_close(db, br.grad, rtol=1e-3, atol=1e-2)
    torch.testing.assert_close(dg, gr.grad, rtol=1e-3, atol=1e-2)
    err = (dx.float() - xr.grad).abs().max() / xr.grad.abs().max()
    assert err < 2e-2, float(err)


def test_add_relu_backward_mask():
    shape = (8, 256, 14, 14)
    x = rand(*shape, seed=7)
    r = rand(*shape, seed=8)
    dy = rand(*shape, seed=9)
    g, b = params(256)
    gd, bd = params(256, seed=11)
    m, i = torch.empty(256, device="cuda"), torch.empty(256, device="cuda")
    md, idd = torch.empty(256, device="cuda"), torch.empty(256, device="cuda")
    bnfused.stats(x, m, i)
    bnfused.stats(r, md, idd)
    y = bnfused.apply(x, m, i, g, b, relu=True, res=r, rstats=(md, idd), rg=gd, rb=bd)
    dz = bnfused.add_relu_bwd(dy, x, m, i, g, b, r, rstats=(md, idd), rg=gd, rb=bd)
    assert torch.equal(dz, torch.where(y > 0, dy, torch.zeros_like(dy)))
    y1 = bnfused.apply(x, m, i, g, b, relu=True, res=r)
    dz1 = bnfused.add_relu_bwd(dy, x, m, i, g, b, r)
    assert torch.equal(dz1, torch.where(y1 > 0, dy, torch.zeros_like(dy)))


def test_add_relu_backward_second_gradient():
    shape = (8, 256, 14, 14)
    x, r, dy, dy2 = (rand(*shape, seed=s) for s in (21, 22, 23, 24))
    g, b = params(256)
    m, i = torch.empty(256, device="cuda"), torch.empty(256, device="cuda")
    bnfused.stats(x, m, i)
    y = bnfused.apply(x, m, i, g, b, relu=True, res=r)
    dz = bnfused.add_relu_bwd(dy, x, m, i, g, b, r, dy2=dy2)
    ref = torch.where(y > 0, dy + dy2, torch.zeros_like(dy))
    assert torch.equal(dz, ref)


@pytest.mark.parametrize("shape", [(64, 64, 28, 28), (8, 2048, 7, 7), (3, 128, 5, 7), (1, 8, 1, 3), (2, 256, 1, 1)])
@pytest.mark.parametrize("residual", [False, True])
def test_stats_apply_fused(shape, residual):
    """stats + apply in one cooperative kernel == the torch fp32 reference,
    and equal to the two separate kernels up to the last bit of the stats."""
    n, c, h, w = shape
    x = rand(*shape, scale=2.0, shift=0.5, seed=31)
    r = rand(*shape, seed=32) if residual else None
    g, b = params(c, seed=33)
    m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    y = bnfused.stats_apply(x, m, i, g, b, relu=True, res=r)
    rm, ri = ref_stats(x)
    torch.testing.assert_close(m, rm, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(i, ri, rtol=1e-4, atol=1e-5)
    pre = ((x.float() - rm[None, :, None, None]) * ri[None, :, None, None] * g.float()[None, :, None, None]
           + b.float()[None, :, None, None])
    if residual:
        pre = pre + r.float()
    torch.testing.assert_close(y.float(), F.relu(pre), **BF16_TOL)
    m2, i2 = torch.empty_like(m), torch.empty_like(i)
    bnfused.stats(x, m2, i2)
    torch.testing.assert_close(m2, m, rtol=1e-6, atol=1e-7)
    y2 = bnfused.apply(x, m, i, g, b, relu=True, res=r)
    assert torch.equal(y, y2)  # same stats -> the apply pass is bit-identical
    # deterministic: a second launch is bitwise equal
    m3, i3 = torch.empty_like(m), torch.empty_like(i)
    y3 = bnfused.stats_apply(x, m3, i3, g, b, relu=True, res=r)
    assert torch.equal(m3, m) and torch.equal(i3, i) and torch.equal(y3, y)


@pytest.mark.parametrize("shape", [(8, 256, 14, 14), (4, 2048, 7, 7), (3, 64, 5, 7)])
@pytest.mark.parametrize("two", [False, True])
def test_add_relu_backward_fused(shape, two):
    """add_relu_bwd + backward(relu=False) fused == the two kernels: dz bitwise,
    dgamma/dbeta/dx within fp32-reduction / bf16 resolution."""
    n, c, h, w = shape
    x, r, dy, dy2 = (rand(*shape, seed=s) for s in (41, 42, 43, 44))
    dy2 = dy2 if two else None
    g, b = params(c, seed=45)
    m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    bnfused.stats(x, m, i)
    dg, db = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    dz, dx = bnfused.add_relu_backward(dy, x, m, i, g, b, r, dgamma=dg, dbeta=db, dy2=dy2)
    dz_ref = bnfused.add_relu_bwd(dy, x, m, i, g, b, r, dy2=dy2)
    assert torch.equal(dz, dz_ref)
    dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
    dx2 = bnfused.backward(dz_ref, x, m, i, g, b, relu=False, dgamma=dg2, dbeta=db2)
    torch.testing.assert_close(db, db2, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(dg, dg2, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(dx.float(), dx2.float(), **BF16_TOL)
    # against autograd of bn (no relu) on dz
    xr = x.float().requires_grad_(True)
    gr, br = g.float().requires_grad_(True), b.float().requires_grad_(True)
    bn_ref_fwd(xr, gr, br).backward(dz.float())
    torch.testing.assert_close(db, br.grad, rtol=1e-3, atol=1e-2)
    torch.testing.assert_close(dg, gr.grad, rtol=1e-3, atol=1e-2)
    err = (dx.float() - xr.grad).abs().max() / xr.grad.abs().max()
    assert err < 2e-2, float(err)


def test_backward_no_dx_and_tiny_rows():
    """dx=None path (reduce only) and rows smaller than one CTA sweep."""
    for shape in [(1, 64, 1, 1), (2, 8, 1, 1), (1, 2048, 1, 2)]:
        n, c, h, w = shape
        x, dy = rand(*shape, seed=51), rand(*shape, seed=52)
        g, b = params(c, seed=53)
        m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
        bnfused.stats(x, m, i)
        dg, db = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
        assert bnfused.backward(dy, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db, need_dx=False) is None
        dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
        bnfused.backward(dy, x, m, i, g, b, relu=True, dgamma=dg2, dbeta=db2)
        torch.testing.assert_close(dg, dg2, rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(db, db2, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("shape,ksp", [((4, 64, 112, 112), (3, 2, 1)), ((3, 16, 9, 7), (3, 2, 1)), ((2, 64, 13, 11), (3, 2, 1)),
                                       ((2, 8, 6, 6), (2, 2, 0)), ((2, 32, 11, 13), (3, 1, 1)), ((2, 64, 10, 10), (5, 3, 2))])
def test_relu_maxpool_matches_aten_bitwise(shape, ksp):
    """maxpool(relu(bn(c))) fused, forward and backward, == apply -> aten
    max_pool2d_with_indices -> max_pool2d_with_indices_backward, bitwise
    (ties included: a coarse input makes equal maxima common)."""
    k, s, p = ksp
    n, c, h, w = shape
    x = (rand(*shape, scale=2.0, seed=61).float() * 4).round().div(4).to(torch.bfloat16)
    x = x.contiguous(memory_format=torch.channels_last)
    g, b = params(c, seed=62)
    m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    bnfused.stats(x, m, i)
    a = bnfused.apply(x, m, i, g, b, relu=True)
    y_ref, idx = torch.ops.aten.max_pool2d_with_indices(a, [k, k], [s, s], [p, p])
    y = bnfused.relu_maxpool(x, m, i, g, b, k, s, p)
    assert y.shape == y_ref.shape and torch.equal(y, y_ref)
    dy = rand(*y.shape, seed=63).contiguous(memory_format=torch.channels_last)
    da_ref = torch.ops.aten.max_pool2d_with_indices_backward(dy, a, [k, k], [s, s], [p, p], [1, 1], False, idx)
    da = bnfused.relu_maxpool_backward(dy, x, m, i, g, b, k, s, p)
    assert torch.equal(da, da_ref)


def test_backward_with_addend():
    """bn backward + residual-gradient addend in one pass == backward then add,
    within one bf16 rounding (the fused version rounds once)."""
    shape = (4, 64, 16, 16)
    x, dy, r = rand(*shape, seed=71), rand(*shape, seed=72), rand(*shape, seed=73)
    g, b = params(64, seed=74)
    m, i = torch.empty(64, device="cuda"), torch.empty(64, device="cuda")
    bnfused.stats(x, m, i)
    dg, db = torch.empty(64, device="cuda"), torch.empty(64, device="cuda")
    dx = bnfused.backward(dy, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db, addend=r)
    dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
    ref = bnfused.backward(dy, x, m, i, g, b, relu=True, dgamma=dg2, dbeta=db2).float() + r.float()
    assert torch.equal(dg, dg2) and torch.equal(db, db2)
    torch.testing.assert_close(dx.float(), ref, **BF16_TOL)
