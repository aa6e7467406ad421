"""tcgen05 1x1-convolution GEMM (csrc/gemm_sm100.cu) vs torch: the GEMM in fp32
(tolerance: bf16 output rounding, one ulp = 2^-8 relative, plus fp32
accumulation-order differences), the fused BN+ReLU prologue and the fused
statistics epilogue (vs the stats kernel on the stored output: rtol 1e-4)."""
import pytest
import torch
import torch.nn.functional as F

from paper_2008_11421_b200 import bnfused

pytestmark = pytest.mark.gpu


def rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(torch.bfloat16)


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


@pytest.mark.parametrize("n,cin,cout,hw", [(2, 64, 64, 8), (4, 256, 64, 14), (2, 64, 256, 7), (3, 128, 512, 5),
                                           (1, 512, 2048, 3), (2, 1024, 256, 6), (2, 256, 1024, 6),
                                           (1, 64, 2048, 5), (3, 128, 512, 17),
                                           # narrow reductions: one 16/32-wide k-block (SWIZZLE_32B/64B)
                                           (2, 16, 64, 8), (3, 32, 128, 9), (2, 16, 256, 7), (1, 32, 64, 17),
                                           # narrow n-tiles: 16/32-column accumulators and epilogue
                                           (2, 64, 16, 8), (3, 128, 32, 9), (1, 16, 16, 17), (2, 32, 32, 13),
                                           (2, 256, 64, 11),
                                           # several tiles per CTA (> 148 x 128 rows): tile groups, accumulators
                                           (8, 64, 16, 96), (4, 128, 32, 100), (2, 256, 64, 150), (2, 64, 256, 130),
                                           (1, 256, 1024, 160)])
@pytest.mark.parametrize("pre", [False, True])
def test_conv1x1_matches_torch(n, cin, cout, hw, pre):
    x = cl(rand((n, cin, hw, hw), 1, 2.0))
    w = cl(rand((cout, cin, 1, 1), 2, cin ** -0.5))
    if pre:
        g = (1 + 0.2 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
        b = (0.1 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
        m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
        bnfused.stats(x, m, i)
        a = bnfused.apply(x, m, i, g, b, relu=True)   # what the prologue must reproduce
        pre_t = (m, i, g, b)
    else:
        a, pre_t = x, None
    sm, si = torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda")
    y = bnfused.conv1x1(x, w, pre=pre_t, stats=(sm, si))
    torch.cuda.synchronize()
    ref = F.conv2d(a.float(), w.float())
    err = (y.float() - ref).abs().max() / ref.abs().max()
    assert err < 1e-2, float(err)
    # fused statistics == statistics of the stored bf16 output
    rm, ri = torch.empty_like(sm), torch.empty_like(si)
    bnfused.stats(y, rm, ri)
    torch.testing.assert_close(sm, rm, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(si, ri, rtol=1e-4, atol=1e-5)
    # deterministic
    sm2, si2 = torch.empty_like(sm), torch.empty_like(si)
    y2 = bnfused.conv1x1(x, w, pre=pre_t, stats=(sm2, si2))
    assert torch.equal(y, y2) and torch.equal(sm, sm2) and torch.equal(si, si2)


def test_conv1x1_ragged_rows_and_out():
    """M not a multiple of the 128-row tile, output into a preallocated view."""
    x = cl(rand((1, 128, 13, 11), 3))      # M = 143
    w = cl(rand((256, 128, 1, 1), 4, 0.1))
    out = torch.empty((1, 256, 13, 11), dtype=torch.bfloat16, device="cuda", memory_format=torch.channels_last)
    y = bnfused.conv1x1(x, w, out=out)
    assert y.data_ptr() == out.data_ptr()
    ref = F.conv2d(x.float(), w.float())
    assert ((y.float() - ref).abs().max() / ref.abs().max()) < 1e-2


@pytest.mark.parametrize("n,cin,cout,hw", [(2, 64, 256, 8), (3, 128, 512, 7), (1, 256, 1024, 6), (2, 512, 2048, 3),
                                           (1, 64, 256, 13)])
def test_conv1x1_dgrad_bn_backward(n, cin, cout, hw):
    """dgrad of conv(relu(bn(x))) through the tcgen05 GEMM with the BN reduce in
    its epilogue == torch conv dgrad + the standalone BN backward kernels:
    dgamma/dbeta at fp32-reduction tolerance, dx at bf16 resolution."""
    x = cl(rand((n, cin, hw, hw), 11, 1.5))
    dy = cl(rand((n, cout, hw, hw), 12))
    w = cl(rand((cout, cin, 1, 1), 13, cin ** -0.5))
    g = (1 + 0.2 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
    b = (0.1 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
    m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
    bnfused.stats(x, m, i)
    dg, db = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
    dx = bnfused.conv1x1_dgrad_bn_backward(dy, w, x, m, i, g, b, dgamma=dg, dbeta=db)
    # reference: torch dgrad in fp32, rounded to bf16 like the stored gradient, then the BN kernels
    da = torch.nn.grad.conv2d_input(x.shape, w.float(), dy.float()).to(torch.bfloat16)
    da = cl(da)
    dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
    dx2 = bnfused.backward(da, x, m, i, g, b, relu=True, dgamma=dg2, dbeta=db2)
    torch.testing.assert_close(db, db2, rtol=2e-3, atol=2e-2)
    torch.testing.assert_close(dg, dg2, rtol=2e-3, atol=2e-2)
    err = (dx.float() - dx2.float()).abs().max() / dx2.float().abs().max()
    assert err < 2e-2, float(err)
    # deterministic
    dx3 = bnfused.conv1x1_dgrad_bn_backward(dy, w, x, m, i, g, b)
    assert torch.equal(dx, dx3)


@pytest.mark.parametrize("n,cin,cout,hw", [(2, 16, 64, 8), (2, 32, 128, 9), (2, 64, 256, 7), (1, 128, 512, 13),
                                           (2, 64, 16, 6), (3, 16, 32, 17), (1, 256, 1024, 5),
                                           # several tiles per CTA: every residual buffer and tile group cycles
                                           (8, 16, 64, 96), (4, 32, 128, 100), (2, 64, 256, 150)])
@pytest.mark.parametrize("pre", [True, False])
def test_conv1x1_residual_epilogue(n, cin, cout, hw, pre):
    """C = relu(bn(x)) . W^T + res, the residual tile TMA-loaded into the
    epilogue (the pre-activation bottleneck's conv3 + shortcut), with and
    without the batch statistics of C."""
    x = cl(rand((n, cin, hw, hw), 5, 2.0))
    w = cl(rand((cout, cin, 1, 1), 6, cin ** -0.5))
    res = cl(rand((n, cout, hw, hw), 7))
    if pre:
        g = (1 + 0.2 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
        b = (0.1 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
        m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
        bnfused.stats(x, m, i)
        a, pre_t = bnfused.apply(x, m, i, g, b, relu=True), (m, i, g, b)
    else:
        a, pre_t = x, None
    y = bnfused.conv1x1(x, w, pre=pre_t, res=res)
    torch.cuda.synchronize()
    ref = F.conv2d(a.float(), w.float()) + res.float()
    err = (y.float() - ref).abs().max() / ref.abs().max()
    assert err < 1e-2, float(err)
    # the sum is rounded once: equal to bf16(acc + res) up to the fp32 accumulation order
    plain = bnfused.conv1x1(x, w, pre=pre_t)
    bound = 2 ** -7 * (plain.float().abs() + res.float().abs()) + 1e-3   # one bf16 ulp of each term
    assert ((y.float() - (plain.float() + res.float())).abs() <= bound).all()
    assert torch.equal(y, bnfused.conv1x1(x, w, pre=pre_t, res=res))   # deterministic
    # EPI 4: the statistics of the stored sum reduced in the same epilogue
    # (the next pre-activation unit's BN0 statistics), vs the stats kernel
    sm, si = torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda")
    y2 = bnfused.conv1x1(x, w, pre=pre_t, res=res, stats=(sm, si))
    assert torch.equal(y2, y)
    rm, ri = torch.empty_like(sm), torch.empty_like(si)
    bnfused.stats(y, rm, ri)
    torch.testing.assert_close(sm, rm, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(si, ri, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("n,cout,cin,hw", [(4, 16, 64, 40), (2, 32, 128, 50), (8, 64, 256, 30), (2, 256, 64, 150)])
def test_conv1x1_dgrad_bn_backward_narrow(n, cout, cin, hw):
    """Narrow reductions (K = Cout = 16/32) in the dgrad + BN-backward-reduce
    GEMM, with the shortcut gradient as addend: vs autograd in fp32 through
    conv(relu(bn(x))) + the addend (tolerance: bf16 rounding of the stored
    intermediate gradient)."""
    x = cl(rand((n, cin, hw, hw), 11, 1.5))
    w = cl(rand((cout, cin, 1, 1), 12, cin ** -0.5))
    dy = cl(rand((n, cout, hw, hw), 13))
    add = cl(rand((n, cin, hw, hw), 14))
    g = (1 + 0.2 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
    b = (0.1 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
    m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
    bnfused.stats(x, m, i)
    dg, db = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
    dx = bnfused.conv1x1_dgrad_bn_backward(dy, w, x, m, i, g, b, dgamma=dg, dbeta=db, addend=add)
    # reference: the unfused kernels on the GEMM's stored da (same rounding point)
    da = F.conv2d(dy.float(), w.float().transpose(0, 1)).to(torch.bfloat16)
    dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
    ref = bnfused.backward(cl(da), x, m, i, g, b, relu=True, dgamma=dg2, dbeta=db2, addend=add)
    torch.cuda.synchronize()
    err = (dx.float() - ref.float()).abs().max() / ref.float().abs().max()
    assert err < 2e-2, float(err)
    torch.testing.assert_close(db, db2, rtol=2e-2, atol=2e-2 * db2.abs().max().item())
    torch.testing.assert_close(dg, dg2, rtol=2e-2, atol=2e-2 * dg2.abs().max().item())


@pytest.mark.parametrize("n,cin,hw,k,s,pad", [(2, 3, 224, 7, 2, 3), (3, 3, 37, 7, 2, 3), (1, 4, 30, 3, 1, 1),
                                              (12, 3, 64, 7, 2, 3)])
def test_conv_gather_matches_torch(n, cin, hw, k, s, pad):
    """Implicit-GEMM stem convolution (im2col gathered in shared memory) vs the
    fp32 convolution; fused statistics vs the stats kernel on the stored output."""
    x = cl(rand((n, cin, hw, hw), 21, 1.0))
    w = cl(rand((64, cin, k, k), 22, (cin * k * k) ** -0.5))
    sm, si = torch.empty(64, device="cuda"), torch.empty(64, device="cuda")
    y = bnfused.conv_gather(x, w, s, pad, stats=(sm, si))
    torch.cuda.synchronize()
    ref = F.conv2d(x.float(), w.float(), stride=s, padding=pad)
    assert y.shape == ref.shape
    err = (y.float() - ref).abs().max() / ref.abs().max()
    assert err < 1e-2, float(err)
    rm, ri = torch.empty_like(sm), torch.empty_like(si)
    bnfused.stats(y, rm, ri)
    torch.testing.assert_close(sm, rm, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(si, ri, rtol=1e-4, atol=1e-5)
    assert torch.equal(y, bnfused.conv_gather(x, w, s, pad))


@pytest.mark.parametrize("pixels", [1, 2, 7, 4107, 100000])
def test_pad_rgb4(pixels):
    from paper_2008_11421_b200 import _lib
    x = rand((pixels, 3), 31)
    y = torch.full((pixels, 4), 7.0, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.lib().krt_pad_rgb4(x.data_ptr(), y.data_ptr(), pixels, None))
    torch.cuda.synchronize()
    assert torch.equal(y[:, :3], x) and bool((y[:, 3] == 0).all())
