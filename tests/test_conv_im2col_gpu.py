"""Implicit-GEMM convolution with im2col TMA tiles (csrc/gemm_sm100.cu,
krt_conv_im2col_bn) vs torch fp32: 3x3 stride 1/2 and 1x1 stride 2, with the
fused relu(bn(.)) prologue (taps in the zero padding must stay zero: the
reference convolves the bn_apply output, zero-padded) and the statistics
epilogue; and the dgrad form with the BN-backward reduce in its epilogue.
Tolerances: bf16 output rounding (one ulp = 2^-8 relative) plus fp32
accumulation order; fused statistics vs the stats kernel on the stored
output at rtol 1e-4."""
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


def bn_params(c, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return ((1 + 0.2 * torch.randn(c, device="cuda", generator=g)).to(torch.bfloat16),
            (0.1 * torch.randn(c, device="cuda", generator=g)).to(torch.bfloat16))


@pytest.mark.parametrize("n,cin,cout,h,k,s", [(2, 64, 64, 8, 3, 1), (2, 128, 128, 14, 3, 1), (1, 256, 256, 7, 3, 1),
                                              (2, 512, 512, 7, 3, 1), (3, 64, 256, 9, 3, 1), (2, 128, 128, 14, 3, 2),
                                              (1, 256, 1024, 14, 1, 2), (4, 64, 128, 30, 3, 1),
                                              (16, 128, 128, 28, 3, 1)])
@pytest.mark.parametrize("pre", [False, True])
def test_conv_im2col_matches_torch(n, cin, cout, h, k, s, pre):
    pad = k // 2
    x = cl(rand((n, cin, h, h), 1, 2.0))
    w = rand((cout, k, k, cin), 2, (cin * k * k) ** -0.5).contiguous()
    if pre:
        g, b = bn_params(cin, 3)
        m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
        bnfused.stats(x, m, i)
        a, pre_t = bnfused.apply(x, m, i, g, b, relu=True), (m, i, g, b)
    else:
        a, pre_t = x, None
    sm, si = torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda")
    y = bnfused.conv_im2col(x, w, s, pad, pre=pre_t, stats=(sm, si))
    torch.cuda.synchronize()
    ref = F.conv2d(a.float(), w.permute(0, 3, 1, 2).float(), stride=s, padding=pad)
    assert y.shape == ref.shape
    err = (y.float() - ref).abs().max() / ref.abs().max()
    assert err < 1e-2, float(err)
    rm, ri = torch.empty_like(sm), torch.empty_like(si)
    bnfused.stats(y, rm, ri)
    torch.testing.assert_close(sm, rm, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(si, ri, rtol=1e-4, atol=1e-5)
    assert torch.equal(y, bnfused.conv_im2col(x, w, s, pad, pre=pre_t))   # deterministic


@pytest.mark.parametrize("n,cin,cout,h", [(2, 64, 64, 8), (2, 128, 128, 14), (1, 256, 256, 7), (2, 512, 512, 7),
                                          (4, 128, 128, 28)])
def test_conv_im2col_dgrad_bn_backward(n, cin, cout, h):
    """dx of conv3x3(relu(bn(x))): the dgrad GEMM (flipped, transposed weight)
    with BN's backward reduce fused == torch's fp32 dgrad rounded to bf16 then
    the standalone BN backward kernel."""
    x = cl(rand((n, cin, h, h), 11, 1.5))
    dy = cl(rand((n, cout, h, h), 12))
    w = rand((cout, 3, 3, cin), 13, (9 * cin) ** -0.5).contiguous()
    g, b = bn_params(cin, 14)
    m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
    bnfused.stats(x, m, i)
    dg, db = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
    dx = bnfused.conv_im2col_dgrad_bn_backward(dy, w, x, m, i, g, b, dgamma=dg, dbeta=db)
    da = cl(torch.nn.grad.conv2d_input(x.shape, w.permute(0, 3, 1, 2).float(), dy.float(), padding=1)
            .to(torch.bfloat16))
    dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
    dx2 = bnfused.backward(da, x, m, i, g, b, relu=True, dgamma=dg2, dbeta=db2)
    torch.cuda.synchronize()
    torch.testing.assert_close(db, db2, rtol=2e-3, atol=2e-2)
    torch.testing.assert_close(dg, dg2, rtol=2e-3, atol=2e-2)
    err = (dx.float() - dx2.float()).abs().max() / dx2.float().abs().max()
    assert err < 2e-2, float(err)
    assert torch.equal(dx, bnfused.conv_im2col_dgrad_bn_backward(dy, w, x, m, i, g, b))
