"""3x3 / stride-1 / pad-1 convolution on the halo-window kernel
(csrc/halo_sm100.cu, reached through krt_conv_im2col_bn) vs torch fp32:
image sizes with and without partial 128-row sub-tiles and junk columns
(every tap crosses the window's swizzle-row phase), single images and
batches, 64 and 128 output channels on 64-channel blocks, the narrow 16 / 32
channel convolutions of ResNet-1001 (32 / 64-byte window rows), images wider
than one 256-pixel TMA box or than shared memory holds (column segments whose
windows take their halo columns from the neighbouring segment), more input
than output channels, with
the relu(bn(.)) prologue (the zero padding must stay zero: the reference
convolves the bn_apply output) and the statistics epilogue (junk rows
excluded).  Tolerances as tests/test_conv_im2col_gpu.py: bf16 output rounding
plus fp32 accumulation order; fused statistics vs the stats kernel on the
stored output at rtol 1e-4; repeat calls bitwise equal."""
import pytest
import torch
import torch.nn.functional as F

from paper_2008_11421_b200 import _lib, bnfused

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


SHAPES = [(1, 64, 64, 1, 1), (2, 64, 64, 5, 9), (3, 64, 64, 56, 56), (2, 128, 128, 28, 28), (5, 64, 128, 14, 14),
          (4, 128, 64, 7, 7), (2, 256, 128, 13, 17), (1, 256, 64, 30, 6), (2, 64, 128, 33, 50),
          (2, 16, 16, 17, 30), (1, 32, 32, 9, 13), (2, 16, 16, 64, 64), (2, 16, 16, 12, 300),
          (1, 32, 32, 21, 520), (1, 64, 64, 11, 600), (1, 16, 16, 130, 2048)]


@pytest.mark.parametrize("n,cin,cout,h,w", SHAPES)
@pytest.mark.parametrize("pre", [False, True])
@pytest.mark.parametrize("stats", [False, True])
def test_conv_halo_matches_torch(n, cin, cout, h, w, pre, stats):
    assert _lib.lib().krt_conv3x3_halo_supported(h, w, cin, cout, int(pre)) == 1
    x = cl(rand((n, cin, h, w), 1, 2.0))
    wt = rand((cout, 3, 3, cin), 2, (cin * 9) ** -0.5).contiguous()
    if pre:
        g, b = bn_params(cin, 3)
        m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
        bnfused.stats(x, m, i)
        a, pre_t = bnfused.apply(x, m, i, g, b, relu=True), (m, i, g, b)
    else:
        a, pre_t = x, None
    st = (torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda")) if stats else None
    y = bnfused.conv_im2col(x, wt, 1, 1, pre=pre_t, stats=st)
    torch.cuda.synchronize()
    ref = F.conv2d(a.float(), wt.permute(0, 3, 1, 2).float(), padding=1)
    assert y.shape == ref.shape
    err = (y.float() - ref).abs().max() / ref.abs().max().clamp_min(1e-6)
    assert err < 1e-2, float(err)
    if stats:
        rm, ri = torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda")
        bnfused.stats(y, rm, ri)
        torch.testing.assert_close(st[0], rm, rtol=1e-4, atol=1e-5)
        torch.testing.assert_close(st[1], ri, rtol=1e-4, atol=1e-5)
    assert torch.equal(y, bnfused.conv_im2col(x, wt, 1, 1, pre=pre_t, stats=st))   # deterministic


def test_halo_declines_other_channel_counts():
    # 256 output channels (and 48 input channels) stay on the im2col GEMM path,
    # which krt_conv_im2col_bn then takes (still correct)
    assert _lib.lib().krt_conv3x3_halo_supported(8, 8, 64, 256, 0) == 0
    assert _lib.lib().krt_conv3x3_halo_supported(8, 8, 48, 48, 0) == 0
    x = cl(rand((1, 64, 8, 8), 4))
    wt = rand((256, 3, 3, 64), 5, (64 * 9) ** -0.5).contiguous()
    y = bnfused.conv_im2col(x, wt, 1, 1)
    ref = F.conv2d(x.float(), wt.permute(0, 3, 1, 2).float(), padding=1)
    assert (y.float() - ref).abs().max() / ref.abs().max() < 1e-2
