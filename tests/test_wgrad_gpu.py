"""tcgen05 weight-gradient GEMM (csrc/wgrad_sm100.cu) vs torch fp32: the
weight gradient of conv(f(x)) for 1x1 and 3x3 kernels, stride 1 and 2, with
and without the fused relu(bn(.)) prologue (f(x) reproduced by the bn_apply
kernel, whose bf16 output the prologue must match bitwise).  Both sides sum
exact bf16 x bf16 products in fp32; only the summation order differs, so the
tolerance is 2e-3 of the largest |dW| (the pixel reduction has up to 1e5
terms).  The split-K reduction runs in a fixed order: bitwise repeatable."""
import pytest
import torch

from paper_2008_11421_b200 import bnfused

pytestmark = pytest.mark.gpu


def rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(torch.bfloat16)


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


CASES = [  # n, cin, h, cout, k, stride
    (2, 64, 8, 128, 1, 1), (3, 256, 14, 512, 1, 1), (2, 128, 7, 256, 1, 1), (1, 512, 5, 2048, 1, 1),
    (2, 64, 8, 128, 3, 1), (2, 128, 14, 128, 3, 1), (1, 256, 7, 256, 3, 1), (2, 512, 7, 512, 3, 1),
    (2, 256, 14, 512, 1, 2), (2, 128, 14, 128, 3, 2), (1, 64, 15, 128, 3, 2),
    (16, 64, 56, 256, 1, 1), (8, 128, 28, 128, 3, 1),    # many k-blocks per split
]


@pytest.mark.parametrize("n,cin,h,cout,k,stride", CASES)
@pytest.mark.parametrize("pre", [False, True])
def test_conv_wgrad_matches_torch(n, cin, h, cout, k, stride, pre):
    pad = k // 2
    x = cl(rand((n, cin, h, h), 1, 2.0))
    ho = (h + 2 * pad - k) // stride + 1
    dy = cl(rand((n, cout, ho, ho), 2, 0.5))
    if pre:
        g = (1 + 0.2 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
        b = (0.1 * torch.randn(cin, device="cuda")).to(torch.bfloat16)
        m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
        bnfused.stats(x, m, i)
        a = bnfused.apply(x, m, i, g, b, relu=True)
        pre_t = (m, i, g, b)
    else:
        a, pre_t = x, None
    dw = torch.empty(cout, k, k, cin, device="cuda")
    bnfused.conv_wgrad(dy, x, dw, k, stride, pad, pre=pre_t)
    torch.cuda.synchronize()
    ref = torch.nn.grad.conv2d_weight(a.float(), (cout, cin, k, k), dy.float(), stride=stride, padding=pad)
    ref = ref.permute(0, 2, 3, 1)
    err = (dw - ref).abs().max() / ref.abs().max()
    assert err < 2e-3, float(err)
    dw2 = torch.empty_like(dw)
    bnfused.conv_wgrad(dy, x, dw2, k, stride, pad, pre=pre_t)
    assert torch.equal(dw, dw2)
