"""Weight gradient of 3x3 / stride-1 / pad-1 convolutions with few channels
(C = cin = cout in {16, 32, 64}: ResNet-1001's widths) on the halo-window
tcgen05 kernel (csrc/wgrad_halo_sm100.cu, krt_wgrad3x3_narrow) vs torch fp32
autograd on the same bf16 operands: images smaller than one tile, partial
tiles, column segments (widths beyond one 256-pixel TMA box), with and
without the relu(bn(.)) prologue (padding stays zero).  Tolerance: fp32
accumulation over many pixels in a different order, 2e-3 of the max |dW|;
repeat calls bitwise equal (fixed-order partial sums)."""
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


@pytest.mark.parametrize("n,c,h,w", [(2, 16, 5, 7), (1, 16, 33, 40), (2, 32, 17, 29), (1, 64, 12, 20),
                                     (2, 16, 9, 300), (1, 32, 7, 600), (1, 64, 5, 513), (2, 16, 64, 64)])
@pytest.mark.parametrize("pre", [False, True])
def test_wgrad_narrow_matches_torch(n, c, h, w, pre):
    assert bnfused.wgrad3x3_narrow_supported(h, w, c)
    x = cl(rand((n, c, h, w), 1, 2.0))
    dy = cl(rand((n, c, h, w), 2))
    if pre:
        g = (1 + 0.2 * torch.randn(c, device="cuda")).to(torch.bfloat16)
        b = (0.1 * torch.randn(c, device="cuda")).to(torch.bfloat16)
        m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
        bnfused.stats(x, m, i)
        a, pre_t = bnfused.apply(x, m, i, g, b, relu=True), (m, i, g, b)
    else:
        a, pre_t = x, None
    dw = torch.empty(c, 3, 3, c, device="cuda")
    bnfused.wgrad3x3_narrow(dy, x, dw, pre=pre_t)
    wr = torch.zeros(c, c, 3, 3, device="cuda", requires_grad=True)
    F.conv2d(a.float(), wr, padding=1).backward(dy.float())
    ref = wr.grad.permute(0, 2, 3, 1)   # OHWI
    err = float((dw - ref).abs().max() / ref.abs().max())
    assert err < 2e-3, err
    dw2 = torch.empty_like(dw)
    bnfused.wgrad3x3_narrow(dy, x, dw2, pre=pre_t)
    assert torch.equal(dw, dw2)


@pytest.mark.parametrize("n,ci,co,h,w", [(2, 64, 16, 9, 13), (1, 16, 64, 33, 20), (2, 128, 32, 17, 9),
                                         (1, 32, 128, 8, 70), (1, 256, 64, 12, 11), (2, 64, 256, 7, 9),
                                         (2, 64, 64, 16, 16)])
@pytest.mark.parametrize("pre", [False, True])
def test_wgrad1x1_narrow_matches_torch(n, ci, co, h, w, pre):
    assert bnfused.wgrad1x1_narrow_supported(ci, co)
    x = cl(rand((n, ci, h, w), 3, 2.0))
    dy = cl(rand((n, co, h, w), 4))
    if pre:
        g = (1 + 0.2 * torch.randn(ci, device="cuda")).to(torch.bfloat16)
        b = (0.1 * torch.randn(ci, device="cuda")).to(torch.bfloat16)
        m, i = torch.empty(ci, device="cuda"), torch.empty(ci, device="cuda")
        bnfused.stats(x, m, i)
        a, pre_t = bnfused.apply(x, m, i, g, b, relu=True), (m, i, g, b)
    else:
        a, pre_t = x, None
    dw = torch.empty(co, 1, 1, ci, device="cuda")
    bnfused.wgrad1x1_narrow(dy, x, dw, pre=pre_t)
    ref = torch.einsum("nchw,nkhw->kc", a.float(), dy.float()).view(co, 1, 1, ci)
    err = float((dw - ref).abs().max() / ref.abs().max())
    assert err < 2e-3, err
    dw2 = torch.empty_like(dw)
    bnfused.wgrad1x1_narrow(dy, x, dw2, pre=pre_t)
    assert torch.equal(dw, dw2)


@pytest.mark.parametrize("n,h", [(2, 224), (3, 30), (1, 8), (5, 64)])
def test_stem_wgrad_matches_torch(n, h):
    x = cl(rand((n, 3, h, h), 8, 2.0))
    ho = (h + 6 - 7) // 2 + 1
    dc = cl(rand((n, 64, ho, ho), 9))
    dw = torch.empty(64, 7, 7, 3, device="cuda")
    bnfused.stem_wgrad(dc, x, dw)
    wr = torch.zeros(64, 3, 7, 7, device="cuda", requires_grad=True)
    F.conv2d(x.float(), wr, stride=2, padding=3).backward(dc.float())
    ref = wr.grad.permute(0, 2, 3, 1)
    err = float((dw - ref).abs().max() / ref.abs().max())
    assert err < 2e-3, err
    dw2 = torch.empty_like(dw)
    bnfused.stem_wgrad(dc, x, dw2)
    assert torch.equal(dw, dw2)
