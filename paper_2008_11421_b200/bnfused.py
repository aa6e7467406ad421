"""Thin torch-facing wrappers of libkrt's fused NHWC batch-norm kernels
(csrc/bn_kernels.cu).  Tensors are NCHW-logical with channels_last strides
(the NHWC storage the kernels read); everything is issued on torch's current
stream, which inside the executor is libkrt's compute stream."""
from __future__ import annotations

import torch

from . import _lib

EPS = 1e-5

# When a list, every launch appends (kind, algorithmic_bytes, start_event,
# end_event, algorithmic_flops) recorded on the launching stream — bench.py's
# live roofline.
PROFILE = None


class _timed:
    def __init__(self, kind, nbytes, flops=0.0):
        self.kind, self.nbytes, self.flops = kind, nbytes, flops

    def __enter__(self):
        if PROFILE is not None:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        return self

    def __exit__(self, *exc):
        if PROFILE is not None:
            self.e1.record()
            PROFILE.append((self.kind, self.nbytes, self.e0, self.e1, self.flops))
        return False


def _ptr(t):
    return None if t is None else t.data_ptr()


def _nhwc(t):
    if not t.is_contiguous(memory_format=torch.channels_last):
        t = t.contiguous(memory_format=torch.channels_last)
    return t


def _rows_c(t):
    n, c, h, w = t.shape
    return n * h * w, c


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _ws(c, device):
    return torch.empty(_lib.lib().krt_bn_workspace_bytes(c), dtype=torch.uint8, device=device)


def supported(c: int) -> bool:
    return c % 8 == 0 and c <= 2048 and 256 % (c // 8) == 0


def stats(c, mean, invstd):
    """Batch statistics of c (N,C,H,W channels_last bf16) into fp32 mean/invstd."""
    rows, C = _rows_c(c)
    ws = _ws(C, c.device)
    with _timed("bn_stats", rows * C * 2):
        _lib.check(_lib.lib().krt_bn_stats(_nhwc(c).data_ptr(), rows, C, EPS, mean.data_ptr(),
                                           invstd.data_ptr(), ws.data_ptr(), _stream()))


def stats_apply(c, mean, invstd, g, b, relu, res=None, out=None):
    """stats() then relu?(bn(c) [+ res]) in one cooperative kernel."""
    c = _nhwc(c)
    rows, C = _rows_c(c)
    y = out if out is not None else torch.empty_like(c, memory_format=torch.channels_last)
    ws = _ws(C, c.device)
    with _timed("bn_stats_apply", rows * C * 2 * (3 if res is None else 4)):
        _lib.check(_lib.lib().krt_bn_stats_apply(c.data_ptr(), rows, C, EPS, mean.data_ptr(), invstd.data_ptr(),
                                                 g.data_ptr(), b.data_ptr(),
                                                 _ptr(None if res is None else _nhwc(res)), int(relu),
                                                 y.data_ptr(), ws.data_ptr(), _stream()))
    return y


def apply(c, mean, invstd, g, b, relu, res=None, rstats=None, rg=None, rb=None, out=None):
    """relu?(bn(c) [+ res | + bn'(res)]) -> new bf16 channels_last tensor (or out)."""
    c = _nhwc(c)
    rows, C = _rows_c(c)
    y = out if out is not None else torch.empty_like(c, memory_format=torch.channels_last)
    rm, ri = (rstats if rstats is not None else (None, None))
    with _timed("bn_apply", rows * C * 2 * (2 if res is None else 3)):
        _lib.check(_lib.lib().krt_bn_apply(c.data_ptr(), mean.data_ptr(), invstd.data_ptr(), g.data_ptr(),
                                       b.data_ptr(), _ptr(None if res is None else _nhwc(res)), _ptr(rm),
                                           _ptr(ri), _ptr(rg), _ptr(rb), int(relu), y.data_ptr(), rows, C,
                                           _stream()))
    return y


def add_relu_bwd(dy, c, mean, invstd, g, b, res, rstats=None, rg=None, rb=None, dy2=None):
    """dz = (dy [+ dy2]) * mask; dy2 is summed in-kernel (never materialised)."""
    c, dy, res = _nhwc(c), _nhwc(dy), _nhwc(res)
    if dy2 is not None:
        dy2 = _nhwc(dy2)
    rows, C = _rows_c(c)
    dz = torch.empty_like(c, memory_format=torch.channels_last)
    rm, ri = (rstats if rstats is not None else (None, None))
    with _timed("bn_add_relu_bwd", rows * C * 2 * (4 if dy2 is None else 5)):
        _lib.check(_lib.lib().krt_bn_add_relu_bwd(dy.data_ptr(), _ptr(dy2), c.data_ptr(), mean.data_ptr(),
                                              invstd.data_ptr(), g.data_ptr(), b.data_ptr(),
                                              res.data_ptr(), _ptr(rm), _ptr(ri), _ptr(rg), _ptr(rb),
                                              dz.data_ptr(), rows, C, _stream()))
    return dz


def backward(dy, c, mean, invstd, g, b, relu, dgamma=None, dbeta=None, need_dx=True, addend=None):
    """BN backward (ReLU mask recomputed from c when relu); dgamma/dbeta fp32
    outputs; addend (a residual gradient) is summed into dx in the same pass."""
    c, dy = _nhwc(c), _nhwc(dy)
    if addend is not None:
        addend = _nhwc(addend)
    rows, C = _rows_c(c)
    dx = torch.empty_like(c, memory_format=torch.channels_last) if need_dx else None
    ws = _ws(C, c.device)
    nb = rows * C * 2 * ((5 if need_dx else 2) + (1 if addend is not None else 0))
    with _timed("bn_backward", nb):
        _lib.check(_lib.lib().krt_bn_backward(dy.data_ptr(), c.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                                              g.data_ptr(), b.data_ptr(), int(relu), _ptr(dx), _ptr(dgamma),
                                              _ptr(dbeta), rows, C, ws.data_ptr(), _ptr(addend), _stream()))
    return dx


def add_relu_backward(dy, c, mean, invstd, g, b, res, dgamma=None, dbeta=None, dy2=None):
    """add_relu_bwd (identity residual) + backward(relu=False) of the same BN in
    one cooperative kernel: returns (dz, dx)."""
    c, dy, res = _nhwc(c), _nhwc(dy), _nhwc(res)
    if dy2 is not None:
        dy2 = _nhwc(dy2)
    rows, C = _rows_c(c)
    dz = torch.empty_like(c, memory_format=torch.channels_last)
    dx = torch.empty_like(c, memory_format=torch.channels_last)
    ws = _ws(C, c.device)
    with _timed("bn_add_relu_backward", rows * C * 2 * (7 if dy2 is None else 8)):
        _lib.check(_lib.lib().krt_bn_add_relu_backward(dy.data_ptr(), _ptr(dy2), c.data_ptr(), mean.data_ptr(),
                                                       invstd.data_ptr(), g.data_ptr(), b.data_ptr(),
                                                       res.data_ptr(), dz.data_ptr(), dx.data_ptr(),
                                                       _ptr(dgamma), _ptr(dbeta), rows, C, ws.data_ptr(),
                                                       _stream()))
    return dz, dx


def relu_maxpool(c, mean, invstd, g, b, k=3, s=2, p=1):
    """maxpool_{k,s,p}(relu(bn(c))) without materialising relu(bn(c))."""
    c = _nhwc(c)
    n, C, h, w = c.shape
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    y = torch.empty((n, C, oh, ow), dtype=c.dtype, device=c.device, memory_format=torch.channels_last)
    with _timed("bn_relu_maxpool", c.numel() * 2 + y.numel() * 2):
        _lib.check(_lib.lib().krt_bn_relu_maxpool(c.data_ptr(), mean.data_ptr(), invstd.data_ptr(), g.data_ptr(),
                                                  b.data_ptr(), y.data_ptr(), n, h, w, C, k, s, p, _stream()))
    return y


def relu_maxpool_backward(dy, c, mean, invstd, g, b, k=3, s=2, p=1):
    """Gradient w.r.t. relu(bn(c)) of maxpool_{k,s,p}; argmaxes recomputed from c."""
    c, dy = _nhwc(c), _nhwc(dy)
    n, C, h, w = c.shape
    ws = torch.empty(_lib.lib().krt_bn_relu_maxpool_bwd_workspace(n, h, w, C, k, s, p), dtype=torch.uint8,
                     device=c.device)
    dx = torch.empty_like(c, memory_format=torch.channels_last)
    # bytes: c read for the argmax pass, argmax bytes written + read, dy read, dx written
    with _timed("bn_relu_maxpool_bwd", c.numel() * 2 * 2 + ws.numel() * 2 + dy.numel() * 2):
        _lib.check(_lib.lib().krt_bn_relu_maxpool_bwd(dy.data_ptr(), c.data_ptr(), mean.data_ptr(),
                                                      invstd.data_ptr(), g.data_ptr(), b.data_ptr(), dx.data_ptr(),
                                                      ws.data_ptr(), n, h, w, C, k, s, p, _stream()))
    return dx


def conv1x1_supported(cin, cout, pre=False):
    return (cin in (16, 32) or cin % 64 == 0) and (cout in (16, 32, 64, 128) or cout % 256 == 0) and (not pre or cin <= 1024)


def conv1x1(x, w, out=None, pre=None, stats=None, res=None):
    """Stride-1 1x1 convolution on the sm_100a tcgen05 GEMM (csrc/gemm_sm100.cu).

    x: (N, Cin, H, W) channels_last bf16; w: (Cout, Cin, 1, 1) bf16.
    pre=(mean, invstd, gamma, beta): convolve relu(bn(x)) instead of x, without
    writing relu(bn(x)).  stats=(mean, invstd): fp32 outputs, the batch
    statistics of the (bf16) result, reduced in the GEMM epilogue.
    res: (N, Cout, H, W) channels_last bf16 added to the result in the
    epilogue (fp32 sum, one rounding).
    """
    import ctypes as C
    x = _nhwc(x)
    n, cin, h, ww = x.shape
    cout = w.shape[0]
    wm = w.reshape(cout, cin)
    if not wm.is_contiguous():
        wm = wm.contiguous()
    y = out if out is not None else torch.empty((n, cout, h, ww), dtype=x.dtype, device=x.device,
                                                memory_format=torch.channels_last)
    M = n * h * ww
    part = None
    rows = C.c_int(0)
    if stats is not None:
        part = torch.empty(_lib.lib().krt_conv1x1_partials_bytes(cout) // 4, dtype=torch.float32, device=x.device)
    pm, pi, pg, pb = pre if pre is not None else (None, None, None, None)
    # bytes: A read, C written (the statistics pass this replaces would re-read C)
    if res is not None:
        res = _nhwc(res)
        assert res.shape == y.shape and res.dtype == y.dtype
    with _timed("conv1x1_bn", M * (cin + cout * (1 if res is None else 2)) * 2, 2.0 * M * cin * cout):
        if res is None:
            _lib.check(_lib.lib().krt_conv1x1_bn(x.data_ptr(), wm.data_ptr(), y.data_ptr(), M, cout, cin, _ptr(pm),
                                                 _ptr(pi), _ptr(pg), _ptr(pb), _ptr(part), C.byref(rows), _stream()))
        else:
            _lib.check(_lib.lib().krt_conv1x1_bn_res(x.data_ptr(), wm.data_ptr(), y.data_ptr(), M, cout, cin,
                                                     _ptr(pm), _ptr(pi), _ptr(pg), _ptr(pb), res.data_ptr(),
                                                     _ptr(part), C.byref(rows), _stream()))
        if stats is not None:
            _lib.check(_lib.lib().krt_bn_partials_finalize(part.data_ptr(), rows.value, cout, M, EPS,
                                                           stats[0].data_ptr(), stats[1].data_ptr(), _stream()))
    return y


def stem_wgrad(dc, x, dw):
    """Weight gradient of the ResNet stem convolution (7x7 / stride 2 / pad 3,
    3 -> 64 channels) on tcgen05 (krt_stem_wgrad): fp32 into dw (64, 7, 7, 3)
    OHWI contiguous.  dc: (N, 64, Ho, Wo) channels_last bf16 output gradient;
    x: (N, 3, H, W) channels_last bf16 input."""
    x, dc = _nhwc(x), _nhwc(dc)
    n, cin, h, ww = x.shape
    assert cin == 3 and dc.shape[1] == 64 and dw.dtype == torch.float32 and dw.is_contiguous()
    assert dw.numel() == 64 * 49 * 3
    x4 = torch.empty((n, 4, h, ww), dtype=x.dtype, device=x.device, memory_format=torch.channels_last)
    with _timed("pad_rgb4", n * h * ww * (6 + 8)):
        _lib.check(_lib.lib().krt_pad_rgb4(x.data_ptr(), x4.data_ptr(), n * h * ww, _stream()))
    L = _lib.lib()
    ws = torch.empty(L.krt_stem_wgrad_workspace(), dtype=torch.uint8, device=x.device)
    P = dc.numel() // 64
    with _timed("conv_wgrad", x4.numel() * 2 + dc.numel() * 2 + dw.numel() * 4, 2.0 * P * 64 * 49 * 3):
        _lib.check(L.krt_stem_wgrad(x4.data_ptr(), dc.data_ptr(), dw.data_ptr(), n, h, ww, ws.data_ptr(), ws.numel(),
                                    _stream()))
    return dw


def conv_gather(x, w, stride, pad, out=None, stats=None):
    """Implicit-GEMM convolution on tcgen05 (the ResNet stem, 64 output
    channels): im2col rows gathered into shared memory, never written.
    x: (N, Cin, H, W) channels_last bf16; w: (64, Cin, k, k) bf16.
    stats=(mean, invstd): the BN statistics of the result from the epilogue."""
    import ctypes as C
    x = _nhwc(x)
    n, cin, h, ww = x.shape
    cout, _, k, _ = w.shape
    if cin == 3:
        # RGB -> 4 channels (zero), so the gather moves one 8-byte pixel per load
        x4 = torch.empty((n, 4, h, ww), dtype=x.dtype, device=x.device, memory_format=torch.channels_last)
        with _timed("pad_rgb4", n * h * ww * (6 + 8)):
            _lib.check(_lib.lib().krt_pad_rgb4(x.data_ptr(), x4.data_ptr(), n * h * ww, _stream()))
        w4 = torch.zeros((cout, 4, k, k), dtype=w.dtype, device=w.device)
        w4[:, :3] = w
        x, w, cin = x4, w4, 4
    ho, wo = (h + 2 * pad - k) // stride + 1, (ww + 2 * pad - k) // stride + 1
    kk = k * k * cin
    K = (kk + 31) // 32 * 32
    wk = torch.zeros((cout, K), dtype=w.dtype, device=w.device)
    wk[:, :kk] = w.permute(0, 2, 3, 1).reshape(cout, kk)      # k = (kh*k + kw)*cin + c
    y = out if out is not None else torch.empty((n, cout, ho, wo), dtype=x.dtype, device=x.device,
                                                memory_format=torch.channels_last)
    M = n * ho * wo
    part = None
    rows = C.c_int(0)
    if stats is not None:
        part = torch.empty(_lib.lib().krt_conv1x1_partials_bytes(cout) // 4, dtype=torch.float32, device=x.device)
    with _timed("conv_gather_bn", n * h * ww * cin * 2 + M * cout * 2, 2.0 * M * kk * cout):
        _lib.check(_lib.lib().krt_conv_gather_bn(x.data_ptr(), wk.data_ptr(), y.data_ptr(), n, h, ww, cin, ho, wo,
                                                 k, stride, pad, cout, K, _ptr(part), C.byref(rows), _stream()))
        if stats is not None:
            _lib.check(_lib.lib().krt_bn_partials_finalize(part.data_ptr(), rows.value, cout, M, EPS,
                                                           stats[0].data_ptr(), stats[1].data_ptr(), _stream()))
    return y


def conv1x1_dgrad_bn_backward(dy, w, x, mean, invstd, g, b, dgamma=None, dbeta=None, relu=True, addend=None):
    """d(input of relu(bn(x)))-chain through a stride-1 1x1 convolution:
    da = dy . W (tcgen05 GEMM, W transposed to K-major) with the BN backward
    reduce of (da, x) in its epilogue, then the BN backward elementwise pass.
    dy: (N, Cout, H, W) grad of the conv output; w: (Cout, Cin, 1, 1); x: the
    BN input (N, Cin, H, W).  Returns dx = d/dx of conv(relu(bn(x))), plus
    addend (a gradient of x from another path, e.g. the identity shortcut)."""
    import ctypes as C
    dy, x = _nhwc(dy), _nhwc(x)
    n, cout, h, ww = dy.shape
    cin = w.shape[1]
    wt = w.reshape(cout, cin).t().contiguous()          # [Cin, Cout]: the K-major B operand
    M = n * h * ww
    da = torch.empty((n, cin, h, ww), dtype=dy.dtype, device=dy.device, memory_format=torch.channels_last)
    part = torch.empty(_lib.lib().krt_conv1x1_partials_bytes(cin) // 4, dtype=torch.float32, device=dy.device)
    coef = torch.empty(3 * cin, dtype=torch.float32, device=dy.device)
    rows = C.c_int(0)
    with _timed("conv1x1_dgrad_bn", M * (cout + 2 * cin) * 2, 2.0 * M * cin * cout):
        _lib.check(_lib.lib().krt_conv1x1_bn_dgrad(dy.data_ptr(), wt.data_ptr(), da.data_ptr(), M, cin, cout,
                                                   x.data_ptr(), mean.data_ptr(), invstd.data_ptr(), g.data_ptr(),
                                                   b.data_ptr(), part.data_ptr(), C.byref(rows), _stream()))
        _lib.check(_lib.lib().krt_bn_partials_bwd_finalize(part.data_ptr(), rows.value, cin, M, mean.data_ptr(),
                                                           invstd.data_ptr(), g.data_ptr(), _ptr(dgamma),
                                                           _ptr(dbeta), coef.data_ptr(), _stream()))
    dx = torch.empty_like(x, memory_format=torch.channels_last)
    with _timed("bn_backward_elemt", M * cin * 2 * (3 if addend is None else 4)):
        _lib.check(_lib.lib().krt_bn_backward_elemt(da.data_ptr(), x.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                                                    g.data_ptr(), b.data_ptr(), coef.data_ptr(),
                                                    None if addend is None else _nhwc(addend).data_ptr(),
                                                    int(relu), dx.data_ptr(), M, cin, _stream()))
    return dx


def conv1x1_dgrad_supported(cout, cin):
    """conv1x1_dgrad_bn_backward for a (Cout, Cin) 1x1 weight: the GEMM
    reduces over K = Cout into N = Cin columns (BN-backward epilogue: N >= 64)."""
    return conv1x1_supported(cout, cin) and cin >= 64 and supported(cin)


def conv_wgrad_supported(cout, cin, k, stride, pre=False):
    """krt_conv_wgrad's shape rules (csrc/wgrad_sm100.cu)."""
    return cout % 128 == 0 and cin % 64 == 0 and k in (1, 3) and stride in (1, 2) and (not pre or cin <= 1024)


def conv_wgrad(dy, x, dw, k, stride, pad, pre=None):
    """Weight gradient of conv(f(x), w) on the tcgen05 wgrad GEMM, written in
    fp32 into dw (Cout, k, k, Cin) OHWI contiguous (the executor's gradient
    view).  dy: (N, Cout, Ho, Wo) channels_last bf16 gradient of the conv
    output; x: (N, Cin, H, W) channels_last bf16; pre=(mean, invstd, gamma,
    beta): f = relu(bn(.)) applied in shared memory (relu(bn(x)) is never
    materialised), else f = identity."""
    import ctypes as C
    dy, x = _nhwc(dy), _nhwc(x)
    n, cout, ho, wo = dy.shape
    _, cin, h, w = x.shape
    assert dw.dtype == torch.float32 and dw.is_contiguous() and dw.numel() == cout * k * k * cin
    L = _lib.lib()
    ws = torch.empty(L.krt_conv_wgrad_workspace_bytes(n, ho, wo, cout, cin, k), dtype=torch.uint8, device=x.device)
    pm, pi, pg, pb = pre if pre is not None else (None, None, None, None)
    P = n * ho * wo
    with _timed("conv_wgrad", P * cout * 2 + n * h * w * cin * 2 + dw.numel() * 4, 2.0 * P * cout * k * k * cin):
        _lib.check(L.krt_conv_wgrad(dy.data_ptr(), x.data_ptr(), dw.data_ptr(), n, h, w, cin, ho, wo, cout, k, stride,
                                    pad, _ptr(pm), _ptr(pi), _ptr(pg), _ptr(pb), ws.data_ptr(), ws.numel(),
                                    _stream()))
    return dw


def conv_im2col_supported(cin, cout, pre=False, dgrad=False):
    """krt_conv_im2col_bn's shape rules (csrc/gemm_sm100.cu) for any stride;
    3x3 / stride 1 also takes 16 -> 16 and 32 -> 32 channels (halo kernel,
    conv3x3_halo_supported)."""
    if cin % 64 or (pre and cin > 1024):
        return False
    return cout in (64, 128) or cout % (128 if dgrad else 256) == 0


def conv3x3_halo_supported(h, w, cin, cout, pre=False):
    """krt_conv_im2col_bn runs this 3x3 / stride-1 / pad-1 shape on the halo kernel."""
    return bool(_lib.lib().krt_conv3x3_halo_supported(h, w, cin, cout, int(pre)))


def wgrad1x1_narrow_supported(cin, cout):
    return bool(_lib.lib().krt_wgrad1x1_narrow_supported(cin, cout))


def wgrad1x1_narrow(dy, x, dw, pre=None):
    """Weight gradient of a 1x1 / stride-1 convolution with few channels on
    tcgen05 (krt_wgrad1x1_narrow), fp32 into dw (Cout, 1, 1, Cin) contiguous.
    pre=(mean, invstd, gamma, beta): the forward convolved relu(bn(x))."""
    dy, x = _nhwc(dy), _nhwc(x)
    n, ci, h, w = x.shape
    co = dy.shape[1]
    assert dw.dtype == torch.float32 and dw.is_contiguous() and dw.numel() == ci * co
    L = _lib.lib()
    ws = torch.empty(L.krt_wgrad1x1_narrow_workspace(ci, co), dtype=torch.uint8, device=x.device)
    pm, pi, pg, pb = pre if pre is not None else (None, None, None, None)
    M = n * h * w
    with _timed("conv_wgrad", (x.numel() + dy.numel()) * 2 + dw.numel() * 4, 2.0 * M * ci * co):
        _lib.check(L.krt_wgrad1x1_narrow(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), M, ci, co, _ptr(pm), _ptr(pi),
                                          _ptr(pg), _ptr(pb), ws.data_ptr(), ws.numel(), _stream()))
    return dw


def wgrad3x3_narrow_supported(h, w, c):
    return bool(_lib.lib().krt_wgrad3x3_narrow_supported(h, w, c))


def wgrad3x3_narrow(dy, x, dw, pre=None):
    """Weight gradient of a 3x3 / stride-1 / pad-1 convolution with C = cin =
    cout in {16, 32, 64} (halo windows on tcgen05), written in fp32 into dw
    (C, 3, 3, C) OHWI contiguous.  pre=(mean, invstd, gamma, beta): the
    forward convolved relu(bn(x)) (never materialised here)."""
    dy, x = _nhwc(dy), _nhwc(x)
    n, c, h, w = x.shape
    assert dw.dtype == torch.float32 and dw.is_contiguous() and dw.numel() == c * 9 * c
    L = _lib.lib()
    ws = torch.empty(L.krt_wgrad3x3_narrow_workspace(c), dtype=torch.uint8, device=x.device)
    pm, pi, pg, pb = pre if pre is not None else (None, None, None, None)
    with _timed("conv_wgrad", 2 * x.numel() * 2 + dw.numel() * 4, 2.0 * n * h * w * 9 * c * c):
        _lib.check(L.krt_wgrad3x3_narrow(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), n, h, w, c, _ptr(pm), _ptr(pi),
                                          _ptr(pg), _ptr(pb), ws.data_ptr(), ws.numel(), _stream()))
    return dw


def conv3x3_dgrad(dy, w, out=None):
    """Data gradient of a 3x3 / stride-1 / pad-1 convolution (w: (Cout, 3, 3,
    Cin) OHWI): the same convolution of dy with the flipped, transposed
    weights, on the halo kernel when conv3x3_halo_supported."""
    wt = w.flip(1, 2).permute(3, 1, 2, 0).contiguous()
    return conv_im2col(dy, wt, 1, 1, out=out)


def conv_im2col(x, w, stride, pad, out=None, pre=None, stats=None):
    """k x k convolution on the tcgen05 implicit GEMM (im2col TMA tiles).
    x: (N, Cin, H, W) channels_last bf16; w: (Cout, k, k, Cin) bf16 OHWI
    contiguous (the executor's weight view).  pre=(mean, invstd, gamma, beta):
    convolve relu(bn(x)) (never written; the padding stays zero); stats=(mean,
    invstd): batch statistics of the bf16 result from the epilogue."""
    import ctypes as C
    x = _nhwc(x)
    n, cin, h, ww = x.shape
    cout, k = w.shape[0], w.shape[1]
    assert w.shape == (cout, k, k, cin) and w.is_contiguous()
    ho, wo = (h + 2 * pad - k) // stride + 1, (ww + 2 * pad - k) // stride + 1
    y = out if out is not None else torch.empty((n, cout, ho, wo), dtype=x.dtype, device=x.device,
                                                memory_format=torch.channels_last)
    M = n * ho * wo
    part = None
    rows = C.c_int(0)
    if stats is not None:
        part = torch.empty(_lib.lib().krt_conv1x1_partials_bytes(cout) // 4, dtype=torch.float32, device=x.device)
    pm, pi, pg, pb = pre if pre is not None else (None, None, None, None)
    with _timed("conv_im2col_bn", n * h * ww * cin * 2 + M * cout * 2, 2.0 * M * k * k * cin * cout):
        _lib.check(_lib.lib().krt_conv_im2col_bn(x.data_ptr(), w.data_ptr(), y.data_ptr(), n, h, ww, cin, ho, wo, k,
                                                 stride, pad, cout, _ptr(pm), _ptr(pi), _ptr(pg), _ptr(pb),
                                                 _ptr(part), C.byref(rows), None, None, None, None, None,
                                                 _stream()))
        if stats is not None:
            _lib.check(_lib.lib().krt_bn_partials_finalize(part.data_ptr(), rows.value, cout, M, EPS,
                                                           stats[0].data_ptr(), stats[1].data_ptr(), _stream()))
    return y


def conv_im2col_dgrad_bn_backward(dy, w, x, mean, invstd, g, b, dgamma=None, dbeta=None, relu=True, addend=None):
    """Gradient w.r.t. x of conv_kxk(relu(bn(x))) (stride 1, 'same' padding):
    da = conv(dy, W flipped and transposed) on the im2col GEMM with the BN
    backward reduce of (da, x) in its epilogue, then the BN backward
    elementwise pass.  dy: (N, Cout, H, W); w: (Cout, k, k, Cin) OHWI."""
    import ctypes as C
    dy, x = _nhwc(dy), _nhwc(x)
    n, cout, h, ww = dy.shape
    k, cin = w.shape[1], w.shape[3]
    pad = k // 2
    wt = w.flip(1, 2).permute(3, 1, 2, 0).contiguous()      # [Cin][k][k][Cout]
    M = n * h * ww
    da = torch.empty((n, cin, h, ww), dtype=dy.dtype, device=dy.device, memory_format=torch.channels_last)
    part = torch.empty(_lib.lib().krt_conv1x1_partials_bytes(cin) // 4, dtype=torch.float32, device=dy.device)
    coef = torch.empty(3 * cin, dtype=torch.float32, device=dy.device)
    rows = C.c_int(0)
    with _timed("conv_im2col_dgrad_bn", M * (cout + 2 * cin) * 2, 2.0 * M * k * k * cin * cout):
        _lib.check(_lib.lib().krt_conv_im2col_bn(dy.data_ptr(), wt.data_ptr(), da.data_ptr(), n, h, ww, cout, h, ww,
                                                 k, 1, pad, cin, None, None, None, None, part.data_ptr(),
                                                 C.byref(rows), x.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                                                 g.data_ptr(), b.data_ptr(), _stream()))
        _lib.check(_lib.lib().krt_bn_partials_bwd_finalize(part.data_ptr(), rows.value, cin, M, mean.data_ptr(),
                                                           invstd.data_ptr(), g.data_ptr(), _ptr(dgamma),
                                                           _ptr(dbeta), coef.data_ptr(), _stream()))
    dx = torch.empty_like(x, memory_format=torch.channels_last)
    with _timed("bn_backward_elemt", M * cin * 2 * (3 if addend is None else 4)):
        _lib.check(_lib.lib().krt_bn_backward_elemt(da.data_ptr(), x.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                                                    g.data_ptr(), b.data_ptr(), coef.data_ptr(),
                                                    None if addend is None else _nhwc(addend).data_ptr(),
                                                    int(relu), dx.data_ptr(), M, cin, _stream()))
    return dx
