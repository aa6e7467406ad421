"""Executor units: the layers of the model IR the planner partitions.

Every unit saves its input first (see executor.Unit), then whatever its own
backward needs.  Parameters live in libkrt's device weight region; gradients
are written in fp32 into libkrt's gradient region, from where the runtime
moves them (grad_out / exchange, distsim.py:205-236) or updates them in place.

Model-IR mapping (model_ir.py:8-25 format, measured overrides per
cost_model.py:203-213): ``mem_fwd`` = the bytes the unit really keeps in its
arena slot, ``mem_wt=0`` because weights are HBM-resident outside the swap
unit, ``mem_grad`` = its fp32 gradient bytes.
"""
from __future__ import annotations

import math
import os
from typing import Optional

import torch
import torch.nn.functional as F

from . import bnfused, lnfused
from .executor import SavedSpec, Unit, _align


class FCUnit(Unit):
    """FullyConnected layer without bias (zoo.fc_chain_model, zoo.py:57-63):
    y = x W^T, W: [out, in].  Saved: x."""

    name = "fc"

    def __init__(self, fin: int, fout: int, act_dtype=torch.float32):
        self.fin, self.fout, self.dt = fin, fout, act_dtype

    def param_specs(self):
        return [(self.fout, self.fin)]

    def saved_specs(self, batch):
        return [SavedSpec((batch, self.fin), self.dt)]

    def init_params(self, gen):
        bound = 1.0 / math.sqrt(self.fin)
        return [torch.empty(self.fout, self.fin).uniform_(-bound, bound, generator=gen)]

    def forward(self, x, params, saved):
        (w,) = params
        if saved is not None:
            saved[0].copy_(x)
        return torch.mm(x, w.t())

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        (w,) = params
        x = saved[0]
        if dy.dtype == torch.float32 and x.dtype == torch.float32:
            torch.mm(dy.t(), x, out=grads[0])
        else:
            grads[0].copy_(torch.mm(dy.t(), x, out_dtype=torch.float32))
        return torch.mm(dy, w)

    def fwd_flops(self, batch):
        return 2.0 * batch * self.fin * self.fout

    def ir_line(self, lid, batch, analytic=False):
        if analytic:
            return f"{lid} FullyConnected X={self.fin} Y={self.fout} elem=4"
        return (f"{lid} FullyConnected X={self.fin} Y={self.fout} elem=4 "
                f"mem_fwd={self.saved_bytes(batch)} mem_wt=0 mem_grad={4 * self.fin * self.fout}")


def mse_zero_loss(y, target=None):
    """MSE against zero targets: mean(y^2), dy = 2y/numel."""
    loss = (y.float() * y.float()).mean()
    dy = y * (2.0 / y.numel())
    return loss, dy


def model_text(units, batch, analytic=False) -> str:
    """Model IR text for the reference planner (model_ir.py:281-330)."""
    lines = ["version = 1", f"batch_size = {batch}", "", "[layers]"]
    for i, u in enumerate(units, start=1):
        lines.append(u.ir_line(i, batch, analytic) if analytic else u.ir_line(i, batch))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# ResNet (bottleneck, [3, 24, 36, 3] = ResNet-200; stride on the 3x3 conv)
# Activations bf16 NHWC (channels_last); BN statistics fp32.  Each conv's
# output is saved once; BN-apply/ReLU are recomputed inside backward from the
# saved conv output and the BN statistics (elementwise, HBM-bound).
# ---------------------------------------------------------------------------
_aten = torch.ops.aten
BN_EPS = 1e-5
# bottleneck 1x1 convolutions on the own tcgen05 GEMM (csrc/gemm_sm100.cu) with
# the BN work fused in; KRT_TC_CONV1X1=0 selects cuDNN + separate BN kernels
TC_CONV1X1 = os.environ.get("KRT_TC_CONV1X1", "1") != "0"
# GPT attention on cuDNN's sm100 fused kernels (KRT_ATTN_CUDNN=0: aten flash)
ATTN_CUDNN = os.environ.get("KRT_ATTN_CUDNN", "1") != "0"
# linear layers' bias gradient in the weight-gradient GEMM's epilogue
# (cuBLASLt BGRADB), opt-in with KRT_LINEAR_BGRAD=1: measured slower than
# GEMM + a separate column sum on B200 (Megatron L36: GEMMs 2841 -> 2959
# ms/step, 33.8 -> 33.0 samples/s; profiles/round2_s4/README.md)
LINEAR_BGRAD = os.environ.get("KRT_LINEAR_BGRAD", "0") == "1"
# head dims above cuDNN's backward limit (128): aten's flash backward by
# default; KRT_ATTN_UNFUSED_BW=1 selects the unfused cuBLAS + own-pass form,
# measured 2.1x slower at Turing-NLG's shape (1576 vs 766 ms/step: its fp32
# s x s score / score-gradient matrices cost ~30 MB of HBM traffic per
# (sequence, head) pair at seq 1024; profiles/round2_s4/README.md)
ATTN_UNFUSED_BW = os.environ.get("KRT_ATTN_UNFUSED_BW", "0") == "1"
# the pre-activation unit's 1x1 dgrads on the same GEMM with the BN-backward
# reduce fused (narrow, HBM-bound shapes)
TC_DGRAD_PREACT = os.environ.get("KRT_TC_DGRAD_PREACT", "1") != "0"
# conv3's backward data gradient on the same GEMM with BN2's reduce fused.  Off
# by default: measured 1% slower per step than cuDNN dgrad + the bwd_reduce
# kernel (3643-3655 vs 3685-3689 samples/s, same box, with the x tile
# TMA-prefetched); KRT_TC_DGRAD=1 selects it
TC_DGRAD = os.environ.get("KRT_TC_DGRAD", "0") == "1"
# bottleneck weight gradients on the own tcgen05 wgrad GEMM (csrc/wgrad_sm100.cu)
# where it measured faster than cuDNN (scripts/bench_conv3_bwd.py, b1024,
# profiles/round2_conv3_bwd_b1024.log): conv3's wgrad with relu(bn2(c2))
# applied in shared memory at the 64/128-wide stages (a2 is never
# materialised; with conv3's dgrad + BN2 reduce also own at width 64: 1.083 ->
# 0.932 ms; width 128: 0.585 -> 0.532 ms), and conv1's wgrad at width 256
# (0.121 -> 0.113 ms).  KRT_TC_WGRAD=0: cuDNN for all of them
TC_WGRAD = os.environ.get("KRT_TC_WGRAD", "1") != "0"
# GPT MLP: fc1's bias + GELU and, in the backward, GELU's derivative and fc1's
# bias gradient in the cuBLASLt epilogues of the GEMMs around them
# (csrc/mlp_lt.cpp); KRT_MLP_LT=0: separate aten GELU / own gelu_bwd_colsum
MLP_LT = os.environ.get("KRT_MLP_LT", "1") != "0"
# the pre-activation unit's 3x3 convolution on the own halo-window kernel
# (csrc/halo_sm100.cu) where it measured faster than cuDNN
# (scripts/bench_narrow3x3.py, ResNet-1001 2048^2 b2, profiles/round2_s3):
# forward with relu(bn1) in its prologue and BN2's statistics in its epilogue
# at 16 / 32 channels (0.35 vs 0.46 ms, 0.18 vs 0.20 ms for cuDNN + apply +
# stats), data gradient at 16 channels (0.30 vs 0.34 ms).  KRT_HALO_UNITS=0:
# cuDNN for all of them
HALO_UNITS = os.environ.get("KRT_HALO_UNITS", "1") != "0"
# its weight gradient on the own narrow-channel wgrad kernel
# (csrc/wgrad_halo_sm100.cu), relu(bn1(c1)) applied in shared memory so the
# backward never rebuilds a1: 0.32 vs 0.90 + 0.10 ms (16 channels), 0.16 vs
# 0.31 + 0.06 ms (32), 0.11 vs 0.09 + 0.03 ms (64) against cuDNN wgrad + the
# bn_apply it needs (scripts/bench_narrow3x3.py).  KRT_WGRAD_UNITS=0: cuDNN
WGRAD_UNITS = os.environ.get("KRT_WGRAD_UNITS", "1") != "0"
# BN0 statistics of a pre-activation unit's input taken from the previous
# unit's conv3 + shortcut GEMM epilogue instead of a bn_stats pass over it.
# The executor hands a unit its producer's latest forward output in every
# path (handoff or regeneration, executor.py _block_input), so in-core and
# out-of-core runs take the statistics from the same place (bitwise equal).
# KRT_STATS_HANDOFF=0: bn_stats
STATS_HANDOFF = os.environ.get("KRT_STATS_HANDOFF", "1") != "0"


def _cl(t):
    """NHWC storage -> NCHW logical tensor with channels_last strides."""
    return t.permute(0, 3, 1, 2)


def _conv_cost(x, w, y):
    """(algorithmic bytes, flops) of y = conv(x, w): operands read once, output written once."""
    return (x.numel() + w.numel() + y.numel()) * x.element_size(), 2.0 * y.numel() * (w.numel() // w.shape[0])


def _conv(x, w, stride, pad):
    with bnfused._timed("cudnn_conv_fwd", 0) as t:
        y = _aten.convolution(x, w, None, [stride, stride], [pad, pad], [1, 1], False, [0, 0], 1)
        t.nbytes, t.flops = _conv_cost(x, w, y)
    return y


class GradPair(tuple):
    """(a, b) standing for the gradient a + b, handed unsummed to the previous
    unit so a fused kernel can add it on the fly (bn_add_relu_bwd dy2)."""


def _dense(dy):
    """Materialise a GradPair (bf16 a + b, rounded like a fused add would)."""
    if isinstance(dy, GradPair):
        return dy[0] + dy[1]
    return dy


def _save_input(dst, x):
    """Copy the unit input into its slot unless the previous unit wrote it there."""
    if dst.data_ptr() != x.data_ptr():
        dst.copy_(x)


def _conv_into(x, w, stride, pad, out=None):
    """conv written straight into `out` (an arena-slot view) when given."""
    if out is None:
        return _conv(x, w, stride, pad)
    cb = torch.backends.cudnn
    with bnfused._timed("cudnn_conv_fwd", 0) as t:
        _aten.cudnn_convolution.out(x, w, [pad, pad], [stride, stride], [1, 1], 1, cb.benchmark,
                                    cb.deterministic, cb.allow_tf32, out=out)
        t.nbytes, t.flops = _conv_cost(x, w, out)
    return out


def _conv_bw(dy, x, w, stride, pad, need_dx=True, need_dw=True):
    # bytes: dy read; wgrad: x read, dw written; dgrad: w read, dx written
    es = dy.element_size()
    nb = dy.numel() * es + (x.numel() + w.numel()) * es * need_dw + (w.numel() + x.numel()) * es * need_dx
    fl = 2.0 * dy.numel() * (w.numel() // w.shape[0]) * (int(need_dx) + int(need_dw))
    with bnfused._timed("cudnn_conv_bwd", nb, fl):
        return _aten.convolution_backward(dy, x, w, None, [stride, stride], [pad, pad], [1, 1], False,
                                          [0, 0], 1, [need_dx, need_dw, False])


def _bn_fw(c, g, b):
    return _aten.native_batch_norm(c, g, b, None, None, True, 0.0, BN_EPS)


def _bn_apply(c, g, b, m, i):
    return _aten.batch_norm_elemt(c, g, b, m, i, BN_EPS)


def _bn_bw(dy, c, g, m, i):
    return _aten.native_batch_norm_backward(dy, c, g, None, None, m, i, True, BN_EPS,
                                            [True, True, True])


def _kaiming(shape_ohwi, gen):
    fan_in = shape_ohwi[1] * shape_ohwi[2] * shape_ohwi[3]
    return torch.randn(shape_ohwi, generator=gen) * math.sqrt(2.0 / fan_in)


class _ConvNetUnit(Unit):
    act = torch.bfloat16

    def saved_input(self, saved):
        return _cl(saved[0])

    def _ir(self, lid, batch, kind_fields):
        grad_bytes = 4 * sum(math.prod(p) for p in self.param_specs())
        return (f"{lid} {kind_fields} elem=2 mem_fwd={self.saved_bytes(batch)} mem_wt=0 "
                f"mem_grad={grad_bytes}")


class StemUnit(_ConvNetUnit):
    """conv7x7/2 (3->64) + BN + ReLU + maxpool3x3/2."""

    name = "stem"

    def __init__(self, res=224, cout=64):
        self.res, self.cout = res, cout
        self.co = res // 2          # conv output side
        self.po = self.co // 2      # pool output side

    def param_specs(self):
        return [(self.cout, 7, 7, 3), (self.cout,), (self.cout,)]

    def saved_specs(self, n):
        return [SavedSpec((n, self.res, self.res, 3), self.act),
                SavedSpec((n, self.co, self.co, self.cout), self.act),
                SavedSpec((2 * self.cout,), torch.float32)]

    def init_params(self, gen):
        return [_kaiming((self.cout, 7, 7, 3), gen), torch.ones(self.cout), torch.zeros(self.cout)]

    def _fused(self):
        return self.act == torch.bfloat16 and bnfused.supported(self.cout)

    def forward(self, x, params, saved):
        w, g, b = params
        wv = _cl(w)
        if saved is not None:
            _cl(saved[0]).copy_(x)
        if self._fused():
            st = saved[2] if saved is not None else torch.empty(2 * self.cout, device=x.device)
            m, i = st[:self.cout], st[self.cout:]
            if TC_CONV1X1 and self.cout == 64:
                # implicit GEMM on tcgen05 with the BN statistics in its epilogue
                # (cuDNN runs a 3-channel NHWC conv on a legacy sm80 kernel)
                c = bnfused.conv_gather(x, wv, 2, 3, out=None if saved is None else _cl(saved[1]), stats=(m, i))
            else:
                c = _conv_into(x, wv, 2, 3, None if saved is None else _cl(saved[1]))
                bnfused.stats(c, m, i)
            return bnfused.relu_maxpool(c, m, i, g, b, 3, 2, 1)   # relu(bn(c)) never materialised
        c = _conv(x, wv, 2, 3)
        o, m, i = _bn_fw(c, g, b)
        if saved is not None:
            _cl(saved[1]).copy_(c)
            saved[2][:self.cout].copy_(m)
            saved[2][self.cout:].copy_(i)
        a = o.relu_()
        y, _ = _aten.max_pool2d_with_indices(a, [3, 3], [2, 2], [1, 1])
        return y

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        w, g, b = params
        x, c = _cl(saved[0]), _cl(saved[1])
        m, i = saved[2][:self.cout], saved[2][self.cout:]
        if self._fused():
            da = bnfused.relu_maxpool_backward(dy, c, m, i, g, b, 3, 2, 1)
            del dy
            dc = bnfused.backward(da, c, m, i, g, b, relu=True, dgamma=grads[1], dbeta=grads[2])
            del da   # (the weight gradient below allocates the padded input)
            if WGRAD_UNITS and self.cout == 64 and self.res % 2 == 0:
                # own tcgen05 kernel, 7x7 windows gathered in shared memory
                # (cuDNN: a legacy sm80 kernel after an NHWC padding pass)
                bnfused.stem_wgrad(dc, x, grads[0])
                return None
            _, dw, _ = _conv_bw(dc, x, _cl(w), 2, 3, need_dx=False)
            _cl(grads[0]).copy_(dw)
            return None
        a = _bn_apply(c, g, b, m, i).relu_()
        _, idx = _aten.max_pool2d_with_indices(a, [3, 3], [2, 2], [1, 1])
        da = _aten.max_pool2d_with_indices_backward(dy, a, [3, 3], [2, 2], [1, 1], [1, 1], False, idx)
        da = _aten.threshold_backward(da, a, 0)
        dc, dg, db = _bn_bw(da, c, g, m, i)
        _, dw, _ = _conv_bw(dc, x, _cl(w), 2, 3, need_dx=False)
        _cl(grads[0]).copy_(dw)
        grads[1].copy_(dg)
        grads[2].copy_(db)
        return None

    def fwd_flops(self, n):
        return 2.0 * n * self.co * self.co * self.cout * 49 * 3

    def ir_line(self, lid, batch, analytic=False):
        return self._ir(lid, batch, f"Conv Wout={self.co} Hout={self.co} Cin=3 Cout={self.cout} K=7")


class BottleneckUnit(_ConvNetUnit):
    """1x1 (cin->w) / 3x3 stride s (w->w) / 1x1 (w->4w), BN after each conv,
    identity or 1x1/s projection shortcut, ReLU after the add."""

    name = "bottleneck"

    def __init__(self, cin, width, stride, side_in):
        self.cin, self.w, self.s = cin, width, stride
        self.cout = 4 * width
        self.hi = side_in
        self.ho = side_in // stride
        self.down = stride != 1 or cin != self.cout

    def param_specs(self):
        p = [(self.w, 1, 1, self.cin), (self.w,), (self.w,),
             (self.w, 3, 3, self.w), (self.w,), (self.w,),
             (self.cout, 1, 1, self.w), (self.cout,), (self.cout,)]
        if self.down:
            p += [(self.cout, 1, 1, self.cin), (self.cout,), (self.cout,)]
        return p

    def _nstats(self):
        return 2 * (2 * self.w + self.cout + (self.cout if self.down else 0))

    def saved_specs(self, n):
        s = [SavedSpec((n, self.hi, self.hi, self.cin), self.act),
             SavedSpec((n, self.hi, self.hi, self.w), self.act),
             SavedSpec((n, self.ho, self.ho, self.w), self.act),
             SavedSpec((n, self.ho, self.ho, self.cout), self.act)]
        if self.down:
            s.append(SavedSpec((n, self.ho, self.ho, self.cout), self.act))
        s.append(SavedSpec((self._nstats(),), torch.float32))
        return s

    def init_params(self, gen):
        out = []
        for shp in self.param_specs():
            if len(shp) == 4:
                out.append(_kaiming(shp, gen))
            else:
                out.append(torch.ones(shp) if len(out) % 3 == 1 else torch.zeros(shp))
        # zero-init the last BN gamma of the residual branch (standard practice)
        out[7] = torch.zeros(self.cout)
        return out

    def _stats_views(self, st):
        sizes = [self.w, self.w, self.w, self.w, self.cout, self.cout]
        if self.down:
            sizes += [self.cout, self.cout]
        views, o = [], 0
        for k in sizes:
            views.append(st[o:o + k])
            o += k
        return views

    def _fused(self):
        return self.act == torch.bfloat16 and all(bnfused.supported(c) for c in (self.w, self.cout))

    def _tc1x1(self):
        # both 1x1 convolutions (stride 1 in this bottleneck) fit the tcgen05 GEMM
        return (self._fused() and TC_CONV1X1 and bnfused.conv1x1_supported(self.cin, self.w)
                and bnfused.conv1x1_supported(self.w, self.cout, pre=True))

    def _forward_fused(self, x, params, saved, out=None):
        w1, g1, b1, w2, g2, b2, w3, g3, b3 = params[:9]
        if saved is not None:
            _save_input(_cl(saved[0]), x)
            st = self._stats_views(saved[-1])
        else:
            st = self._stats_views(torch.empty(self._nstats(), device=x.device))
        sv = (lambda k: None) if saved is None else (lambda k: _cl(saved[k]))
        if self._tc1x1():
            # 1x1 convolutions on the tcgen05 GEMM: BN statistics of c1 and c3
            # reduced in its epilogue, relu(bn2(c2)) applied in its prologue
            c1 = bnfused.conv1x1(x, _cl(w1), out=sv(1), stats=(st[0], st[1]))
            a1 = bnfused.apply(c1, st[0], st[1], g1, b1, relu=True)
            c2 = _conv_into(a1, _cl(w2), self.s, 1, sv(2))
            del a1
            bnfused.stats(c2, st[2], st[3])
            c3 = bnfused.conv1x1(c2, _cl(w3), out=sv(3), pre=(st[2], st[3], g2, b2), stats=(st[4], st[5]))
        else:
            c1 = _conv_into(x, _cl(w1), 1, 0, sv(1))
            a1 = bnfused.stats_apply(c1, st[0], st[1], g1, b1, relu=True)
            c2 = _conv_into(a1, _cl(w2), self.s, 1, sv(2))
            del a1
            a2 = bnfused.stats_apply(c2, st[2], st[3], g2, b2, relu=True)
            c3 = _conv_into(a2, _cl(w3), 1, 0, sv(3))
            del a2
        if self.down:
            wd, gd, bd = params[9:12]
            if not self._tc1x1():
                bnfused.stats(c3, st[4], st[5])
            cd = _conv_into(x, _cl(wd), self.s, 0, sv(4))
            bnfused.stats(cd, st[6], st[7])
            return bnfused.apply(c3, st[4], st[5], g3, b3, relu=True, res=cd, rstats=(st[6], st[7]),
                                 rg=gd, rb=bd, out=out)
        if self._tc1x1():
            return bnfused.apply(c3, st[4], st[5], g3, b3, relu=True, res=x, out=out)
        return bnfused.stats_apply(c3, st[4], st[5], g3, b3, relu=True, res=x, out=out)

    def _backward_fused(self, dy, params, saved, grads):
        w1, g1, b1, w2, g2, b2, w3, g3, b3 = params[:9]
        x, c1, c2, c3 = (_cl(t) for t in saved[:4])
        st = self._stats_views(saved[-1])
        dy, dy2 = (dy[0], dy[1]) if isinstance(dy, GradPair) else (dy, None)
        if self.down:
            wd, gd, bd = params[9:12]
            cd = _cl(saved[4])
            dz = bnfused.add_relu_bwd(dy, c3, st[4], st[5], g3, b3, cd, rstats=(st[6], st[7]), rg=gd, rb=bd,
                                      dy2=dy2)
            dc3 = bnfused.backward(dz, c3, st[4], st[5], g3, b3, relu=False, dgamma=grads[7], dbeta=grads[8])
        else:
            dz, dc3 = bnfused.add_relu_backward(dy, c3, st[4], st[5], g3, b3, x, dgamma=grads[7],
                                                dbeta=grads[8], dy2=dy2)
        del dy, dy2
        if self._own_wgrad3():
            # conv3's weight gradient on the tcgen05 wgrad GEMM, relu(bn2(c2))
            # applied in shared memory (a2 never materialised)
            bnfused.conv_wgrad(dc3, c2, grads[6].view(-1), 1, 1, 0, pre=(st[2], st[3], g2, b2))
            if self.w == 64 and bnfused.conv1x1_dgrad_supported(self.cout, self.w):
                # its data gradient with BN2's backward reduce in the epilogue
                dc2 = bnfused.conv1x1_dgrad_bn_backward(dc3, _cl(w3), c2, st[2], st[3], g2, b2,
                                                        dgamma=grads[4], dbeta=grads[5])
            else:
                da2, _, _ = _conv_bw(dc3, c2, _cl(w3), 1, 0, need_dw=False)
                dc2 = bnfused.backward(da2, c2, st[2], st[3], g2, b2, relu=True, dgamma=grads[4],
                                       dbeta=grads[5])
                del da2
            del dc3
            return self._backward_tail(dz, params, saved, grads, c1, st, dc2)
        a2 = bnfused.apply(c2, st[2], st[3], g2, b2, relu=True)
        if self._tc1x1() and TC_DGRAD:
            # conv3 dgrad on the tcgen05 GEMM with BN2's backward reduce in its
            # epilogue; cuDNN keeps the weight gradient
            _, dw3, _ = _conv_bw(dc3, a2, _cl(w3), 1, 0, need_dx=False)
            del a2
            _cl(grads[6]).copy_(dw3)
            dc2 = bnfused.conv1x1_dgrad_bn_backward(dc3, _cl(w3), c2, st[2], st[3], g2, b2,
                                                    dgamma=grads[4], dbeta=grads[5])
            del dc3
        else:
            da2, dw3, _ = _conv_bw(dc3, a2, _cl(w3), 1, 0)
            del dc3, a2
            _cl(grads[6]).copy_(dw3)
            dc2 = bnfused.backward(da2, c2, st[2], st[3], g2, b2, relu=True, dgamma=grads[4], dbeta=grads[5])
            del da2
        return self._backward_tail(dz, params, saved, grads, c1, st, dc2)

    def _own_wgrad3(self):
        return (self._tc1x1() and TC_WGRAD and self.w in (64, 128)
                and bnfused.conv_wgrad_supported(self.cout, self.w, 1, 1, pre=True))

    def _backward_tail(self, dz, params, saved, grads, c1, st, dc2):
        """conv2 / BN1 / conv1 (and the downsample branch) backward from dc2."""
        w1, g1, b1, w2 = params[:4]
        x = _cl(saved[0])
        a1 = bnfused.apply(c1, st[0], st[1], g1, b1, relu=True)
        da1, dw2, _ = _conv_bw(dc2, a1, _cl(w2), self.s, 1)
        del dc2, a1
        _cl(grads[3]).copy_(dw2)
        dc1 = bnfused.backward(da1, c1, st[0], st[1], g1, b1, relu=True, dgamma=grads[1], dbeta=grads[2])
        del da1
        if TC_WGRAD and self._tc1x1() and self.w == 256 and bnfused.conv_wgrad_supported(self.w, self.cin, 1, 1):
            # conv1's weight gradient on the tcgen05 wgrad GEMM (x is the unit input)
            bnfused.conv_wgrad(dc1, x, grads[0].view(-1), 1, 1, 0)
            dx, _, _ = _conv_bw(dc1, x, _cl(w1), 1, 0, need_dw=False)
        else:
            dx, dw1, _ = _conv_bw(dc1, x, _cl(w1), 1, 0)
            _cl(grads[0]).copy_(dw1)
        del dc1
        if self.down:
            wd, gd, bd = params[9:12]
            cd = _cl(saved[4])
            dcd = bnfused.backward(dz, cd, st[6], st[7], gd, bd, relu=False, dgamma=grads[10],
                                   dbeta=grads[11])
            dxd, dwd, _ = _conv_bw(dcd, x, _cl(wd), self.s, 0)
            _cl(grads[9]).copy_(dwd)
            return GradPair((dx, dxd))
        return GradPair((dx, dz))

    @property
    def writes_out(self):
        return self._fused()

    def forward(self, x, params, saved, out=None):
        if self._fused():
            return self._forward_fused(x, params, saved, out)
        w1, g1, b1, w2, g2, b2, w3, g3, b3 = params[:9]
        if saved is not None:
            _cl(saved[0]).copy_(x)
        c1 = _conv(x, _cl(w1), 1, 0)
        o1, m1, i1 = _bn_fw(c1, g1, b1)
        a1 = o1.relu_()
        c2 = _conv(a1, _cl(w2), self.s, 1)
        o2, m2, i2 = _bn_fw(c2, g2, b2)
        a2 = o2.relu_()
        c3 = _conv(a2, _cl(w3), 1, 0)
        o3, m3, i3 = _bn_fw(c3, g3, b3)
        stats = [m1, i1, m2, i2, m3, i3]
        if self.down:
            wd, gd, bd = params[9:12]
            cd = _conv(x, _cl(wd), self.s, 0)
            od, md, idd = _bn_fw(cd, gd, bd)
            stats += [md, idd]
            o3.add_(od)
        else:
            o3.add_(x)
        if saved is not None:
            _cl(saved[1]).copy_(c1)
            _cl(saved[2]).copy_(c2)
            _cl(saved[3]).copy_(c3)
            if self.down:
                _cl(saved[4]).copy_(cd)
            for v, t in zip(self._stats_views(saved[-1]), stats):
                v.copy_(t)
        return o3.relu_()

    def backward(self, dy, params, saved, grads):
        if self._fused():
            return self._backward_fused(dy, params, saved, grads)
        dy = _dense(dy)
        w1, g1, b1, w2, g2, b2, w3, g3, b3 = params[:9]
        x, c1, c2, c3 = (_cl(t) for t in saved[:4])
        st = self._stats_views(saved[-1])
        m1, i1, m2, i2, m3, i3 = st[:6]
        a1 = _bn_apply(c1, g1, b1, m1, i1).relu_()
        a2 = _bn_apply(c2, g2, b2, m2, i2).relu_()
        y = _bn_apply(c3, g3, b3, m3, i3)
        if self.down:
            wd, gd, bd = params[9:12]
            cd = _cl(saved[4])
            md, idd = st[6], st[7]
            y.add_(_bn_apply(cd, gd, bd, md, idd))
        else:
            y.add_(x)
        y.relu_()
        dz = _aten.threshold_backward(dy, y, 0)
        del y
        dc3, dg3, db3 = _bn_bw(dz, c3, g3, m3, i3)
        da2, dw3, _ = _conv_bw(dc3, a2, _cl(w3), 1, 0)
        del dc3
        da2 = _aten.threshold_backward(da2, a2, 0)
        dc2, dg2, db2 = _bn_bw(da2, c2, g2, m2, i2)
        del da2
        da1, dw2, _ = _conv_bw(dc2, a1, _cl(w2), self.s, 1)
        del dc2
        da1 = _aten.threshold_backward(da1, a1, 0)
        dc1, dg1, db1 = _bn_bw(da1, c1, g1, m1, i1)
        del da1
        dx, dw1, _ = _conv_bw(dc1, x, _cl(w1), 1, 0)
        del dc1
        gs = [dw1, dg1, db1, dw2, dg2, db2, dw3, dg3, db3]
        if self.down:
            dcd, dgd, dbd = _bn_bw(dz, cd, gd, md, idd)
            dxd, dwd, _ = _conv_bw(dcd, x, _cl(wd), self.s, 0)
            dx.add_(dxd)
            gs += [dwd, dgd, dbd]
        else:
            dx.add_(dz)
        for gv, t in zip(grads, gs):
            (_cl(gv) if gv.dim() == 4 else gv).copy_(t)
        return dx

    def fwd_flops(self, n):
        macs = (self.hi * self.hi * self.cin * self.w + self.ho * self.ho * 9 * self.w * self.w
                + self.ho * self.ho * self.w * self.cout)
        if self.down:
            macs += self.ho * self.ho * self.cin * self.cout
        return 2.0 * n * macs

    def ir_line(self, lid, batch, analytic=False):
        params = sum(math.prod(p) for p in self.param_specs() if len(p) == 4)
        return self._ir(lid, batch, f"Conv Wout={self.ho} Hout={self.ho} Cin=1 Cout={params} K=1")


class HeadUnit(_ConvNetUnit):
    """global average pool + FullyConnected (with bias) -> logits."""

    name = "head"

    def __init__(self, cin=2048, classes=1000, side=7):
        self.cin, self.k, self.side = cin, classes, side

    def param_specs(self):
        return [(self.k, self.cin), (self.k,)]

    def saved_specs(self, n):
        return [SavedSpec((n, self.side, self.side, self.cin), self.act)]

    def init_params(self, gen):
        bound = 1.0 / math.sqrt(self.cin)
        return [torch.empty(self.k, self.cin).uniform_(-bound, bound, generator=gen),
                torch.empty(self.k).uniform_(-bound, bound, generator=gen)]

    def forward(self, x, params, saved):
        w, b = params
        if saved is not None:
            _cl(saved[0]).copy_(x)
        p = x.mean(dim=(2, 3))
        return torch.addmm(b, p, w.t())

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        w, b = params
        x = _cl(saved[0])
        p = x.mean(dim=(2, 3))
        grads[0].copy_(torch.mm(dy.t(), p, out_dtype=torch.float32))
        grads[1].copy_(dy.float().sum(0))
        dp = torch.mm(dy, w) * (1.0 / (self.side * self.side))
        n = dp.shape[0]
        return dp[:, :, None, None].expand(n, self.cin, self.side, self.side).contiguous(
            memory_format=torch.channels_last)

    def fwd_flops(self, n):
        return 2.0 * n * self.cin * self.k

    def ir_line(self, lid, batch, analytic=False):
        return self._ir(lid, batch, f"FullyConnected X={self.cin} Y={self.k}")


def cross_entropy_loss(logits, target):
    """Softmax cross-entropy, mean over the batch; dlogits in the logits dtype."""
    lf = logits.float()
    loss = F.cross_entropy(lf, target)
    p = torch.softmax(lf, dim=1)
    p[torch.arange(p.shape[0], device=p.device), target] -= 1.0
    return loss, (p * (1.0 / p.shape[0])).to(logits.dtype)


RESNET_DEPTHS = {50: (3, 4, 6, 3), 101: (3, 4, 23, 3), 152: (3, 8, 36, 3), 200: (3, 24, 36, 3)}


def resnet_units(depth: int = 200, res: int = 224, classes: int = 1000, stages=None,
                 act_dtype=torch.bfloat16):
    """ImageNet bottleneck ResNet as executor units: stem, sum(stages) bottlenecks, head."""
    stages = stages or RESNET_DEPTHS[depth]
    units = [StemUnit(res)]
    side = res // 4
    cin = 64
    for si, count in enumerate(stages):
        width = 64 * 2 ** si
        for k in range(count):
            stride = 2 if (k == 0 and si > 0) else 1
            units.append(BottleneckUnit(cin, width, stride, side))
            side //= stride
            cin = 4 * width
    units.append(HeadUnit(cin, classes, side))
    for u in units:
        u.act = act_dtype
    return units


# ---------------------------------------------------------------------------
# Pre-activation bottleneck ResNet (He et al. 2016, "Identity Mappings"):
# ResNet-1001 for CIFAR-style inputs, cfg2 = 2048x2048 images.
# unit: a0 = relu(bn0(x)); c1 = conv1x1(a0); c2 = conv3x3/s(relu(bn1(c1)));
#       y = conv1x1(relu(bn2(c2))) + (x | conv1x1/s(a0)).
# Saved: x, c1, c2 and the three BN statistics; a0/a1/a2 are recomputed in
# backward and c3 is never needed (no BN after the last conv).
# ---------------------------------------------------------------------------
def _stats_fw(c, st_m, st_i):
    """Batch statistics into (mean, invstd) views; fused kernel for bf16."""
    if c.dtype == torch.bfloat16 and bnfused.supported(c.shape[1]):
        bnfused.stats(c, st_m, st_i)
    else:
        m = c.float().mean(dim=(0, 2, 3))
        v = c.float().var(dim=(0, 2, 3), unbiased=False)
        st_m.copy_(m)
        st_i.copy_(torch.rsqrt(v + BN_EPS))


def _stats_bn_relu(c, st_m, st_i, g, b):
    """_stats_fw then _bn_relu; one cooperative kernel for bf16."""
    if c.dtype == torch.bfloat16 and bnfused.supported(c.shape[1]):
        return bnfused.stats_apply(c, st_m, st_i, g, b, relu=True)
    _stats_fw(c, st_m, st_i)
    return _bn_relu(c, st_m, st_i, g, b)


def _bn_relu(c, m, i, g, b):
    if c.dtype == torch.bfloat16 and bnfused.supported(c.shape[1]):
        return bnfused.apply(c, m, i, g, b, relu=True)
    return _bn_apply(c, g, b, m, i).relu_()


def _bn_relu_bw(da, c, m, i, g, b, dg, db, addend=None):
    """Backward through relu(bn(c)) given d(relu output); writes dgamma/dbeta.
    addend: a residual gradient summed into the result (fused for bf16)."""
    if c.dtype == torch.bfloat16 and bnfused.supported(c.shape[1]):
        return bnfused.backward(da, c, m, i, g, b, relu=True, dgamma=dg, dbeta=db, addend=addend)
    a = _bn_apply(c, g, b, m, i).relu_()
    dpre = _aten.threshold_backward(da, a, 0)
    dc, dgg, dbb = _bn_bw(dpre, c, g, m, i)
    dg.copy_(dgg)
    db.copy_(dbb)
    return dc if addend is None else dc.add_(addend)


class PreActBottleneckUnit(_ConvNetUnit):
    name = "preact_bottleneck"

    def __init__(self, cin, width, stride, side_in):
        self.cin, self.w, self.s = cin, width, stride
        self.cout = 4 * width
        self.hi, self.ho = side_in, side_in // stride
        self.down = stride != 1 or cin != self.cout
        self.prev_unit = None     # set by the executor: the unit whose output this one takes
        self._ostats = None       # fp32 [2, cout]: batch statistics of the latest forward output
        self._ostats_ptr = None   # ... and that output's address

    def param_specs(self):
        p = [(self.cin,), (self.cin,), (self.w, 1, 1, self.cin),
             (self.w,), (self.w,), (self.w, 3, 3, self.w),
             (self.w,), (self.w,), (self.cout, 1, 1, self.w)]
        if self.down:
            p.append((self.cout, 1, 1, self.cin))
        return p

    def _nstats(self):
        return 2 * (self.cin + 2 * self.w)

    def saved_specs(self, n):
        return [SavedSpec((n, self.hi, self.hi, self.cin), self.act),
                SavedSpec((n, self.hi, self.hi, self.w), self.act),
                SavedSpec((n, self.ho, self.ho, self.w), self.act),
                SavedSpec((self._nstats(),), torch.float32)]

    def init_params(self, gen):
        out = []
        for shp in self.param_specs():
            if len(shp) == 4:
                out.append(_kaiming(shp, gen))
            else:
                out.append(torch.ones(shp) if len(out) % 3 == 0 else torch.zeros(shp))
        return out

    def _st(self, st):
        k = [self.cin, self.cin, self.w, self.w, self.w, self.w]
        v, o = [], 0
        for n in k:
            v.append(st[o:o + n])
            o += n
        return v

    writes_out = True

    def _tc1x1(self):
        # both 1x1 convolutions on the tcgen05 GEMM (K and N down to 16)
        return (self.act == torch.bfloat16 and TC_CONV1X1
                and all(bnfused.supported(c) for c in (self.cin, self.w))
                and bnfused.conv1x1_supported(self.cin, self.w, pre=True)
                and bnfused.conv1x1_supported(self.w, self.cout, pre=True))

    def _forward_tc(self, x, params, st, sv, out):
        """relu(bn0) applied in conv1's prologue (a0 never written unless the
        shortcut is strided), BN1 statistics from conv1's epilogue, relu(bn2)
        in conv3's prologue and the shortcut added in its epilogue."""
        g0, b0, w1, g1, b1, w2, g2, b2, w3 = params[:9]
        src = self._input_stats(x)
        if src is not None:
            st[0].copy_(src[0])
            st[1].copy_(src[1])
        else:
            _stats_fw(x, st[0], st[1])
        bn0 = (st[0], st[1], g0, b0)
        c1 = bnfused.conv1x1(x, _cl(w1), out=sv(1), pre=bn0, stats=(st[2], st[3]))
        if not self.down:
            sc = x
        elif self.s == 1 and bnfused.conv1x1_supported(self.cin, self.cout, pre=True):
            sc = bnfused.conv1x1(x, _cl(params[9]), pre=bn0)
        else:
            a0 = _bn_relu(x, st[0], st[1], g0, b0)
            sc = _conv(a0, _cl(params[9]), self.s, 0)
            del a0
        if self._halo_fwd():
            # the 3x3 convolution of relu(bn1(c1)) (never written) with BN2's
            # statistics in the epilogue
            c2 = bnfused.conv_im2col(c1, w2, 1, 1, out=sv(2), pre=(st[2], st[3], g1, b1), stats=(st[4], st[5]))
        else:
            a1 = _bn_relu(c1, st[2], st[3], g1, b1)
            c2 = _conv_into(a1, _cl(w2), self.s, 1, sv(2))
            del a1
            _stats_fw(c2, st[4], st[5])
        ostats = None
        if STATS_HANDOFF:
            if self._ostats is None or self._ostats.device != c2.device:
                self._ostats = torch.empty(2, self.cout, dtype=torch.float32, device=c2.device)
            ostats = (self._ostats[0], self._ostats[1])
        y = bnfused.conv1x1(c2, _cl(w3), out=out, pre=(st[4], st[5], g2, b2), res=sc, stats=ostats)
        self._ostats_ptr = y.data_ptr() if ostats is not None else None
        return y

    def _input_stats(self, x):
        """The producer's epilogue statistics of x, when x is its latest output."""
        p = self.prev_unit
        if (STATS_HANDOFF and isinstance(p, PreActBottleneckUnit) and p._ostats_ptr is not None
                and p._ostats_ptr == x.data_ptr() and p.cout == self.cin):
            return p._ostats[0], p._ostats[1]
        return None

    def _halo_fwd(self):
        return (HALO_UNITS and self.act == torch.bfloat16 and self.s == 1 and self.w in (16, 32)
                and bnfused.conv3x3_halo_supported(self.ho, self.ho, self.w, self.w, pre=True))

    def _halo_dgrad(self):
        return (HALO_UNITS and self.act == torch.bfloat16 and self.s == 1 and self.w == 16
                and bnfused.conv3x3_halo_supported(self.ho, self.ho, self.w, self.w))

    def forward(self, x, params, saved, out=None):
        g0, b0, w1, g1, b1, w2, g2, b2, w3 = params[:9]
        if saved is not None:
            _save_input(_cl(saved[0]), x)
            st = self._st(saved[3])
        else:
            st = self._st(torch.empty(self._nstats(), device=x.device))
        sv = (lambda k: None) if saved is None else (lambda k: _cl(saved[k]))
        if self._tc1x1():
            return self._forward_tc(x, params, st, sv, out)
        a0 = _stats_bn_relu(x, st[0], st[1], g0, b0)
        c1 = _conv_into(a0, _cl(w1), 1, 0, sv(1))
        sc = _conv(a0, _cl(params[9]), self.s, 0) if self.down else x
        del a0
        a1 = _stats_bn_relu(c1, st[2], st[3], g1, b1)
        c2 = _conv_into(a1, _cl(w2), self.s, 1, sv(2))
        del a1
        a2 = _stats_bn_relu(c2, st[4], st[5], g2, b2)
        y = _conv(a2, _cl(w3), 1, 0)
        if out is not None:
            return torch.add(y, sc, out=out)
        return y.add_(sc)

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        g0, b0, w1, g1, b1, w2, g2, b2, w3 = params[:9]
        x, c1, c2 = (_cl(t) for t in saved[:3])
        st = self._st(saved[3])
        tc = self._tc1x1() and TC_DGRAD_PREACT
        if tc and self._narrow_wgrad1(self.w, self.cout) and bnfused.conv1x1_dgrad_supported(self.cout, self.w):
            # conv3's weight gradient from c2 with relu(bn2) in shared memory
            # (a2 never rebuilt); its dgrad with BN2's backward reduce on the GEMM
            bnfused.wgrad1x1_narrow(dy, c2, grads[8], pre=(st[4], st[5], g2, b2))
            dc2 = bnfused.conv1x1_dgrad_bn_backward(dy, _cl(w3), c2, st[4], st[5], g2, b2, dgamma=grads[6],
                                                    dbeta=grads[7])
        elif tc and bnfused.conv1x1_dgrad_supported(self.cout, self.w):
            a2 = _bn_relu(c2, st[4], st[5], g2, b2)
            # conv3 dgrad on the tcgen05 GEMM with BN2's backward reduce in its epilogue
            _, dw3, _ = _conv_bw(dy, a2, _cl(w3), 1, 0, need_dx=False)
            del a2
            _cl(grads[8]).copy_(dw3)
            dc2 = bnfused.conv1x1_dgrad_bn_backward(dy, _cl(w3), c2, st[4], st[5], g2, b2, dgamma=grads[6],
                                                    dbeta=grads[7])
        else:
            a2 = _bn_relu(c2, st[4], st[5], g2, b2)
            da2, dw3, _ = _conv_bw(dy, a2, _cl(w3), 1, 0)
            del a2
            _cl(grads[8]).copy_(dw3)
            dc2 = _bn_relu_bw(da2, c2, st[4], st[5], g2, b2, grads[6], grads[7])
            del da2
        if self._narrow_wgrad():
            # weight gradient from c1 with relu(bn1) in shared memory (a1 is
            # never rebuilt); the data gradient on the halo kernel or cuDNN
            bnfused.wgrad3x3_narrow(dc2, c1, grads[5], pre=(st[2], st[3], g1, b1))
            if self._halo_dgrad():
                da1 = bnfused.conv3x3_dgrad(dc2, w2)
            else:
                da1, _, _ = _conv_bw(dc2, c1, _cl(w2), self.s, 1, need_dw=False)
            del dc2
            dc1 = _bn_relu_bw(da1, c1, st[2], st[3], g1, b1, grads[3], grads[4])
            del da1
            return self._backward_conv1(dy, params, x, st, grads, dc1, tc)
        a1 = _bn_relu(c1, st[2], st[3], g1, b1)
        if self._halo_dgrad():
            # data gradient on the halo kernel (flipped, transposed weights);
            # cuDNN keeps the weight gradient
            _, dw2, _ = _conv_bw(dc2, a1, _cl(w2), self.s, 1, need_dx=False)
            da1 = bnfused.conv3x3_dgrad(dc2, w2)
        else:
            da1, dw2, _ = _conv_bw(dc2, a1, _cl(w2), self.s, 1)
        del dc2, a1
        _cl(grads[5]).copy_(dw2)
        dc1 = _bn_relu_bw(da1, c1, st[2], st[3], g1, b1, grads[3], grads[4])
        del da1
        return self._backward_conv1(dy, params, x, st, grads, dc1, tc)

    def _narrow_wgrad(self):
        return (WGRAD_UNITS and self.act == torch.bfloat16 and self.s == 1 and self.w in (16, 32, 64)
                and bnfused.wgrad3x3_narrow_supported(self.ho, self.ho, self.w))

    def _narrow_wgrad1(self, cin, cout):
        return WGRAD_UNITS and self.act == torch.bfloat16 and bnfused.wgrad1x1_narrow_supported(cin, cout)

    def _backward_conv1(self, dy, params, x, st, grads, dc1, tc):
        """BN0 / conv1 (and the projection shortcut) backward from dc1."""
        g0, b0, w1 = params[:3]
        if (tc and not self.down and self._narrow_wgrad1(self.cin, self.w)
                and bnfused.conv1x1_dgrad_supported(self.w, self.cin)):
            # conv1's weight gradient from x with relu(bn0) in shared memory (a0
            # never rebuilt); dgrad + BN0's backward reduce on the GEMM, the
            # identity shortcut's gradient dy added in the elementwise pass
            bnfused.wgrad1x1_narrow(dc1, x, grads[2], pre=(st[0], st[1], g0, b0))
            return bnfused.conv1x1_dgrad_bn_backward(dc1, _cl(w1), x, st[0], st[1], g0, b0, dgamma=grads[0],
                                                     dbeta=grads[1], addend=dy)
        a0 = _bn_relu(x, st[0], st[1], g0, b0)
        if tc and not self.down and bnfused.conv1x1_dgrad_supported(self.w, self.cin):
            # conv1 dgrad + BN0's backward reduce on the GEMM; the identity
            # shortcut's gradient dy added in the elementwise pass
            _, dw1, _ = _conv_bw(dc1, a0, _cl(w1), 1, 0, need_dx=False)
            del a0
            _cl(grads[2]).copy_(dw1)
            return bnfused.conv1x1_dgrad_bn_backward(dc1, _cl(w1), x, st[0], st[1], g0, b0, dgamma=grads[0],
                                                     dbeta=grads[1], addend=dy)
        da0, dw1, _ = _conv_bw(dc1, a0, _cl(w1), 1, 0)
        del dc1
        _cl(grads[2]).copy_(dw1)
        if self.down:
            das, dws, _ = _conv_bw(dy, a0, _cl(params[9]), self.s, 0)
            _cl(grads[9]).copy_(dws)
            da0.add_(das)
            dx = _bn_relu_bw(da0, x, st[0], st[1], g0, b0, grads[0], grads[1])
        else:   # identity shortcut: its gradient dy is added inside the BN backward pass
            dx = _bn_relu_bw(da0, x, st[0], st[1], g0, b0, grads[0], grads[1], addend=dy)
        return dx

    def fwd_flops(self, n):
        macs = (self.hi ** 2 * self.cin * self.w + self.ho ** 2 * 9 * self.w * self.w
                + self.ho ** 2 * self.w * self.cout)
        if self.down:
            macs += self.ho ** 2 * self.cin * self.cout
        return 2.0 * n * macs

    def ir_line(self, lid, batch, analytic=False):
        params = sum(math.prod(p) for p in self.param_specs() if len(p) == 4)
        return self._ir(lid, batch, f"Conv Wout={self.ho} Hout={self.ho} Cin=1 Cout={params} K=1")


class CifarStemUnit(_ConvNetUnit):
    """conv3x3 (3 -> 16), no BN/ReLU (the pre-activation units normalise)."""

    name = "cifar_stem"

    def __init__(self, res, cout=16):
        self.res, self.cout = res, cout

    def param_specs(self):
        return [(self.cout, 3, 3, 3)]

    def saved_specs(self, n):
        return [SavedSpec((n, self.res, self.res, 3), self.act)]

    def init_params(self, gen):
        return [_kaiming((self.cout, 3, 3, 3), gen)]

    def forward(self, x, params, saved):
        if saved is not None:
            _cl(saved[0]).copy_(x)
        return _conv(x, _cl(params[0]), 1, 1)

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        _, dw, _ = _conv_bw(dy, _cl(saved[0]), _cl(params[0]), 1, 1, need_dx=False)
        _cl(grads[0]).copy_(dw)
        return None

    def fwd_flops(self, n):
        return 2.0 * n * self.res * self.res * self.cout * 27

    def ir_line(self, lid, batch, analytic=False):
        return self._ir(lid, batch, f"Conv Wout={self.res} Hout={self.res} Cin=3 Cout={self.cout} K=3")


class PreActHeadUnit(_ConvNetUnit):
    """relu(bn(x)) -> global average pool -> FullyConnected (bias)."""

    name = "preact_head"

    def __init__(self, cin, classes, side):
        self.cin, self.k, self.side = cin, classes, side

    def param_specs(self):
        return [(self.cin,), (self.cin,), (self.k, self.cin), (self.k,)]

    def saved_specs(self, n):
        return [SavedSpec((n, self.side, self.side, self.cin), self.act),
                SavedSpec((2 * self.cin,), torch.float32)]

    def init_params(self, gen):
        bound = 1.0 / math.sqrt(self.cin)
        return [torch.ones(self.cin), torch.zeros(self.cin),
                torch.empty(self.k, self.cin).uniform_(-bound, bound, generator=gen),
                torch.empty(self.k).uniform_(-bound, bound, generator=gen)]

    def forward(self, x, params, saved):
        g, b, w, bias = params
        st = saved[1] if saved is not None else torch.empty(2 * self.cin, device=x.device)
        if saved is not None:
            _cl(saved[0]).copy_(x)
        a = _stats_bn_relu(x, st[:self.cin], st[self.cin:], g, b)
        p = a.float().mean(dim=(2, 3)).to(a.dtype)
        return torch.addmm(bias, p, w.t())

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        g, b, w, bias = params
        x, st = _cl(saved[0]), saved[1]
        a = _bn_relu(x, st[:self.cin], st[self.cin:], g, b)
        p = a.float().mean(dim=(2, 3)).to(a.dtype)
        grads[2].copy_(torch.mm(dy.t(), p, out_dtype=torch.float32) if dy.dtype != torch.float32
                       else torch.mm(dy.t(), p))
        grads[3].copy_(dy.float().sum(0))
        dp = torch.mm(dy, w) * (1.0 / (self.side * self.side))
        n = dp.shape[0]
        da = dp[:, :, None, None].expand(n, self.cin, self.side, self.side).contiguous(
            memory_format=torch.channels_last)
        return _bn_relu_bw(da, x, st[:self.cin], st[self.cin:], g, b, grads[0], grads[1])

    def fwd_flops(self, n):
        return 2.0 * n * self.cin * self.k

    def ir_line(self, lid, batch, analytic=False):
        return self._ir(lid, batch, f"FullyConnected X={self.cin} Y={self.k}")


def resnet1001_units(res: int = 2048, classes: int = 10, depth: int = 1001, act_dtype=torch.bfloat16):
    """CIFAR-style pre-activation bottleneck ResNet: (depth-2)/9 units per stage, widths 16/32/64."""
    per = (depth - 2) // 9
    units = [CifarStemUnit(res, 16)]
    side, cin = res, 16
    for si in range(3):
        width = 16 * 2 ** si
        for k in range(per):
            stride = 2 if (k == 0 and si > 0) else 1
            units.append(PreActBottleneckUnit(cin, width, stride, side))
            side //= stride
            cin = 4 * width
    units.append(PreActHeadUnit(cin, classes, side))
    for u in units:
        u.act = act_dtype
    return units


# ---------------------------------------------------------------------------
# GPT-style transformer (cfg3 Megatron-8.3B shape, cfg4 Turing-NLG-17B shape):
# token+position embedding, pre-LN decoder layers, final LN + LM head.
# Tokens are flattened to rows T = batch*seq.  Each decoder layer saves x,
# qkv, the attention output, x2 = x + attn, the fc1 pre-activation and the
# LN statistics (+ softmax logsumexp for flash attention); LN outputs, GELU
# and the attention probabilities are recomputed in backward.
# IR mapping: a layer is `Conv Wout=seq Hout=1 K=1 Cin=H Cout=12H` so the
# reference cost model counts seq*12H^2 MACs per sample and 12H^2 weights.
# ---------------------------------------------------------------------------
LN_EPS = 1e-5


def _ln_fw(x, g, b, mean, rstd, residual=None, x2_out=None):
    """LayerNorm(x [+ residual]); bf16 on the fused kernel (x2 = x + residual
    written to x2_out), otherwise aten.  Returns the normalised rows."""
    if lnfused.supported(x):
        t = x.shape[0]
        m = mean if mean is not None else torch.empty(t, device=x.device)
        r = rstd if rstd is not None else torch.empty(t, device=x.device)
        if residual is not None and x2_out is None:
            x2_out = torch.empty_like(x)
        h = lnfused.ln_fwd(x, g, b, LN_EPS, m, r, residual=residual, x2_out=x2_out)
        return h, (x2_out if residual is not None else x)
    if residual is not None:
        x = torch.add(x, residual, out=x2_out) if x2_out is not None else x + residual
    y, m, r = _aten.native_layer_norm(x, [x.shape[-1]], g, b, LN_EPS)
    if mean is not None:
        mean.copy_(m.view(-1))
        rstd.copy_(r.view(-1))
    return y, x


def _ln_apply(x, g, b, mean, rstd):
    """The forward's LayerNorm output again (deterministic recompute from the
    same input: bitwise the forward's), one pass."""
    if lnfused.supported(x):
        t = x.shape[0]
        return lnfused.ln_fwd(x, g, b, LN_EPS, torch.empty(t, device=x.device), torch.empty(t, device=x.device))
    return _aten.native_layer_norm(x, [x.shape[-1]], g, b, LN_EPS)[0]


def _ln_bw(dy, x, g, b, mean, rstd, dg, db, addend=None):
    """LayerNorm backward (+ the residual branch's gradient `addend`): the own
    one-pass kernel for bf16 (dgamma/dbeta straight into the fp32 gradient
    region), aten otherwise."""
    if lnfused.supported(x) and dy.dtype == torch.bfloat16 and dg.is_contiguous() and db.is_contiguous():
        return lnfused.ln_bwd(dy, x, g, mean.view(-1), rstd.view(-1), dg, db, addend=addend)
    dx, dgg, dbb = _aten.native_layer_norm_backward(dy, x, [x.shape[-1]], mean.view(-1, 1), rstd.view(-1, 1),
                                                    g, b, [True, True, True])
    dg.copy_(dgg)
    db.copy_(dbb)
    return dx if addend is None else dx + addend


def _gemm_cost(m, n, k, es=2):
    return (m * k + n * k + m * n) * es, 2.0 * m * n * k


def _linear(x, w, b, out=None):
    with bnfused._timed("cublas_gemm", *_gemm_cost(x.shape[0], w.shape[0], x.shape[1], x.element_size())):
        return torch.addmm(b, x, w.t(), out=out) if out is not None else torch.addmm(b, x, w.t())


def _mm_f32_into(a, b, out):
    """out (fp32) = a @ b: cuBLAS writes fp32 straight into the gradient region."""
    with bnfused._timed("cublas_gemm", *_gemm_cost(a.shape[0], b.shape[1], a.shape[1], a.element_size())):
        _mm_f32_into_raw(a, b, out)


def _mm_f32_into_raw(a, b, out):
    if a.dtype == torch.float32:
        torch.mm(a, b, out=out)
    elif a.is_cuda:
        torch.mm(a, b, out_dtype=torch.float32, out=out)
    else:
        out.copy_(torch.mm(a, b).float())


def _linear_bw(dy, x, w, gw, gb, need_dx=True):
    """y = x W^T + b: writes fp32 dW, db (gb None: already written); returns dx.
    KRT_LINEAR_BGRAD=1: dW and db from one cuBLASLt GEMM (BGRADB epilogue)."""
    if gb is None or not (dy.is_cuda and LINEAR_BGRAD and lnfused.linear_wgrad_bgrad(dy, x, gw, gb)):
        _mm_f32_into(dy.t(), x, gw)
        if gb is not None:
            torch.sum(dy, 0, dtype=torch.float32, out=gb)   # fp32 accumulation, no fp32 copy of dy
    if not need_dx:
        return None
    with bnfused._timed("cublas_gemm", *_gemm_cost(dy.shape[0], w.shape[1], dy.shape[1], dy.element_size())):
        return torch.mm(dy, w)


class EmbeddingUnit(Unit):
    name = "embedding"

    def __init__(self, vocab, hidden, seq, act_dtype=torch.bfloat16):
        self.v, self.h, self.s, self.act = vocab, hidden, seq, act_dtype

    def param_specs(self):
        return [(self.v, self.h), (self.s, self.h)]

    def saved_specs(self, n):
        return [SavedSpec((n * self.s,), torch.int32)]

    def init_params(self, gen):
        return [torch.randn(self.v, self.h, generator=gen) * 0.02, torch.randn(self.s, self.h, generator=gen) * 0.01]

    def forward(self, tok, params, saved):
        we, wp = params
        t = tok.reshape(-1)
        if saved is not None:
            saved[0].copy_(t)
        n = t.numel() // self.s
        x = we.index_select(0, t.long()).view(n, self.s, self.h) + wp.unsqueeze(0)
        return x.view(-1, self.h)

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        t = saved[0].long()
        grads[0].zero_().index_add_(0, t, dy.float())
        grads[1].copy_(dy.float().view(-1, self.s, self.h).sum(0))
        return None

    def fwd_flops(self, n):
        return 0.0

    def ir_line(self, lid, batch, analytic=False):
        return (f"{lid} ElementWise X={self.s * self.h} elem=2 mem_fwd={self.saved_bytes(batch)} mem_wt=0 "
                f"mem_grad={4 * (self.v + self.s) * self.h}")


class TransformerLayerUnit(Unit):
    name = "decoder_layer"

    def __init__(self, hidden, heads, seq, act_dtype=torch.bfloat16):
        self.h, self.nh, self.s, self.act = hidden, heads, seq, act_dtype
        self.hd = hidden // heads

    def param_specs(self):
        h = self.h
        return [(h,), (h,), (3 * h, h), (3 * h,), (h, h), (h,),
                (h,), (h,), (4 * h, h), (4 * h,), (h, 4 * h), (h,)]

    def _flash(self):
        return self.act in (torch.bfloat16, torch.float16)

    def saved_specs(self, n):
        t, h = n * self.s, self.h
        s = [SavedSpec((t, h), self.act), SavedSpec((t, 3 * h), self.act), SavedSpec((t, h), self.act),
             SavedSpec((t, h), self.act), SavedSpec((t, 4 * h), self.act),
             SavedSpec((4 * t,), torch.float32)]                      # ln1/ln2 mean, rstd
        if self._flash():
            s.append(SavedSpec((n, self.nh, self.s), torch.float32))  # logsumexp
        return s

    def init_params(self, gen):
        h = self.h
        std = 0.02
        return [torch.ones(h), torch.zeros(h), torch.randn(3 * h, h, generator=gen) * std, torch.zeros(3 * h),
                torch.randn(h, h, generator=gen) * std, torch.zeros(h), torch.ones(h), torch.zeros(h),
                torch.randn(4 * h, h, generator=gen) * std, torch.zeros(4 * h),
                torch.randn(h, 4 * h, generator=gen) * std, torch.zeros(h)]

    def _heads(self, qkv):
        n = qkv.shape[0] // self.s
        q, k, v = qkv.view(n, self.s, 3, self.nh, self.hd).unbind(2)
        return [z.transpose(1, 2) for z in (q, k, v)]   # [n, nh, s, hd]

    def _merge(self, o):
        return o.transpose(1, 2).reshape(-1, self.h)

    def _cudnn_attn(self, backward=False):
        # cuDNN's sm100 fused attention (2.2x the forward, 2x the backward of
        # aten's flash kernel at these shapes, scripts/probe_attention.py);
        # its backward is not bitwise repeatable (dQ accumulation order), so
        # deterministic mode (the bitwise out-of-core == in-core tests) runs
        # the flash kernel's deterministic backward instead.  cuDNN's backward
        # takes head dims <= 128 only: Turing-NLG's 152 runs the cuDNN forward
        # (its natural-log logsumexp is the flash backward's softmax statistic)
        # and the flash backward
        return (ATTN_CUDNN and not torch.are_deterministic_algorithms_enabled()
                and (not backward or self.hd <= 128))

    def _unfused_bw(self):
        # head dims cuDNN's fused backward rejects (Turing-NLG's 152): aten's
        # flash backward runs them at ~100 TFLOP/s (sm80 mma.sync kernels);
        # the unfused form puts the five s x s x hd contractions on cuBLAS
        # tensor-core GEMMs (the two fp32-output ones as TF32 on the exactly
        # representable bf16 inputs) and the softmax-gradient middle on one
        # own pass -- opt-in only: the materialised fp32 s x s matrices make
        # it HBM-bound and 2.1x slower than flash at seq 1024.  Not in
        # deterministic mode (the flash backward there).
        return (self.hd > 128 and ATTN_CUDNN and ATTN_UNFUSED_BW and not torch.are_deterministic_algorithms_enabled()
                and self.s % 8 == 0)

    def _attn_bw_unfused(self, dO, q, k, v, O, lse, n, chunk=8):
        """Causal attention backward for [n, nh, s, hd] bf16 views: per chunk
        of sequences S = Q K^T and dP = dO V^T in fp32, P and dS in bf16 from
        one pass of krt_attn_softmax_bwd (lse: the forward's [n, nh, s]), then
        dV = P^T dO, dQ = dS K, dK = dS^T Q (bf16 GEMMs, fp32 accumulation)
        written straight into the [n, s, 3, nh, hd] gradient of qkv."""
        d = torch.empty((n, self.s, 3, self.nh, self.hd), dtype=dO.dtype, device=dO.device)
        dq, dk, dv = (d[:, :, i].transpose(1, 2) for i in range(3))
        scale = 1.0 / math.sqrt(self.hd)
        tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        try:
            for b0 in range(0, n, chunk):
                sl = slice(b0, min(n, b0 + chunk))
                qs, ks, vs, dos = q[sl], k[sl], v[sl], dO[sl]
                dof = dos.float()
                S = torch.matmul(qs.float(), ks.float().transpose(-1, -2))
                dP = torch.matmul(dof, vs.float().transpose(-1, -2))
                D = (dof * O[sl].float()).sum(-1)
                del dof
                P = torch.empty(S.shape, dtype=dO.dtype, device=dO.device)
                dS = torch.empty_like(P)
                lnfused.attn_softmax_bwd(S, dP, lse[sl], D, P, dS, scale)
                del S, dP, D
                dv[sl] = torch.matmul(P.transpose(-1, -2), dos)
                dq[sl] = torch.matmul(dS, ks)
                dk[sl] = torch.matmul(dS.transpose(-1, -2), qs)
                del P, dS
        finally:
            torch.backends.cuda.matmul.allow_tf32 = tf32
        return d.reshape(-1, 3 * self.h)

    def _attn_fw(self, qkv, lse_out):
        q, k, v = self._heads(qkv)
        if self._flash():
            n = qkv.shape[0] // self.s
            cud = self._cudnn_attn()
            with bnfused._timed("cudnn_attn_fwd" if cud else "flash_attn_fwd", 4 * qkv.shape[0] * self.h * qkv.element_size(),
                                2.0 * n * self.nh * self.s * self.s * self.hd):   # causal: half of 4*s^2*hd
                if cud:
                    r = _aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
                else:
                    r = _aten._scaled_dot_product_flash_attention(q, k, v, 0.0, True, False)
            if lse_out is not None:
                lse_out.copy_(r[1].reshape(lse_out.shape))
            return self._merge(r[0])
        p = self._probs(q, k)
        return self._merge(p @ v)

    def _probs(self, q, k):
        sc = (q @ k.transpose(-1, -2)) * (1.0 / math.sqrt(self.hd))
        mask = torch.ones(self.s, self.s, dtype=torch.bool, device=q.device).triu(1)
        return torch.softmax(sc.masked_fill(mask, float("-inf")), dim=-1)

    def _attn_bw(self, do, qkv, o, lse):
        q, k, v = self._heads(qkv)
        n = do.shape[0] // self.s
        dO = do.view(n, self.s, self.nh, self.hd).transpose(1, 2)
        if self._flash() and self._unfused_bw():
            O = o.view(n, self.s, self.nh, self.hd).transpose(1, 2)
            with bnfused._timed("attn_bwd_unfused", 8 * do.shape[0] * self.h * do.element_size(),
                                10.0 * n * self.nh * self.s * self.s * self.hd):   # 5 full s x s x hd GEMMs
                return self._attn_bw_unfused(dO, q, k, v, O, lse, n)
        if self._flash():
            O = o.view(n, self.s, self.nh, self.hd).transpose(1, 2)
            z = torch.zeros((), dtype=torch.int64, device=q.device)
            cud = self._cudnn_attn(backward=True)
            with bnfused._timed("cudnn_attn_bwd" if cud else "flash_attn_bwd", 8 * do.shape[0] * self.h * do.element_size(),
                                5.0 * n * self.nh * self.s * self.s * self.hd):   # causal, 2.5x the forward
                if cud:
                    dq, dk, dv = _aten._scaled_dot_product_cudnn_attention_backward(
                        dO, q, k, v, O, lse.view(n, self.nh, self.s, 1), z, z, None, None, None, self.s, self.s,
                        0.0, True)
                else:
                    dq, dk, dv = _aten._scaled_dot_product_flash_attention_backward(
                        dO, q, k, v, O, lse, None, None, self.s, self.s, 0.0, True, z, z)
        else:
            p = self._probs(q, k)
            dv = p.transpose(-1, -2) @ dO
            dp = dO @ v.transpose(-1, -2)
            ds = p * (dp - (dp * p).sum(-1, keepdim=True)) * (1.0 / math.sqrt(self.hd))
            dq = ds @ k
            dk = ds.transpose(-1, -2) @ q
        d = torch.stack([z.transpose(1, 2) for z in (dq, dk, dv)], dim=2)   # [n, s, 3, nh, hd]
        return d.reshape(-1, 3 * self.h)

    writes_out = True

    def forward(self, x, params, saved, out=None):
        g1, b1, wqkv, bqkv, wo, bo, g2, b2, w1, bf1, w2, bf2 = params
        t = x.shape[0]
        if saved is not None:
            _save_input(saved[0], x)
            st = saved[5]
            m1, r1, m2, r2 = st[:t], st[t:2 * t], st[2 * t:3 * t], st[3 * t:]
        else:
            m1 = r1 = m2 = r2 = None
        sv = (lambda k: None) if saved is None else (lambda k: saved[k])
        h1, _ = _ln_fw(x, g1, b1, m1, r1)
        qkv = _linear(h1, wqkv, bqkv, out=sv(1))          # GEMMs write straight into the saved slots
        del h1
        o = self._attn_fw(qkv, saved[6] if (saved is not None and self._flash()) else None)
        if saved is not None:
            saved[2].copy_(o)
        # x2 = x + attn-proj and LN2(x2) in one kernel; x2 lands in its saved slot
        h2, x2 = _ln_fw(x, g2, b2, m2, r2, residual=_linear(o, wo, bo), x2_out=sv(3))
        if MLP_LT and lnfused.supported(h2):
            f1, gl = lnfused.mlp_fc1_gelu(h2, w1, bf1, f1_out=sv(4))
            del h2
            # y = x2 + gelu(f1) W2^T + b2: the residual add in fc2's epilogue
            return lnfused.mlp_fc2_residual(gl, w2, bf2, x2, out=out)
        else:
            f1 = _linear(h2, w1, bf1, out=sv(4))
            del h2
            mlp = _linear(F.gelu(f1, approximate="tanh"), w2, bf2)
        y = torch.add(x2, mlp, out=out) if out is not None else x2 + mlp
        del mlp
        return y

    def saved_input(self, saved):
        return saved[0]

    def backward(self, dy, params, saved, grads):
        dy = _dense(dy)
        g1, b1, wqkv, bqkv, wo, bo, g2, b2, w1, bf1, w2, bf2 = params
        x, qkv, o, x2, f1, st = saved[:6]
        t = x.shape[0]
        m1, r1, m2, r2 = st[:t], st[t:2 * t], st[2 * t:3 * t], st[3 * t:]
        gl = F.gelu(f1, approximate="tanh")
        if MLP_LT and lnfused.supported(f1):
            # dW2 from the recomputed GELU; the data gradient with GELU's
            # derivative in the GEMM's epilogue (fc1's bias gradient: the fp32
            # column sum with fc1's weight gradient below)
            _linear_bw(dy, gl, w2, grads[10], grads[11], need_dx=False)
            del gl
            df1 = lnfused.mlp_fc2_dgelu(dy, w2, f1)
            gb1 = grads[9]
            dg = None
        else:
            dg = _linear_bw(dy, gl, w2, grads[10], grads[11])
            del gl
        if dg is None:
            pass
        elif lnfused.supported(f1):   # GELU backward + fc1's bias gradient in one pass
            df1 = lnfused.gelu_bwd_colsum(dg, f1, grads[9])
            gb1 = None
        else:
            df1 = _aten.gelu_backward(dg, f1, approximate="tanh")
            gb1 = grads[9]
        del dg
        h2 = _ln_apply(x2, g2, b2, m2, r2)
        dh2 = _linear_bw(df1, h2, w1, grads[8], gb1)
        del df1, h2
        dx2 = _ln_bw(dh2, x2, g2, b2, m2, r2, grads[6], grads[7], addend=dy)
        del dh2
        do = _linear_bw(dx2, o, wo, grads[4], grads[5])
        dqkv = self._attn_bw(do, qkv, o, saved[6] if self._flash() else None)
        del do
        h1 = _ln_apply(x, g1, b1, m1, r1)
        dh1 = _linear_bw(dqkv, h1, wqkv, grads[2], grads[3])
        del dqkv, h1
        return _ln_bw(dh1, x, g1, b1, m1, r1, grads[0], grads[1], addend=dx2)

    def fwd_flops(self, n):
        t = n * self.s
        return 2.0 * t * 12 * self.h * self.h + 2.0 * n * self.nh * self.s * self.s * self.hd  # + causal attn

    def ir_line(self, lid, batch, analytic=False):
        grad = 4 * sum(math.prod(p) for p in self.param_specs())
        return (f"{lid} Conv Wout={self.s} Hout=1 Cin={self.h} Cout={12 * self.h} K=1 elem=2 "
                f"mem_fwd={self.saved_bytes(batch)} mem_wt=0 mem_grad={grad}")


class LMHeadUnit(Unit):
    """final LayerNorm + LM head (untied) -> logits [T, vocab]."""

    name = "lm_head"

    def __init__(self, hidden, vocab, seq, act_dtype=torch.bfloat16):
        self.h, self.v, self.s, self.act = hidden, vocab, seq, act_dtype

    def param_specs(self):
        return [(self.h,), (self.h,), (self.v, self.h)]

    def saved_specs(self, n):
        t = n * self.s
        return [SavedSpec((t, self.h), self.act), SavedSpec((2 * t,), torch.float32)]

    def init_params(self, gen):
        return [torch.ones(self.h), torch.zeros(self.h), torch.randn(self.v, self.h, generator=gen) * 0.02]

    def forward(self, x, params, saved):
        g, b, w = params
        t = x.shape[0]
        if saved is not None:
            saved[0].copy_(x)
            m, r = saved[1][:t], saved[1][t:]
        else:
            m = r = None
        h, _ = _ln_fw(x, g, b, m, r)
        with bnfused._timed("cublas_gemm", *_gemm_cost(h.shape[0], w.shape[0], h.shape[1], h.element_size())):
            return torch.mm(h, w.t())

    def backward(self, dlogits, params, saved, grads):
        g, b, w = params
        x, st = saved
        t = x.shape[0]
        m, r = st[:t], st[t:]
        h = _ln_apply(x, g, b, m, r)
        _mm_f32_into(dlogits.t(), h, grads[2])
        with bnfused._timed("cublas_gemm", *_gemm_cost(dlogits.shape[0], w.shape[1], w.shape[0],
                                                       dlogits.element_size())):
            dh = torch.mm(dlogits, w)
        return _ln_bw(dh, x, g, b, m, r, grads[0], grads[1])

    def fwd_flops(self, n):
        return 2.0 * n * self.s * self.h * self.v

    def ir_line(self, lid, batch, analytic=False):
        return (f"{lid} Conv Wout={self.s} Hout=1 Cin={self.h} Cout={self.v} K=1 elem=2 "
                f"mem_fwd={self.saved_bytes(batch)} mem_wt=0 mem_grad={4 * (2 * self.h + self.v * self.h)}")


def gpt_units(hidden, heads, layers, seq, vocab, act_dtype=torch.bfloat16):
    return ([EmbeddingUnit(vocab, hidden, seq, act_dtype)]
            + [TransformerLayerUnit(hidden, heads, seq, act_dtype) for _ in range(layers)]
            + [LMHeadUnit(hidden, vocab, seq, act_dtype)])


def lm_loss(logits, target, chunk_rows=8192):
    """Next-token cross-entropy over all rows; dlogits in the logits dtype.
    Row chunks keep the fp32 softmax transient small (the full [T, vocab]
    fp32 matrix would be 30 GB at the 2.5B bench shape).  bf16 logits: the
    fused one-pass kernel (csrc/ln_kernels.cu lm_xent), per-row losses
    summed by torch in a fixed order."""
    t = target.reshape(-1)
    n = logits.shape[0]
    if lnfused.supported(logits) and logits.shape[1] <= 65536:
        rl, dl = lnfused.lm_xent(logits, t, 1.0 / n)
        return rl.sum() * (1.0 / n), dl
    dl = torch.empty_like(logits)
    total = torch.zeros((), dtype=torch.float32, device=logits.device)
    inv = 1.0 / n
    for r0 in range(0, n, chunk_rows):
        lf = logits[r0:r0 + chunk_rows].float()
        tc = t[r0:r0 + chunk_rows]
        lse = torch.logsumexp(lf, dim=1)
        total += (lse - lf.gather(1, tc.view(-1, 1)).squeeze(1)).sum()
        p = torch.exp(lf - lse.view(-1, 1))
        p[torch.arange(p.shape[0], device=p.device), tc] -= 1.0
        dl[r0:r0 + chunk_rows] = (p * inv).to(logits.dtype)
    return total * inv, dl
