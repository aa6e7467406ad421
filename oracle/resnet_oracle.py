"""TEST INFRASTRUCTURE ONLY — torch CPU fp32 in-core reference for the
bottleneck-ResNet units (cfg1/cfg2 model family).

A plain autograd model (conv / batch-stat BatchNorm / ReLU / residual add,
stride on the 3x3 conv) (post-activation ImageNet bottleneck and the pre-activation CIFAR bottleneck of
ResNet-1001) rebuilt from the same parameter tensors the executor
holds (its conv weights are stored O-H-W-I; converted here to O-I-H-W).  The
reference has no tensor code (numerics parity unpinned); this is
the in-core result the out-of-core executor must reproduce.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

EPS = 1e-5


class _RoundBf16(torch.autograd.Function):
    """bf16 storage point of the product path: the value is rounded to bf16 on
    the way forward and its gradient on the way back (both are bf16 tensors
    in the executor)."""

    @staticmethod
    def forward(ctx, x):
        return x.to(torch.bfloat16).float()

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).float()


def _rounder(bf16):
    return _RoundBf16.apply if bf16 else (lambda t: t)


def _w(t):
    return t.permute(0, 3, 1, 2).contiguous() if t.dim() == 4 else t


def _bn(x, g, b):
    return F.batch_norm(x, None, None, g, b, training=True, momentum=0.0, eps=EPS)


def forward(units, params, x, bf16=False):
    """params: unit index (1-based) -> list of fp32 CPU tensors requiring grad.
    bf16=True rounds (value and gradient) at the points where the executor's
    bf16 path stores a tensor: conv outputs, BN+ReLU activations, unit outputs."""
    R = _rounder(bf16)
    from paper_2008_11421_b200.units import (BottleneckUnit, CifarStemUnit, HeadUnit,
                                             PreActBottleneckUnit, PreActHeadUnit, StemUnit)
    h = x
    for k, u in enumerate(units, start=1):
        p = params[k]
        if isinstance(u, StemUnit):
            h = R(F.conv2d(h, _w(p[0]), stride=2, padding=3))
            h = F.relu(_bn(h, p[1], p[2]))
            h = R(F.max_pool2d(h, 3, 2, 1))
        elif isinstance(u, BottleneckUnit):
            o = R(F.relu(_bn(R(F.conv2d(h, _w(p[0]))), p[1], p[2])))
            o = R(F.relu(_bn(R(F.conv2d(o, _w(p[3]), stride=u.s, padding=1)), p[4], p[5])))
            o = _bn(R(F.conv2d(o, _w(p[6]))), p[7], p[8])
            idn = _bn(R(F.conv2d(h, _w(p[9]), stride=u.s)), p[10], p[11]) if u.down else h
            h = R(F.relu(o + idn))
        elif isinstance(u, HeadUnit):
            h = h.mean(dim=(2, 3)) @ p[0].t() + p[1]
        elif isinstance(u, CifarStemUnit):
            h = R(F.conv2d(h, _w(p[0]), padding=1))
        elif isinstance(u, PreActBottleneckUnit):
            a0 = R(F.relu(_bn(h, p[0], p[1])))
            o = R(F.conv2d(a0, _w(p[2])))
            o = R(F.conv2d(R(F.relu(_bn(o, p[3], p[4]))), _w(p[5]), stride=u.s, padding=1))
            o = F.conv2d(R(F.relu(_bn(o, p[6], p[7]))), _w(p[8]))
            h = R(o + (R(F.conv2d(a0, _w(p[9]), stride=u.s)) if u.down else h))
        elif isinstance(u, PreActHeadUnit):
            h = F.relu(_bn(h, p[0], p[1])).mean(dim=(2, 3)) @ p[2].t() + p[3]
        else:
            raise TypeError(type(u))
    return h


def train(units, init, inputs, targets, lr=0.1, optimizer="sgd", bf16=False):
    """In-core fp32 training: returns (losses, final params)."""
    params = {k: [t.detach().clone().float().requires_grad_(True) for t in ts] for k, ts in init.items()}
    flat = [t for k in sorted(params) for t in params[k]]
    opt = (torch.optim.SGD(flat, lr=lr, foreach=False) if optimizer == "sgd"
           else torch.optim.Adam(flat, lr=lr, foreach=False))
    losses = []
    for x, y in zip(inputs, targets):
        opt.zero_grad(set_to_none=True)
        loss = F.cross_entropy(forward(units, params, x.float(), bf16), y)
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    return losses, {k: [t.detach() for t in ts] for k, ts in params.items()}


def gradients(units, init, x, y, bf16=False):
    """One in-core fp32 forward/backward: (loss, {unit: [grad per param]})."""
    params = {k: [t.detach().clone().float().requires_grad_(True) for t in ts] for k, ts in init.items()}
    loss = F.cross_entropy(forward(units, params, x.float(), bf16), y)
    loss.backward()
    return float(loss.detach()), {k: [t.grad.detach().clone() for t in ts] for k, ts in params.items()}
