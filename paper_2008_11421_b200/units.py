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
from typing import Optional

import torch
import torch.nn.functional as F

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
