"""TEST INFRASTRUCTURE ONLY — torch CPU fp32 in-core reference for the GPT
decoder units (cfg3/cfg4 model family): token + position embedding, pre-LN
decoder layers (causal attention, tanh-GELU MLP), final LN, untied LM head,
next-token cross-entropy.  Rebuilt from the executor's parameter tensors.
Numerics parity vs the reference is unpinned (no tensor code upstream)."""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

EPS = 1e-5


def forward(units, params, tokens, bf16=False):
    """bf16=True rounds (value and gradient) where the executor's bf16 path
    stores a tensor: embeddings, LN outputs, GEMM outputs, attention output,
    GELU output, the residual stream and the logits."""
    from paper_2008_11421_b200.units import EmbeddingUnit, LMHeadUnit, TransformerLayerUnit
    from oracle.resnet_oracle import _rounder
    R = _rounder(bf16)
    h = None
    for k, u in enumerate(units, start=1):
        p = params[k]
        if isinstance(u, EmbeddingUnit):
            h = R(p[0][tokens] + p[1].unsqueeze(0))
        elif isinstance(u, TransformerLayerUnit):
            n, s, d = h.shape
            a = R(F.layer_norm(h, [d], p[0], p[1], EPS))
            qkv = R(a @ p[2].t() + p[3])
            q, kk, v = qkv.view(n, s, 3, u.nh, u.hd).unbind(2)
            q, kk, v = (z.transpose(1, 2) for z in (q, kk, v))
            sc = (q @ kk.transpose(-1, -2)) / math.sqrt(u.hd)
            sc = sc.masked_fill(torch.ones(s, s, dtype=torch.bool).triu(1), float("-inf"))
            o = R((torch.softmax(sc, -1) @ v).transpose(1, 2).reshape(n, s, d))
            h = R(h + R(o @ p[4].t() + p[5]))
            m = R(F.layer_norm(h, [d], p[6], p[7], EPS))
            f = R(F.gelu(R(m @ p[8].t() + p[9]), approximate="tanh"))
            h = R(h + R(f @ p[10].t() + p[11]))
        elif isinstance(u, LMHeadUnit):
            h = R(R(F.layer_norm(h, [h.shape[-1]], p[0], p[1], EPS)) @ p[2].t())
        else:
            raise TypeError(type(u))
    return h


def train(units, init, inputs, targets, lr=0.1, optimizer="sgd", bf16=False):
    params = {k: [t.detach().clone().float().requires_grad_(True) for t in ts] for k, ts in init.items()}
    flat = [t for k in sorted(params) for t in params[k]]
    opt = (torch.optim.SGD(flat, lr=lr, foreach=False) if optimizer == "sgd"
           else torch.optim.Adam(flat, lr=lr, foreach=False))
    losses = []
    for x, y in zip(inputs, targets):
        opt.zero_grad(set_to_none=True)
        logits = forward(units, params, x, bf16)
        loss = F.cross_entropy(logits.reshape(-1, logits.shape[-1]), y.reshape(-1))
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    return losses, {k: [t.detach() for t in ts] for k, ts in params.items()}


def gradients(units, init, x, y, bf16=False):
    """One in-core fp32 forward/backward: (loss, {unit: [grad per param]})."""
    params = {k: [t.detach().clone().float().requires_grad_(True) for t in ts] for k, ts in init.items()}
    logits = forward(units, params, x, bf16)
    loss = F.cross_entropy(logits.reshape(-1, logits.shape[-1]), y.reshape(-1))
    loss.backward()
    return float(loss.detach()), {k: [t.grad.detach().clone() for t in ts] for k, ts in params.items()}
