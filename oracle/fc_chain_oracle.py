"""TEST INFRASTRUCTURE ONLY — numpy fp32 in-core data-parallel training of the
reference's small synthetic model (cfg0).

cfg0 (SURVEY §8d / BASELINE.json configs[0]): ``zoo.fc_chain_model(6, 64,
batch 2)`` (zoo.py:57-63 — six bias-free FullyConnected 64->64 layers, batch
2 per worker) trained data-parallel on P workers with the gradient exchange
the paper's pipeline performs (all-reduce mean) and the
host-side update.  No reference code computes tensors, so
numerics parity is UNPINNED against the reference; this oracle is the
in-core result the out-of-core executor must reproduce ("no impact on
accuracy").

Update rules follow torch.optim.SGD / torch.optim.Adam (single-tensor path)
in float32: Adam m <- lerp(m, g, 1-b1); v <- v*b2 + (1-b2) g g;
p <- p - lr/(1-b1^t) * m / (sqrt(v)/sqrt(1-b2^t) + eps).
"""
from __future__ import annotations

import numpy as np

F = np.float32


def inputs(rank: int, it: int, batch: int = 2, features: int = 64) -> np.ndarray:
    """Synthetic N(0,1) input of worker ``rank`` at iteration ``it`` (1-based)."""
    return np.random.RandomState(1000 * rank + it).standard_normal((batch, features)).astype(F)


def init_weights(layers: int = 6, features: int = 64, seed: int = 0) -> list[np.ndarray]:
    rs = np.random.RandomState(seed)
    b = 1.0 / np.sqrt(features)
    return [rs.uniform(-b, b, (features, features)).astype(F) for _ in range(layers)]


def forward_backward(ws, x):
    """MSE-to-zero loss and per-layer weight gradients of y = x W1^T ... W6^T."""
    acts = [x]
    for w in ws:
        acts.append(acts[-1] @ w.T)
    y = acts[-1]
    loss = F(np.mean(y.astype(np.float64) ** 2))
    dy = (y * F(2.0 / y.size)).astype(F)
    grads = [None] * len(ws)
    for i in range(len(ws) - 1, -1, -1):
        grads[i] = (dy.T @ acts[i]).astype(F)
        dy = (dy @ ws[i]).astype(F)
    return loss, grads


class Optim:
    def __init__(self, kind, lr, b1=0.9, b2=0.999, eps=1e-8):
        self.kind, self.lr, self.b1, self.b2, self.eps = kind, lr, b1, b2, eps
        self.t = 0
        self.m = self.v = None

    def step(self, ws, grads):
        self.t += 1
        if self.kind == "sgd":
            return [(w + F(-self.lr) * g).astype(F) for w, g in zip(ws, grads)]
        if self.m is None:
            self.m = [np.zeros_like(w) for w in ws]
            self.v = [np.zeros_like(w) for w in ws]
        bc1 = 1.0 - self.b1 ** self.t
        bc2s = F(np.sqrt(1.0 - self.b2 ** self.t))
        out = []
        for i, (w, g) in enumerate(zip(ws, grads)):
            wgt = F(1.0 - self.b1)
            self.m[i] = (self.m[i] + wgt * (g - self.m[i])).astype(F)
            self.v[i] = (self.v[i] * F(self.b2) + (F(1.0 - self.b2) * g) * g).astype(F)
            denom = (np.sqrt(self.v[i]) / bc2s + F(self.eps)).astype(F)
            out.append((w + F(-self.lr / bc1) * (self.m[i] / denom)).astype(F))
        return out


def train(workers: int = 2, iterations: int = 3, optimizer: str = "sgd", lr: float = 1e-2,
          batch: int = 2, layers: int = 6, features: int = 64, weights=None):
    """In-core DP reference: returns (losses[it][rank], final weights)."""
    ws = [w.copy() for w in (weights if weights is not None else init_weights(layers, features))]
    opt = Optim(optimizer, lr)
    losses = []
    for it in range(1, iterations + 1):
        per = [forward_backward(ws, inputs(r, it, batch, features)) for r in range(workers)]
        losses.append([p[0] for p in per])
        grads = []
        for i in range(len(ws)):
            acc = per[0][1][i].copy()
            for r in range(1, workers):
                acc = (acc + per[r][1][i]).astype(F)
            grads.append((acc * F(1.0 / workers)).astype(F))
        ws = opt.step(ws, grads)
    return losses, ws
