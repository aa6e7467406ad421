"""Parity of the bf16 product path (own fused kernels on: tcgen05 1x1 GEMM
with BN prologue/statistics/residual epilogues, fused BN/ReLU/add kernels, LN
and GELU kernels) against fp32 autograd on the SAME bf16-rounded inputs and
weights (oracle/, CPU), run twice: plain fp32 ("fp32 oracle") and with the
product's bf16 storage points emulated (value and gradient rounded to bf16
where the executor stores a bf16 tensor: "bf16 oracle").

Tolerances, relative L2 error ||got - ref|| / ||ref||:
* unit level (real widths), every tensor (output, dX, every dW, dgamma,
  dbeta): within BF16_UNIT = 3e-2 of the bf16 oracle, and no further from the
  fp32 oracle than 1.5x the bf16 oracle's own distance from it + 5e-3.
  Measured: 0.2-2.8% from the bf16 oracle; the bf16 oracle itself sits 3-9%
  from fp32 on these random-gradient probes (a ReLU mask flip at 0.1% of the
  elements moves a sum of random terms by sqrt(0.1%) ~ 3%).
* step level (the full-model gradient recovered from one plain-SGD step with
  lr = 1 from the fp32 masters, g = w0 - w1, through the out-of-core plan):
  the small parity models at random init are ill-conditioned in bf16 (batch
  statistics over 32 values at 2x2 spatial): an independent bf16
  implementation (the bf16 oracle) lands 25-75% from fp32.  The bar is that
  the product is no further from fp32 than that: median over tensors of the
  product's fp32 distance <= 1.2x the bf16 oracle's median + 1e-2.  The GPT
  model is well conditioned and is held per tensor to BF16_STEP = 3e-2 of the
  bf16 oracle.
* Adam with the host path on every block (the GPT bench configuration,
  host_path_all), 3 steps: cosine of each tensor's update w3 - w0 with the
  fp32 oracle's, averaged over tensors, >= the bf16 oracle's average - 0.03.
  Adam takes an lr-sized step on every element whatever its gradient's size,
  so elements whose gradient is structurally zero (e.g. the key third of the
  QKV bias) or within bf16 noise of zero move in random directions in any
  bf16 implementation.
"""
import math

import pytest
import torch

from oracle import gpt_oracle, resnet_oracle
from paper_2008_11421_b200 import workloads as W
from paper_2008_11421_b200.executor import ExecConfig, Executor
from paper_2008_11421_b200.units import (BottleneckUnit, GradPair, PreActBottleneckUnit, _cl,
                                         cross_entropy_loss, lm_loss)

pytestmark = pytest.mark.gpu

BF16_UNIT = 3e-2
BF16_STEP = 3e-2


def rel_l2(got, ref):
    got, ref = got.double().cpu(), ref.double().cpu()
    d = (got - ref).norm().item()
    n = ref.norm().item()
    return d / n if n > 0 else d


@pytest.fixture(autouse=True)
def strict_fp32():
    old = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = old


def unit_params(u, gen):
    """bf16-representable parameters with random (non-trivial) BN affine."""
    ps = []
    for shp in u.param_specs():
        if len(shp) == 4:
            fan = shp[1] * shp[2] * shp[3]
            t = torch.randn(shp, generator=gen) * math.sqrt(2.0 / fan)
        elif len(ps) and len(u.param_specs()[len(ps) - 1]) != 1:
            t = 1.0 + 0.2 * torch.randn(shp, generator=gen)   # gamma follows a weight
        else:
            t = 0.2 * torch.randn(shp, generator=gen)
        ps.append(t.to(torch.bfloat16).float())
    if isinstance(u, PreActBottleneckUnit):   # (g0, b0) lead the list
        ps[0] = (1.0 + 0.2 * torch.randn(u.cin, generator=gen)).to(torch.bfloat16).float()
    return ps


def run_unit(u, n, seed):
    gen = torch.Generator().manual_seed(seed)
    params = unit_params(u, gen)
    x = torch.randn(n, u.hi, u.hi, u.cin, generator=gen).to(torch.bfloat16)
    dy = torch.randn(n, u.ho, u.ho, u.cout, generator=gen).to(torch.bfloat16)
    dev = torch.device("cuda")
    pd = [p.to(dev, torch.bfloat16) for p in params]
    saved = [torch.zeros(s.shape, dtype=s.dtype, device=dev) for s in u.saved_specs(n)]
    grads = [torch.zeros(p.shape, dtype=torch.float32, device=dev) for p in params]
    xd = _cl(x.to(dev))
    y = u.forward(xd, pd, saved)
    g = u.backward(_cl(dy.to(dev)), pd, saved, grads)
    if isinstance(g, GradPair):
        g = g[0].float() + g[1].float()
    torch.cuda.synchronize()
    got = {"y": y.float(), "dx": g.float()}
    got.update({f"p{k}": gd for k, gd in enumerate(grads)})
    ref = {}
    for bf16 in (False, True):
        # oracle: fp32 autograd on the same bf16 values, without / with the
        # product's bf16 storage points
        op = {1: [p.clone().requires_grad_(True) for p in params]}
        xr = x.permute(0, 3, 1, 2).float().requires_grad_(True)
        yr = resnet_oracle.forward([u], op, xr, bf16=bf16)
        yr.backward(dy.permute(0, 3, 1, 2).float())
        r = {"y": yr.detach(), "dx": xr.grad}
        r.update({f"p{k}": p.grad for k, p in enumerate(op[1])})
        ref[bf16] = r
    return {k: (rel_l2(got[k], ref[True][k]), rel_l2(got[k], ref[False][k]), rel_l2(ref[True][k], ref[False][k]))
            for k in got}


def check_unit(kind, shape, err):
    """err[t] = (product vs bf16-storage oracle, product vs fp32 oracle,
    bf16-storage oracle vs fp32 oracle)."""
    print(kind, shape, {k: "/".join(f"{x:.1e}" for x in v) for k, v in err.items()})
    bad = {k: v for k, v in err.items() if not (v[0] <= BF16_UNIT and v[1] <= 1.5 * v[2] + 5e-3)}
    assert not bad, bad


# real ResNet-200 widths (64 -> 2048 output channels), every unit shape class:
# (cin, width, stride, side_in, batch)
BOTTLENECK = [(64, 64, 1, 56, 4),      # stage 1 first unit: projection shortcut
              (256, 64, 1, 56, 4),     # stage 1 identity
              (256, 128, 2, 56, 4),    # stage 2 first: strided projection
              (512, 128, 1, 28, 4),
              (1024, 256, 1, 14, 8),
              (1024, 512, 2, 14, 8),
              (2048, 512, 1, 7, 16)]
# ResNet-1001 pre-activation widths (16 -> 256 output channels)
PREACT = [(16, 16, 1, 64, 4), (64, 16, 1, 64, 4), (64, 32, 2, 64, 4), (128, 32, 1, 32, 4),
          (128, 64, 2, 32, 4), (256, 64, 1, 16, 8)]


@pytest.mark.parametrize("cin,w,s,side,n", BOTTLENECK)
def test_bottleneck_unit_gradients_bf16(cin, w, s, side, n):
    u = BottleneckUnit(cin, w, s, side)
    assert u._fused() and u._tc1x1(), "the own fused kernels must be on"
    check_unit("bottleneck", (cin, w, s, side, n), run_unit(u, n, seed=cin + w + s))


@pytest.mark.parametrize("cin,w,s,side,n", PREACT)
def test_preact_unit_gradients_bf16(cin, w, s, side, n):
    u = PreActBottleneckUnit(cin, w, s, side)
    assert u._tc1x1(), "the own fused kernels must be on"
    check_unit("preact", (cin, w, s, side, n), run_unit(u, n, seed=cin + w + s))


# ---------------------------------------------------------------- step level
def _inputs(rec, iters, seed=0):
    g = torch.Generator().manual_seed(seed)
    m = rec["meta"]
    if m["family"] == "gpt":
        xs = [torch.randint(0, m["vocab"], (m["batch"], m["seq"]), generator=g) for _ in range(iters)]
        ys = [torch.randint(0, m["vocab"], (m["batch"], m["seq"]), generator=g) for _ in range(iters)]
    else:
        n, r, k = m["batch"], m["res"], m["classes"]
        xs = [torch.randn(n, 3, r, r, generator=g).to(torch.bfloat16).float() for _ in range(iters)]
        ys = [torch.randint(0, k, (n,), generator=g) for _ in range(iters)]
    return xs, ys


def _executor(rec, **cfg):
    units = W.units_for(rec)
    gpt = rec["meta"]["family"] == "gpt"
    ex = Executor(units, W.bundle_for(rec), batch=rec["meta"]["batch"],
                  loss_fn=lm_loss if gpt else cross_entropy_loss,
                  cfg=ExecConfig(weight_dtype=torch.bfloat16, **cfg))
    gen = torch.Generator().manual_seed(11)
    init = {i + 1: [t.to(torch.bfloat16).float() for t in u.init_params(gen)] for i, u in enumerate(units)}
    if not gpt:   # non-zero residual-branch gammas so every gradient is exercised
        for i, u in enumerate(units):
            if isinstance(u, BottleneckUnit):
                init[i + 1][7] = torch.full_like(init[i + 1][7], 0.5)
    ex.load_weights(init)
    return units, ex, init


def _step(ex, rec, x, y):
    if rec["meta"]["family"] == "gpt":
        return float(ex.step(x.cuda().int(), y.cuda()))
    return float(ex.step(x.cuda().to(torch.bfloat16).contiguous(memory_format=torch.channels_last), y.cuda()))


def _masters(ex, units):
    """fp32 master weights per unit (host or device optimizer state)."""
    out = {}
    for b, lo, hi in ex.blocks:
        flat = ex.master(b)
        o = 0
        for ui in range(lo, hi + 1):
            ts = []
            for shp in units[ui - 1].param_specs():
                k = math.prod(shp)
                ts.append(flat[o:o + k].view(shp).clone())
                o += k
            out[ui] = ts
    return out


@pytest.mark.parametrize("name", ["resnet_small_bf16", "preact29_small_bf16", "gpt_small_bf16"])
def test_step_gradients_bf16_out_of_core(name):
    """One plain SGD step, lr = 1: w0 - w1 is the whole model's gradient as the
    out-of-core bf16 product path computed it (swap, recompute, regeneration)."""
    rec = W.load(name)
    assert "in" in rec["plan_string"]   # the plan swaps
    units, ex, init = _executor(rec, optimizer="sgd", lr=1.0)
    xs, ys = _inputs(rec, 1)
    w0 = _masters(ex, units)
    loss = _step(ex, rec, xs[0], ys[0])
    ex.synchronize()
    w1 = _masters(ex, units)
    st = ex.stats()
    ex.close()
    assert st["iter_bytes_h2d"] > 0
    orc = gpt_oracle if rec["meta"]["family"] == "gpt" else resnet_oracle
    ref_loss, ref32 = orc.gradients(units, init, xs[0], ys[0])
    _, ref16 = orc.gradients(units, init, xs[0], ys[0], bf16=True)
    assert abs(loss - ref_loss) <= 1e-2 * abs(ref_loss)
    bad, rows = [], []
    for ui in ref32:
        for k, (a, b, r32, r16) in enumerate(zip(w0[ui], w1[ui], ref32[ui], ref16[ui])):
            if r32.norm() == 0:
                continue
            g = a - b
            e = (rel_l2(g, r16), rel_l2(g, r32), rel_l2(r16, r32))
            rows.append((ui, k, e))
            if rec["meta"]["family"] == "gpt" and not e[0] <= BF16_STEP:
                bad.append((ui, k, e))
    print(name, "step gradients (vs bf16 oracle / vs fp32 / bf16 oracle vs fp32):",
          " ".join(f"{ui}.{k}={e[0]:.1e}/{e[1]:.1e}/{e[2]:.1e}" for ui, k, e in rows))
    med = lambda v: sorted(v)[len(v) // 2]   # noqa: E731
    m32, minh = med([e[1] for _, _, e in rows]), med([e[2] for _, _, e in rows])
    print(name, f"median vs fp32 {m32:.3e}, bf16 oracle median vs fp32 {minh:.3e}")
    assert m32 <= 1.2 * minh + 1e-2, (m32, minh)
    assert not bad, bad


@pytest.mark.parametrize("name", ["resnet_small_bf16", "preact29_small_bf16", "gpt_small_bf16"])
def test_adam_host_path_all_updates_bf16(name):
    """Adam on the host for every block (host_path_all), 3 steps: updated fp32
    masters vs the oracle's torch.optim.Adam on the same inputs."""
    rec = W.load(name)
    lr = 1e-3
    units, ex, init = _executor(rec, optimizer="adam", lr=lr, host_path_all=True)
    xs, ys = _inputs(rec, 3)
    losses = [_step(ex, rec, x, y) for x, y in zip(xs, ys)]
    ex.synchronize()
    got = _masters(ex, units)
    st = ex.stats()
    ex.close()
    assert st["iter_bytes_d2h"] > 0
    orc = gpt_oracle if rec["meta"]["family"] == "gpt" else resnet_oracle
    ref_losses, ref32 = orc.train(units, init, xs, ys, lr=lr, optimizer="adam")
    _, ref16 = orc.train(units, init, xs, ys, lr=lr, optimizer="adam", bf16=True)
    torch.testing.assert_close(torch.tensor(losses), torch.tensor(ref_losses), rtol=2e-2, atol=2e-2)

    def cos(a, b):
        a, b = a.double().flatten(), b.double().flatten()
        return float(a @ b / (a.norm() * b.norm() + 1e-30))

    rows = []
    for ui in ref32:
        for k, (g, r32, r16, w0) in enumerate(zip(got[ui], ref32[ui], ref16[ui], init[ui])):
            if (r32 - w0).norm() == 0:
                continue
            c = (cos(g - w0, r16 - w0), cos(g - w0, r32 - w0), cos(r16 - w0, r32 - w0))
            rows.append((ui, k, c))
    print(name, "Adam update cosines (vs bf16 oracle / vs fp32 / bf16 oracle vs fp32):",
          " ".join(f"{ui}.{k}={c[0]:.3f}/{c[1]:.3f}/{c[2]:.3f}" for ui, k, c in rows))
    c32 = sum(c[1] for _, _, c in rows) / len(rows)
    cinh = sum(c[2] for _, _, c in rows) / len(rows)
    print(name, f"mean update cosine vs fp32 {c32:.4f}, bf16 oracle vs fp32 {cinh:.4f}")
    assert c32 >= cinh - 0.03, (c32, cinh)
