"""Bottleneck-ResNet units under reference-planner plans (swap + recompute +
input regeneration) vs the CPU fp32 in-core oracle, and out-of-core vs
in-core bitwise on the GPU."""
import pytest
import torch

from oracle import resnet_oracle
from paper_2008_11421_b200 import workloads as W
from paper_2008_11421_b200.executor import ExecConfig, Executor
from paper_2008_11421_b200.units import cross_entropy_loss

pytestmark = pytest.mark.gpu


def batches(rec, iters, seed=0):
    g = torch.Generator().manual_seed(seed)
    m = rec["meta"]
    n, r, k = m["batch"], m["res"], m["classes"]
    xs = [torch.randn(n, 3, r, r, generator=g) for _ in range(iters)]
    ys = [torch.randint(0, k, (n,), generator=g) for _ in range(iters)]
    return xs, ys


def run(rec, plan=None, iters=3, lr=0.1, optimizer="sgd", capacity=None):
    units = W.units_for(rec)
    b = W.bundle_for(rec, plan)
    if capacity:
        b.set_capacity(capacity)
    act = units[0].act
    ex = Executor(units, b, batch=rec["meta"]["batch"], loss_fn=cross_entropy_loss,
                  cfg=ExecConfig(optimizer=optimizer, lr=lr, weight_dtype=act))
    gen = torch.Generator().manual_seed(7)
    init = {i + 1: u.init_params(gen) for i, u in enumerate(units)}
    ex.load_weights(init)
    xs, ys = batches(rec, iters)
    losses = []
    for x, y in zip(xs, ys):
        xd = x.cuda().to(act).contiguous(memory_format=torch.channels_last)
        losses.append(float(ex.step(xd, y.cuda())))
    w = ex.unit_weights()
    stats = ex.stats()
    ex.close()
    return units, init, losses, w, stats


@pytest.fixture(autouse=True)
def strict_fp32():
    old = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32,
           torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    yield
    (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32,
     torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark) = old


@pytest.mark.parametrize("name", ["resnet_small_f32_a", "resnet_small_f32_b"])
def test_resnet_plan_matches_cpu_oracle(name):
    rec = W.load(name)
    assert "F" in rec["plan_string"] and "in" in rec["plan_string"]
    assert any(b["recompute"] for b in rec["plan"]["blocks"])
    units, init, losses, w, stats = run(rec)
    xs, ys = batches(rec, 3)
    ref_losses, ref_w = resnet_oracle.train(units, init, xs, ys, lr=0.1)
    # fp32 tolerance (cuDNN vs CPU conv/BN summation order), stated in DESIGN.md
    torch.testing.assert_close(torch.tensor(losses), torch.tensor(ref_losses), rtol=2e-4, atol=2e-5)
    for k in ref_w:
        for got, ref in zip(w[k], ref_w[k]):
            got = got.cpu().float()   # both in the executor's O-H-W-I layout
            torch.testing.assert_close(got, ref, rtol=2e-3, atol=2e-4)
    assert stats["iter_bytes_d2h"] > 0 and stats["iter_bytes_h2d"] > 0


@pytest.mark.parametrize("name", ["resnet_small_f32_b", "resnet_small_bf16"])
def test_resnet_out_of_core_equals_in_core_bitwise(name):
    rec = W.load(name)
    _, _, l_ooc, w_ooc, s_ooc = run(rec, iters=3)
    _, _, l_inc, w_inc, s_inc = run(rec, plan=W.incore_plan(rec["plan"]), iters=3, capacity=1e12)
    assert s_inc["iter_bytes_h2d"] == 0 and s_ooc["iter_bytes_h2d"] > 0
    assert l_ooc == l_inc
    for k in w_inc:
        for a, b in zip(w_ooc[k], w_inc[k]):
            assert torch.equal(a, b), k


def test_resnet_bf16_fused_tracks_fp32_oracle():
    """bf16 activations/weights through the fused NHWC BN kernels: losses
    follow the fp32 CPU oracle at bf16 tolerance (3%)."""
    rec = W.load("resnet_small_bf16")
    units, init, losses, w, stats = run(rec, iters=3, lr=0.05)
    assert all(u._fused() for u in units[:-1])
    xs, ys = batches(rec, 3)
    ref_losses, ref_w = resnet_oracle.train(units, init, xs, ys, lr=0.05)
    torch.testing.assert_close(torch.tensor(losses), torch.tensor(ref_losses), rtol=3e-2, atol=3e-2)


def test_preact_plan_matches_cpu_oracle():
    rec = W.load("preact29_small_f32")
    assert any(b["recompute"] for b in rec["plan"]["blocks"])
    units, init, losses, w, stats = run(rec)
    xs, ys = batches(rec, 3)
    ref_losses, ref_w = resnet_oracle.train(units, init, xs, ys, lr=0.1)
    torch.testing.assert_close(torch.tensor(losses), torch.tensor(ref_losses), rtol=2e-4, atol=2e-5)
    for k in ref_w:
        for got, ref in zip(w[k], ref_w[k]):
            torch.testing.assert_close(got.cpu().float(), ref, rtol=2e-3, atol=2e-4)


def test_preact_bf16_out_of_core_equals_in_core_and_tracks_oracle():
    rec = W.load("preact29_small_bf16")
    units, init, l_ooc, w_ooc, s_ooc = run(rec, iters=3, lr=0.05)
    _, _, l_inc, w_inc, _ = run(rec, plan=W.incore_plan(rec["plan"]), iters=3, lr=0.05, capacity=1e12)
    assert s_ooc["iter_bytes_h2d"] > 0 and l_ooc == l_inc
    for k in w_inc:
        for a, b in zip(w_ooc[k], w_inc[k]):
            assert torch.equal(a, b), k
    xs, ys = batches(rec, 3)
    ref_losses, _ = resnet_oracle.train(units, init, xs, ys, lr=0.05)
    torch.testing.assert_close(torch.tensor(l_ooc), torch.tensor(ref_losses), rtol=3e-2, atol=3e-2)


def test_resnet_fused_dgrad_path_matches_default(monkeypatch):
    """The optional conv3 dgrad + BN2-reduce GEMM path (KRT_TC_DGRAD=1) trains
    the bf16 ResNet plan to the same losses as the default path, within bf16
    resolution."""
    from paper_2008_11421_b200 import units as U
    rec = W.load("resnet_small_bf16")
    _, _, ref, _, _ = run(rec, iters=2)
    monkeypatch.setattr(U, "TC_DGRAD", True)
    _, _, got, _, _ = run(rec, iters=2)
    for a, b in zip(got, ref):
        assert abs(a - b) <= 2e-2 * abs(b), (got, ref)


def test_preact_gemm_path_matches_cudnn_path(monkeypatch):
    """The pre-activation bottleneck on the tcgen05 GEMM (BN+ReLU prologues,
    statistics and shortcut-add epilogues) trains the bf16 preact plan to the
    cuDNN + separate-BN-kernel losses within bf16 resolution."""
    from paper_2008_11421_b200 import units as U
    rec = W.load("preact29_small_bf16")
    units, _, got, _, _ = run(rec, iters=2, lr=0.05)
    assert all(u._tc1x1() for u in units if isinstance(u, U.PreActBottleneckUnit))
    monkeypatch.setattr(U, "TC_DGRAD_PREACT", False)
    _, _, fwd_only, _, _ = run(rec, iters=2, lr=0.05)
    monkeypatch.setattr(U, "TC_CONV1X1", False)
    _, _, ref, _, _ = run(rec, iters=2, lr=0.05)
    for a, b, c in zip(got, fwd_only, ref):
        assert abs(a - c) <= 2e-2 * abs(c), (got, ref)
        assert abs(b - c) <= 2e-2 * abs(c), (fwd_only, ref)
