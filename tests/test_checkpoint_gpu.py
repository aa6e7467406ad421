"""Checkpoint / restart of the executor's training state (krt_checkpoint_save /
krt_checkpoint_load): a run interrupted after
k steps and restored into a fresh context continues bitwise like the
uninterrupted run — losses and every weight."""

import pytest
import torch

from oracle import fc_chain_oracle as orc
from paper_2008_11421_b200 import _lib
from paper_2008_11421_b200 import workloads as W
from paper_2008_11421_b200.executor import ExecConfig, Executor
from paper_2008_11421_b200.plan import PlanBundle
from paper_2008_11421_b200.units import FCUnit, cross_entropy_loss, mse_zero_loss

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def deterministic_cudnn():
    old = (torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark)
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    yield
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = old


def fc_executor(sched_cases, optimizer):
    c = next(x for x in sched_cases if x["name"] == "cfg0_fc_chain")
    bundle = PlanBundle(c["model"], c["hardware"], c["plan"])
    ex = Executor([FCUnit(64, 64) for _ in range(6)], bundle, batch=2, loss_fn=mse_zero_loss,
                  cfg=ExecConfig(optimizer=optimizer, lr=1e-3 if optimizer == "adam" else 1e-2))
    ex.load_weights({i + 1: [torch.from_numpy(w)] for i, w in enumerate(orc.init_weights())})
    return ex


def fc_steps(ex, first, last):
    return [float(ex.step(torch.from_numpy(orc.inputs(0, it)).cuda())) for it in range(first, last + 1)]


def weights(ex):
    w = ex.unit_weights()
    return {k: [t.cpu().clone() for t in v] for k, v in w.items()}


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_fc_chain_checkpoint_resumes_bitwise(sched_cases, tmp_path, optimizer):
    """cfg0 golden plan (swapped blocks on the host path, recompute): 5 steps
    straight vs 3 steps + checkpoint + restore in a new context + 2 steps."""
    ex = fc_executor(sched_cases, optimizer)
    ref_losses = fc_steps(ex, 1, 5)
    ref_w = weights(ex)
    ex.close()

    ex = fc_executor(sched_cases, optimizer)
    head = fc_steps(ex, 1, 3)
    ex.synchronize()
    ck = tmp_path / "cfg0.krt"
    ex.save_checkpoint(ck)
    ex.close()

    ex = fc_executor(sched_cases, optimizer)   # fresh context, initial weights
    ex.load_checkpoint(ck)
    tail = fc_steps(ex, 4, 5)
    got_w = weights(ex)
    ex.close()
    assert head + tail == ref_losses
    for k in ref_w:
        for a, b in zip(ref_w[k], got_w[k]):
            assert torch.equal(a, b), k


def test_checkpoint_rejects_foreign_files(sched_cases, tmp_path):
    ex = fc_executor(sched_cases, "adam")
    bad = tmp_path / "bad.krt"
    bad.write_bytes(b"not a checkpoint at all" * 8)
    with pytest.raises(_lib.KrtError) as e:
        ex.load_checkpoint(bad)
    assert e.value.code == _lib.KRT_USAGE
    with pytest.raises(_lib.KrtError):
        ex.load_checkpoint(tmp_path / "missing.krt")
    ex.close()


def test_resnet_checkpoint_resumes_bitwise(tmp_path):
    """bf16 bottleneck ResNet under a swap + recompute plan (device-path and
    host-path blocks, SGD with momentum): 4 straight vs 2 + restore + 2."""
    rec = W.load("resnet_small_bf16")
    g = torch.Generator().manual_seed(0)
    m = rec["meta"]
    xs = [torch.randn(m["batch"], 3, m["res"], m["res"], generator=g) for _ in range(4)]
    ys = [torch.randint(0, m["classes"], (m["batch"],), generator=g) for _ in range(4)]

    def make():
        units = W.units_for(rec)
        ex = Executor(units, W.bundle_for(rec), batch=m["batch"], loss_fn=cross_entropy_loss,
                      cfg=ExecConfig(optimizer="sgd", lr=0.05, momentum=0.9, weight_dtype=units[0].act))
        gen = torch.Generator().manual_seed(7)
        ex.load_weights({i + 1: u.init_params(gen) for i, u in enumerate(units)})
        return ex, units[0].act

    def steps(ex, act, idx):
        return [float(ex.step(xs[i].cuda().to(act).contiguous(memory_format=torch.channels_last), ys[i].cuda()))
                for i in idx]

    ex, act = make()
    ref = steps(ex, act, range(4))
    ref_w = weights(ex)
    ex.close()

    ex, act = make()
    head = steps(ex, act, range(2))
    ex.synchronize()
    ex.save_checkpoint(tmp_path / "r.krt")
    ex.close()
    ex, act = make()
    ex.load_checkpoint(tmp_path / "r.krt")
    tail = steps(ex, act, range(2, 4))
    got_w = weights(ex)
    ex.close()
    assert head + tail == ref
    for k in ref_w:
        for a, b in zip(ref_w[k], got_w[k]):
            assert torch.equal(a, b), k
