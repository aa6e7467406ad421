"""Gradient ring (krt_config.grad_slots): R group-sized gradient slots instead
of a whole-model fp32 gradient region, each held from the group's first
backward until its exchange / grad_out / device update consumed it (the
reference holds a block's grad bytes only until grad_out, distsim.py:195-202).
The ring changes where gradients live, never what is computed: every run must
be bitwise identical to the whole-model region."""
import numpy as np
import pytest
import torch

from oracle import fc_chain_oracle as orc
from paper_2008_11421_b200 import workloads as W
from paper_2008_11421_b200.executor import ExecConfig, Executor
from paper_2008_11421_b200.plan import PlanBundle
from paper_2008_11421_b200.units import FCUnit, cross_entropy_loss, lm_loss, mse_zero_loss

pytestmark = pytest.mark.gpu


def run_fc(sched_cases, slots, **cfg):
    c = next(c for c in sched_cases if c["name"] == "cfg0_fc_chain")
    ex = Executor([FCUnit(64, 64) for _ in range(6)], PlanBundle(c["model"], c["hardware"], c["plan"]), batch=2,
                  loss_fn=mse_zero_loss, cfg=ExecConfig(grad_slots=slots, **cfg))
    ex.load_weights({i + 1: [torch.from_numpy(w)] for i, w in enumerate(orc.init_weights())})
    losses = [float(ex.step(torch.from_numpy(orc.inputs(0, it)).cuda())) for it in range(1, 5)]
    w = ex.unit_weights()
    st = ex.stats()
    ex.close()
    return losses, [w[i + 1][0].cpu().numpy() for i in range(6)], st


@pytest.mark.parametrize("slots", [1, 2, 3])
@pytest.mark.parametrize("cfg", [dict(optimizer="sgd", lr=1e-2), dict(optimizer="adam", lr=1e-3),
                                 dict(optimizer="adam", lr=1e-3, host_path_all=True),
                                 dict(optimizer="sgd", lr=1e-2, force_dp_path=True),
                                 dict(optimizer="adam", lr=1e-3, force_dp_path=True, dist_groups=4)])
def test_fc_ring_is_bitwise_the_full_region(sched_cases, slots, cfg):
    l0, w0, s0 = run_fc(sched_cases, 0, **cfg)
    l1, w1, s1 = run_fc(sched_cases, slots, **cfg)
    assert l0 == l1
    for a, b in zip(w0, w1):
        assert np.array_equal(a, b)
    # the ring is used only where it is smaller than the whole-model region
    assert s1["grad_region_bytes"] <= s0["grad_region_bytes"]
    assert (s1["grad_slots"] == slots) == (s1["grad_region_bytes"] < s0["grad_region_bytes"])


@pytest.mark.parametrize("name,slots", [("gpt_small_bf16", 2), ("resnet_small_bf16", 2), ("preact29_small_bf16", 3)])
def test_model_ring_is_bitwise_the_full_region(name, slots):
    rec = W.load(name)
    gpt = rec["meta"]["family"] == "gpt"
    res = []
    for s in (0, slots):
        units = W.units_for(rec)
        ex = Executor(units, W.bundle_for(rec), batch=rec["meta"]["batch"],
                      loss_fn=lm_loss if gpt else cross_entropy_loss,
                      cfg=ExecConfig(weight_dtype=torch.bfloat16, optimizer="adam", lr=1e-3,
                                     host_path_all=gpt, grad_slots=s))
        ex.init_weights(seed=3)
        g = torch.Generator().manual_seed(0)
        m = rec["meta"]
        losses = []
        for _ in range(3):
            if gpt:
                x = torch.randint(0, m["vocab"], (m["batch"], m["seq"]), generator=g).cuda().int()
                y = torch.randint(0, m["vocab"], (m["batch"], m["seq"]), generator=g).cuda()
            else:
                x = torch.randn(m["batch"], 3, m["res"], m["res"], generator=g).cuda().to(torch.bfloat16)
                x = x.contiguous(memory_format=torch.channels_last)
                y = torch.randint(0, m["classes"], (m["batch"],), generator=g).cuda()
            losses.append(float(ex.step(x, y)))
        w = ex.unit_weights()
        st = ex.stats()
        ex.close()
        res.append((losses, w, st))
    assert res[0][0] == res[1][0]
    for k in res[0][1]:
        for a, b in zip(res[0][1][k], res[1][1][k]):
            assert torch.equal(a, b), k
    assert res[1][2]["grad_region_bytes"] <= res[0][2]["grad_region_bytes"]
