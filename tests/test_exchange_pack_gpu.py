"""bf16 exchange pack (krt_config.exchange_bf16): each group's fp32 gradients
are cast into a bf16 pack buffer, reduce-scattered in bf16 over NCCL (half
the NVLink bytes of the fp32 exchange) and the shard unpacked to fp32 for the
D2H and host update.  One GPU runs it through a one-rank communicator
(force_dp_path): the result must equal the fp32 exchange with every gradient
rounded to bf16 once, i.e. match it to bf16 resolution."""
import numpy as np
import pytest
import torch

from oracle import fc_chain_oracle as orc
from paper_2008_11421_b200.executor import ExecConfig, Executor
from paper_2008_11421_b200.plan import PlanBundle
from paper_2008_11421_b200.units import FCUnit, mse_zero_loss

pytestmark = pytest.mark.gpu


def run(sched_cases, **cfg):
    c = next(c for c in sched_cases if c["name"] == "cfg0_fc_chain")
    ex = Executor([FCUnit(64, 64) for _ in range(6)], PlanBundle(c["model"], c["hardware"], c["plan"]), batch=2,
                  loss_fn=mse_zero_loss, cfg=ExecConfig(force_dp_path=True, **cfg))
    w0 = orc.init_weights()
    ex.load_weights({i + 1: [torch.from_numpy(w)] for i, w in enumerate(w0)})
    losses = [float(ex.step(torch.from_numpy(orc.inputs(0, it)).cuda())) for it in range(1, 2)]
    w = ex.unit_weights()
    st = ex.stats()
    ex.close()
    return losses, [w[i + 1][0].cpu().numpy() for i in range(6)], st, w0


@pytest.mark.parametrize("slots", [0, 2])
def test_bf16_pack_sgd_step_is_the_bf16_rounded_gradient(sched_cases, slots):
    lr = 1.0   # w1 = w0 - g: the weight rounding (ulp(w0) ~ 1e-8) stays far below bf16 steps of g
    _, w32, s32, w0 = run(sched_cases, optimizer="sgd", lr=lr, dist_groups=3, grad_slots=slots)
    _, w16, s16, _ = run(sched_cases, optimizer="sgd", lr=lr, dist_groups=3, grad_slots=slots, exchange_bf16=True)
    for a32, a16, p0 in zip(w32, w16, w0):
        g32 = (p0 - a32) / lr                     # the fp32-exchange gradient
        g16 = (p0 - a16) / lr
        want = torch.from_numpy(g32).to(torch.bfloat16).float().numpy()
        # one bf16 rounding of each gradient element: equal to the rounded
        # fp32-exchange gradient, up to one bf16 step where the recovered fp32
        # gradient (w0 - w1, off by ulp(w0) ~ 1e-8) sits on a rounding boundary
        np.testing.assert_allclose(g16, want, rtol=2 ** -7, atol=3e-8)
        assert np.mean(np.abs(g16 - want) <= 3e-8) >= 0.95
        assert not np.array_equal(a32, a16) or np.array_equal(g32, want)
    assert s16["bytes_net_total"] * 2 == s32["bytes_net_total"] or s32["world"] == 1


def test_bf16_pack_adam_tracks_oracle(sched_cases):
    losses, w16, _, w0 = run(sched_cases, optimizer="adam", lr=1e-3, exchange_bf16=True)
    ref_losses, ref_w = orc.train(workers=1, iterations=1, optimizer="adam", lr=1e-3, weights=w0)
    np.testing.assert_allclose(losses, [l[0] for l in ref_losses], rtol=1e-5)
    for a, r, p in zip(w16, ref_w, w0):
        # Adam's first step is lr * sign(g) up to eps: bf16 rounding keeps signs
        np.testing.assert_allclose(a, r, rtol=1e-5, atol=2e-6)
