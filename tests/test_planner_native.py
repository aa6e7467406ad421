"""The C++ planner (krt_plan_model) vs the reference planner's own plans:
plan_to_dict must be identical (blocks, flags, stages, stage durations,
predicted makespan, theta) — index work, so bit-exact."""
import json

import pytest

from paper_2008_11421_b200 import workloads as W
from paper_2008_11421_b200._lib import InfeasiblePlanError
from paper_2008_11421_b200.plan import plan_model


def test_golden_cases_bit_exact(sched_cases):
    n = 0
    for c in sched_cases:
        strategy, solver = c["strategy"], c["solver"]
        if "infeasible" in c:
            with pytest.raises(InfeasiblePlanError):
                plan_model(c["model"], c["hardware"], strategy, solver)
            continue
        got = plan_model(c["model"], c["hardware"], strategy, solver)
        assert got.to_dict() == c["plan"], c["name"]
        assert got.plan_string() == c["plan_string"]
        n += 1
    assert n >= 45


@pytest.mark.parametrize("name", ["resnet_small_f32_a", "resnet_small_f32_b", "resnet_small_bf16",
                                  "preact29_small_f32", "preact29_small_bf16", "gpt_small_f32",
                                  "gpt_small_bf16", "resnet200_b3072", "resnet200_b3072_unbounded",
                                  "resnet200_b512", "resnet200_b2560", "gpt2p5b_b144",
                                  "megatron8p3b_l36_b128", "tnlg17b_l18_b176"])
def test_workload_plans_bit_exact(name):
    rec = W.load(name)
    got = plan_model(rec["model"], rec["hardware"], "capacity-recompute", "auto", rec.get("max_blocks"))
    assert got.to_dict() == rec["plan"]
