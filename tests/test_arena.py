"""Static arena assignment (krt_plan_arena): the physical realisation of the
simulator's capacity ledger (simulator.py:90).  Host-only checks."""
import pytest

from paper_2008_11421_b200 import workloads as W
from paper_2008_11421_b200.plan import PlanBundle


def check_arena(bundle, block_bytes):
    a = bundle.arena(block_bytes)
    inst = a["instances"]
    deps = {}
    for op, d in a["deps"]:
        deps.setdefault(op, set()).add(d)
    assert a["arena_bytes"] >= a["ledger_peak"] - 1e-6 * a["ledger_peak"] - 256 * len(inst)
    for i, x in enumerate(inst):
        assert x["off"] % 256 == 0 and x["off"] + x["bytes"] <= a["arena_bytes"]
        for j, y in enumerate(inst):
            if i == j:
                continue
            if x["off"] < y["off"] + y["bytes"] and y["off"] < x["off"] + x["bytes"]:
                # sharing bytes: one must free before the other allocates, and
                # the later allocation waits for that free explicitly
                later, earlier = (x, y) if (y["free_op"] in deps.get(x["alloc_op"], ())) else (y, x)
                assert earlier["free_op"] in deps.get(later["alloc_op"], ()), (x, y)
    return a


def test_golden_plans_arena_safe(sched_cases):
    n = 0
    for c in sched_cases:
        if "plan" not in c or c["validate"]:
            continue
        b = PlanBundle(c["model"], c["hardware"], c["plan"])
        sizes = [int(blk["swap_bytes"]) for blk in c["plan"]["blocks"]]
        check_arena(b, sizes)
        n += 1
    assert n > 30


@pytest.mark.parametrize("name", ["resnet200_b3072", "resnet200_b512", "resnet_small_f32_a",
                                  "resnet_small_f32_b", "resnet_small_bf16"])
def test_workload_arena_within_ledger(name):
    rec = W.load(name)
    units = W.units_for(rec)
    batch = rec["meta"]["batch"]
    sizes = [sum(u.saved_bytes(batch) for u in units[blk["layers"][0] - 1:blk["layers"][1]])
             for blk in rec["plan"]["blocks"]]
    # the IR's mem_fwd overrides are the physical sizes: plan bytes == slot bytes
    assert sizes == [int(blk["swap_bytes"]) for blk in rec["plan"]["blocks"]]
    a = check_arena(W.bundle_for(rec), sizes)
    assert a["arena_bytes"] <= 1.05 * a["ledger_peak"] + 2 ** 21
