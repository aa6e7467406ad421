"""Generate the schedule/timing golden fixtures from the UNMODIFIED reference.

Run HERE (the reference is importable only in the build container):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It writes ``tests/golden/sched_cases.json``: for every fixture the model text
(``model_ir.serialize_model``), the hardware text (``cost_model.serialize_hardware``),
the planner's plan (``plan.plan_to_dict`` / ``plan_string``), the simulator's
trace (``simulator.simulate``), ``validate_plan`` verdicts for structurally
perturbed plans, and ``distsim.simulate_distributed`` traces at P = 1, 2, 4.
Nothing in the repo imports the reference at run time; the GPU box only sees
the JSON this script produced.
"""
from __future__ import annotations

import json
import random
import sys
from dataclasses import replace
from pathlib import Path

from oocsched.cost_model import parse_hardware_text
from oocsched.distsim import Collective, DistConfig, simulate_distributed
from oocsched.model_ir import serialize_model
from oocsched.plan import Action, PlanOp, Stage, Strategy, plan_string, plan_to_dict
from oocsched.planner import InfeasibleModelError, plan_model, validate_plan
from oocsched.occupancy import analytic_report, find_theta
from oocsched.planner import build_blocks, generate_schedule
from oocsched.simulator import DeadlockError, simulate
from oocsched import zoo

OUT = Path(__file__).with_name("sched_cases.json")


def perturb(plan, rng):
    # same mutation families as the reference's tests/test_planner.py:_perturb
    stages = [Stage(id=s.id, ops=tuple(s.ops), duration=s.duration) for s in plan.stages]
    kind = rng.randrange(5)
    if kind == 0 and len(stages) >= 2:
        i, j = rng.sample(range(len(stages)), 2)
        stages[i], stages[j] = stages[j], stages[i]
    elif kind == 1 and len(stages) >= 2:
        del stages[rng.randrange(len(stages))]
    elif kind == 2:
        i = rng.randrange(len(stages))
        ops = list(stages[i].ops)
        ops.pop(rng.randrange(len(ops)))
        stages[i] = Stage(id=stages[i].id, ops=tuple(ops), duration=stages[i].duration)
    elif kind == 3 and len(plan.blocks) >= 2:
        i = rng.randrange(len(stages))
        ops = list(stages[i].ops)
        j = rng.randrange(len(ops))
        other = rng.choice([b.id for b in plan.blocks if b.id != ops[j].block])
        ops[j] = PlanOp(ops[j].action, other)
        stages[i] = Stage(id=stages[i].id, ops=tuple(ops), duration=stages[i].duration)
    else:   # merge a stage into its successor (same-stage hazards)
        if len(stages) >= 2:
            i = rng.randrange(len(stages) - 1)
            merged = Stage(id=stages[i].id, ops=stages[i].ops + stages[i + 1].ops,
                           duration=stages[i].duration)
            stages[i:i + 2] = [merged]
    return replace(plan, stages=tuple(stages))


def hw_text(hw):
    """serialize_hardware() rounds to 6 significant digits (%g); emit repr() so the
    C++ parser sees the exact doubles the reference simulated with."""
    lines = [f"{k} = {getattr(hw, k)!r}" for k in (
        "capacity_bytes", "far_mem_bw", "near_mem_bw", "interconnect_bw",
        "compute_rate", "host_update_rate", "backward_multiplier")]
    lines.append(f"duplex = {'true' if hw.duplex else 'false'}")
    for kind in sorted(hw.efficiency):
        lines.append(f"efficiency.{kind} = {hw.efficiency[kind]!r}")
    assert parse_hardware_text("\n".join(lines)) == hw
    return "\n".join(lines) + "\n"


def trace_rows(trace):
    return [[e.t_start, e.t_end, e.resource, e.block, e.action.value, e.stall_before]
            for e in trace.events]


def dist_rows(tr):
    return [[e.worker, e.resource, e.t_start, e.t_end, e.action, e.block, e.group,
             e.iteration, e.stall_before] for e in tr.events]


def sim_record(plan, g, hw, enforce=True):
    try:
        tr = simulate(plan, g, hw, enforce_capacity=enforce)
    except DeadlockError as exc:
        return {"deadlock": exc.blocked}
    return {"makespan": tr.makespan, "total_stall": tr.total_stall,
            "peak_mem": tr.peak_mem, "events": trace_rows(tr), "csv": tr.to_csv()}


def occupancy_record(plan, g, hw):
    """analytic_report / find_theta and the trace's own occupancy figures
    (occupancy.py:178-225, simulator.py:200-236, cli.py:115-121)."""
    rep = analytic_report(plan, g, hw)
    theta = find_theta(plan, g, hw)
    rec = {"theta": theta, "mean_occupancy": rep.mean_occupancy,
           "per_step": [[s.step, s.occupancy, s.busy_s, s.idle_s] for s in rep.per_step],
           "csv": rep.to_csv(), "summary": rep.summary()}
    try:
        tr = simulate(plan, g, hw)
    except DeadlockError:
        return rec
    rec["trace"] = {"mean_occupancy": tr.mean_occupancy(),
                    "first_stall_backward_step": tr.first_stall_backward_step(),
                    "boundary_stall": tr.boundary_stall(),
                    "summary_csv": tr.summary_csv(theta=theta)}
    return rec


def case(name, g, hw, strategy=Strategy.CAPACITY_RECOMPUTE, solver="auto",
         rng=None, n_perturb=12, dist=True):
    rec = {"name": name, "model": serialize_model(g), "hardware": hw_text(hw),
           "strategy": strategy.value, "solver": solver}
    try:
        plan = plan_model(g, hw, strategy=strategy, solver=solver)
    except InfeasibleModelError as exc:
        rec["infeasible"] = exc.reason
        return rec
    rec["plan"] = plan_to_dict(plan)
    rec["plan_string"] = plan_string(plan)
    rec["validate"] = validate_plan(plan, g, hw)
    rec["sim"] = sim_record(plan, g, hw)
    rec["occupancy"] = occupancy_record(plan, g, hw)
    rec["sim_open"] = sim_record(plan, g, replace(hw, capacity_bytes=hw.capacity_bytes * 0.5),
                                 enforce=False)
    tight = replace(hw, capacity_bytes=max(b.swap_bytes for b in plan.blocks) * 0.9)
    rec["validate_tight"] = {"capacity_bytes": tight.capacity_bytes,
                             "violations": validate_plan(plan, g, tight)}
    if rng is not None:
        perts = []
        for _ in range(n_perturb):
            broken = perturb(plan, rng)
            perts.append({"plan": plan_to_dict(broken),
                          "violations": validate_plan(broken, g, hw),
                          "sim": sim_record(broken, g, hw)})
        rec["perturbed"] = perts
    if dist:
        drecs = []
        for p, groups, coll in ((1, 0, "ring"), (2, 0, "ring"), (4, 2, "ring"), (3, 0, "flat")):
            cfg = DistConfig(workers=p, collective=Collective(coll),
                             net_bw=hw.interconnect_bw * 0.5, net_latency=1e-3 * (p > 1),
                             groups=groups)
            try:
                tr = simulate_distributed(plan, g, hw, cfg, iterations=3)
            except (DeadlockError, RuntimeError) as exc:
                drecs.append({"workers": p, "groups": groups, "collective": coll,
                              "net_bw": cfg.net_bw, "net_latency": cfg.net_latency,
                              "error": str(exc)})
                continue
            drecs.append({"workers": p, "groups": groups, "collective": coll,
                          "net_bw": cfg.net_bw, "net_latency": cfg.net_latency,
                          "iteration_time": tr.iteration_time,
                          "iteration_times": list(tr.iteration_times),
                          "exposed_comm": tr.exposed_comm, "peak_mem": tr.peak_mem,
                          "makespan": tr.makespan, "events": dist_rows(tr)})
        rec["dist"] = drecs
    return rec


def main():
    rng = random.Random(2008_11421)
    cases = []
    g, hw = zoo.swap_timeline_fixture()
    for st in Strategy:
        cases.append(case(f"timeline_{st.value}", g, hw, strategy=st, rng=rng))
    g = zoo.fc_chain_model(6, 64, 2)
    hw = zoo.uniform_chain_hardware(g, 2.0, 3.0)
    cases.append(case("cfg0_fc_chain", g, hw, solver="exhaustive", rng=rng))
    hw_nd = zoo.uniform_chain_hardware(g, 2.0, 3.0, duplex=False)
    cases.append(case("fc_chain_simplex", g, hw_nd, rng=rng))
    g = zoo.unet_model()
    cases.append(case("unet", g, zoo.unet_hardware(g), rng=rng))
    g = zoo.bottleneck_model()
    cases.append(case("bottleneck", g, zoo.unet_hardware(g, 0.6), rng=rng))
    g = zoo.conv_stack_model(conv_stages=8, batch=8)
    cases.append(case("conv_stack_8", g, zoo.conv_stack_hardware(6e6), solver="dp", rng=rng))
    for i in range(40):
        n = rng.randint(3, 14)
        g = zoo.random_linear_model(rng, n)
        hw = zoo.random_hardware(rng, g)
        solver = "dp" if n > 9 else "auto"
        cases.append(case(f"fuzz_{i}", g, hw, solver=solver, rng=rng, n_perturb=6))
    OUT.write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                               "reference": "oocsched 0.1.0 (/root/reference/pkg)",
                               "cases": cases}, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(cases)} cases)", file=sys.stderr)
    occ_cases()


def occ_cases():
    """The reference's occupancy fixtures (test_occupancy.py:25-33,
    :144-161): CAPACITY schedules of uniform chains, with the fast-link and
    instant-compute variants of test_occupancy.py:87-107."""
    out = []
    for n, ratio, cap in [(6, 2.0, 3.0), (8, 1.2, 3.0), (8, 3.0, 4.0), (10, 2.5, 4.0), (6, 4.0, 3.0)]:
        g = zoo.uniform_chain_model(num_layers=n)
        hw = zoo.uniform_chain_hardware(g, swap_compute_ratio=ratio, capacity_blocks=cap)
        blocks, costs = build_blocks([(i, i) for i in range(1, n + 1)], g, hw)
        plan = generate_schedule(blocks, g, hw, Strategy.CAPACITY, costs=costs)
        for tag, h in (("", hw), ("_fastlink", replace(hw, interconnect_bw=1e15)),
                       ("_instant", replace(hw, compute_rate=1e18))):
            out.append({"name": f"chain{n}_r{ratio}_c{cap}{tag}", "model": serialize_model(g),
                        "hardware": hw_text(h), "plan": plan_to_dict(plan),
                        "occupancy": occupancy_record(plan, g, h)})
    path = OUT.with_name("occupancy_cases.json")
    path.write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                                "reference": "oocsched 0.1.0 (/root/reference/pkg)",
                                "cases": out}, separators=(",", ":")))
    print(f"wrote {path} ({len(out)} cases)", file=sys.stderr)


if __name__ == "__main__":
    main()
