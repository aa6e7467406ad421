"""Committed workloads: plans produced by the reference planner
(scripts/make_plans.py) plus the executor units they were planned for."""
from __future__ import annotations

import copy
import json
from pathlib import Path

import torch

from .plan import PlanBundle
from .units import gpt_units, resnet1001_units, resnet_units

PLANS = Path(__file__).with_name("plans")


def load(name: str) -> dict:
    return json.loads((PLANS / f"{name}.json").read_text())


def units_for(rec: dict):
    m = rec["meta"]
    if m["family"] == "gpt":
        act = torch.float32 if m["act"] == "f32" else torch.bfloat16
        return gpt_units(m["hidden"], m["heads"], m["layers"], m["seq"], m["vocab"], act_dtype=act)
    if m["family"] == "preact":
        act = torch.float32 if m["act"] == "f32" else torch.bfloat16
        return resnet1001_units(m["res"], m["classes"], m["depth"], act_dtype=act)
    if m["family"] == "resnet":
        act = torch.float32 if m["act"] == "f32" else torch.bfloat16
        if "depth" in m:
            return resnet_units(m["depth"], m["res"], m["classes"], act_dtype=act)
        return resnet_units(stages=tuple(m["stages"]), res=m["res"], classes=m["classes"],
                            act_dtype=act)
    raise ValueError(f"unknown family {m['family']}")


def bundle_for(rec: dict, plan: dict | None = None) -> PlanBundle:
    return PlanBundle(rec["model"], rec["hardware"], plan if plan is not None else rec["plan"])


def incore_plan(plan: dict) -> dict:
    """Same blocks, every block resident: F1..Fn then Bn..B1 (no swap, no recompute)."""
    p = copy.deepcopy(plan)
    nb = len(p["blocks"])
    for b in p["blocks"]:
        b["recompute"] = False
        b["checkpoint"] = True
    p["strategy"] = "capacity"
    p["stages"] = ([{"id": i + 1, "duration": 0.0, "ops": [["fw", i + 1]]} for i in range(nb)] +
                   [{"id": nb + i + 1, "duration": 0.0, "ops": [["bw", nb - i]]} for i in range(nb)])
    return p
