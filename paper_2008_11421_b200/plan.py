"""Plan boundary: the reference's plan.json + model + hardware, bound to the
native engine.

The reference planner (oocsched) emits an ``ExecutionPlan`` (plan.py:75-106)
serialized by ``plan_to_dict`` (plan.py:179-202).  ``PlanBundle`` loads that
JSON together with the model text (model_ir.py:281-330) and hardware text
(cost_model.py:308-339) into libkrt, and exposes the reference's functions for
this path with the same names and return shapes:

* ``plan_string``            — plan.py:166-167
* ``validate_plan``          — planner.py:342-413 (list of violation strings)
* ``simulate``               — simulator.py:364-399 (trace dict; raises
                               ``DeadlockError`` like the reference)
* ``simulate_distributed``   — distsim.py:140-266 (plus the executor's own
                               device reduce-scatter variant)
* ``occupancy``              — occupancy.py:202-225 analytic_report

All computation happens in C++ (csrc/engine.cpp); Python only marshals.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import Optional, Union

from . import _lib


class DeadlockError(Exception):
    """Same shape as the reference's DeadlockError (simulator.py:36-39)."""

    def __init__(self, blocked):
        self.blocked = list(blocked)
        super().__init__("simulation deadlock; blocked ops: " + "; ".join(self.blocked))


class DistSimError(RuntimeError):
    pass


@dataclass(frozen=True)
class DistConfig:
    """distsim.py:46-62"""
    workers: int
    collective: str = "ring"
    net_bw: float = 12.5e9
    net_latency: float = 0.0
    groups: int = 0
    # Not in the reference: the B200 executor's P >= 2 pipeline (exchange =
    # device reduce-scatter before a 1/P grad_out, shard host update, shard
    # weight_in + all_gather), and the fix of distsim.py:165's dep offset.
    device_exchange: bool = False
    exact_deps: bool = False


class PlanBundle:
    """A model graph, a hardware spec and an execution plan loaded into libkrt."""

    def __init__(self, model_text: str, hw_text: str, plan: Union[str, dict]):
        if isinstance(plan, dict):
            plan = json.dumps(plan)
        self.model_text, self.hw_text, self.plan_json = model_text, hw_text, plan
        h = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_load(model_text.encode(), hw_text.encode(),
                                            plan.encode(), C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value:
                _lib.lib().krt_plan_free(h)
        except Exception:   # interpreter shutdown
            pass
        self._h = None

    def set_capacity(self, capacity_bytes: float) -> "PlanBundle":
        _lib.check(_lib.lib().krt_plan_set_capacity(self._h, float(capacity_bytes)))
        return self

    def plan_string(self) -> str:
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_string(self._h, C.byref(out)))
        return _lib.take_string(out)

    def to_dict(self) -> dict:
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_json(self._h, C.byref(out)))
        return json.loads(_lib.take_string(out))

    def validate(self) -> list[str]:
        out = C.c_void_p()
        n = C.c_int()
        _lib.check(_lib.lib().krt_plan_validate(self._h, C.byref(out), C.byref(n)))
        return json.loads(_lib.take_string(out))

    def simulate(self, enforce_capacity: bool = True) -> dict:
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_simulate(self._h, int(enforce_capacity), C.byref(out)))
        res = json.loads(_lib.take_string(out))
        if "deadlock" in res:
            raise DeadlockError(res["deadlock"])
        return res

    def arena(self, block_bytes) -> dict:
        """Static arena assignment for physical slot sizes (krt_plan_arena)."""
        arr = (C.c_size_t * len(block_bytes))(*block_bytes)
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_arena(self._h, arr, len(block_bytes), C.byref(out)))
        return json.loads(_lib.take_string(out))

    def costs(self) -> dict:
        """block_cost per block and layer_ops per layer (cost_model.py:97-273)."""
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_costs(self._h, C.byref(out)))
        return json.loads(_lib.take_string(out))

    def occupancy(self) -> dict:
        """analytic_report + find_theta (occupancy.py:178-225): theta (None =
        the device never waits), mean_occupancy, per_step rows, csv, summary."""
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_occupancy(self._h, C.byref(out)))
        return json.loads(_lib.take_string(out))

    def simulate_distributed(self, cfg: DistConfig, iterations: int = 3) -> dict:
        if iterations < 2:
            raise DistSimError("need at least 2 iterations to observe the steady state")
        if cfg.collective not in ("ring", "flat"):
            raise DistSimError(f"unknown collective {cfg.collective!r}")
        c = _lib.DistConfig(cfg.workers, int(cfg.collective == "ring"), cfg.net_bw,
                            cfg.net_latency, cfg.groups,
                            int(cfg.device_exchange) | 2 * int(cfg.exact_deps))
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_plan_simulate_dist(self._h, C.byref(c), int(iterations),
                                                     C.byref(out)))
        res = json.loads(_lib.take_string(out))
        if "error" in res:
            raise DistSimError(res["error"])
        return res


def plan_model(model_text: str, hw_text: str, strategy: str = "capacity-recompute",
               solver: str = "auto", max_blocks: Optional[int] = None) -> PlanBundle:
    """planner.py:890-912 in C++ (csrc/planner.cpp): same plan, bit for bit."""
    h = C.c_void_p()
    _lib.check(_lib.lib().krt_plan_model(model_text.encode(), hw_text.encode(), strategy.encode(),
                                         solver.encode(), int(max_blocks or 0), C.byref(h)))
    b = PlanBundle.__new__(PlanBundle)
    b.model_text, b.hw_text = model_text, hw_text
    b._h = h
    b.plan_json = None
    return b


# reference-named module functions -------------------------------------------------

def read_plan(json_path, model_text: str, hw_text: str) -> PlanBundle:
    """plan.py:244-246, bound to its model and hardware."""
    with open(json_path, "r", encoding="utf-8") as fh:
        return PlanBundle(model_text, hw_text, fh.read())


def plan_string(bundle: PlanBundle) -> str:
    return bundle.plan_string()


def validate_plan(bundle: PlanBundle, capacity_bytes: Optional[float] = None) -> list[str]:
    if capacity_bytes is not None:
        bundle.set_capacity(capacity_bytes)
    return bundle.validate()


def simulate(bundle: PlanBundle, enforce_capacity: bool = True) -> dict:
    return bundle.simulate(enforce_capacity)


def simulate_distributed(bundle: PlanBundle, cfg: DistConfig, iterations: int = 3) -> dict:
    return bundle.simulate_distributed(cfg, iterations)
