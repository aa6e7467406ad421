"""B200 HardwareSpec calibration from measurements.

The reference planner sees the machine only through ``HardwareSpec``
(cost_model.py:49-80): capacity, far/near-memory and interconnect bandwidth,
``compute_rate`` (ops/s, one op = one multiply-add, cost_model.py:3-4), per
layer-kind ``efficiency.<kind>`` multipliers (cost_model.py:225-247),
``backward_multiplier`` and ``host_update_rate`` (elements/s of the host
optimizer, distsim.py:231-236).  This module measures each of them on the
box instead of hand-tuning:

* ``compute_rate``        = the measured sustained dense bf16 peak
                            (MEASURED_PEAKS.json) / 2 (a MAC is 2 flops);
* ``efficiency.<kind>``   = achieved MAC/s of the executor's forward ops of
                            that kind (trace durations, this workload) /
                            compute_rate;
* ``backward_multiplier`` = measured backward time / measured forward time
                            of the same blocks;
* ``interconnect_bw``     = the PCIe probe with both directions busy (the
                            planner's swaps overlap in both directions);
* ``near_mem_bw``         = the measured HBM copy bandwidth;
* ``host_update_rate``    = host Adam elements/s on the runtime's own thread
                            count (krt_host_update, the product's kernel).

``hw_text`` renders the result in the reference's key = value format
(cost_model.py:308-339) for ``scripts/make_plans.py``.
"""
from __future__ import annotations

import os
import time
from collections import defaultdict

import torch

from . import _lib


def runtime_host_threads() -> int:
    """The runtime's default host-update pool size (runtime.cu: hardware
    concurrency - 2)."""
    return max(1, (os.cpu_count() or 1) - 2)


def host_update_rate(n: int = 1 << 25, threads: int = 0, optimizer: str = "adam", reps: int = 3) -> dict:
    """Host Adam/SGD elements per second through krt_host_update (bf16 weight
    copy written, as on the host path); best of ``reps``."""
    threads = threads or runtime_host_threads()
    p = torch.randn(n)
    m = torch.zeros(n)
    v = torch.zeros(n)
    g = torch.randn(n) * 1e-3
    w = torch.empty(n, dtype=torch.bfloat16)
    L = _lib.lib()
    opt = 1 if optimizer == "adam" else 0
    best = float("inf")
    for step in range(1, reps + 2):
        t0 = time.perf_counter()
        _lib.check(L.krt_host_update(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), w.data_ptr(),
                                     1, n, opt, 1e-4, 0.9, 0.999, 1e-8, 0.0, 0.0, step, threads))
        dt = time.perf_counter() - t0
        if step > 1:           # the first call faults the pages in
            best = min(best, dt)
    return {"elements_per_s": n / best, "elements": n, "threads": threads, "optimizer": optimizer,
            "seconds": best}


def from_trace(bundle, trace_csv: str) -> dict:
    """Per-kind achieved MAC/s and the backward multiplier from an executor
    trace (krt_trace_csv: t_start,t_end,resource,block,action,group,stall_before)
    of the plan ``bundle`` describes; the steady-state iteration is the last
    one in the trace."""
    costs = bundle.costs()
    layer_kind = {l["id"]: l["kind"] for l in costs["layers"]}
    layer_ops = {l["id"]: l["ops"] for l in costs["layers"]}
    blk_layers = {b["id"]: range(b["layers"][0], b["layers"][1] + 1) for b in costs["blocks"]}
    fw_t, bw_t = defaultdict(float), defaultdict(float)
    n_fw = defaultdict(int)
    for line in trace_csv.strip().splitlines()[1:]:
        r = line.split(",")
        if r[2] != "compute":
            continue
        b, act, dur = int(r[3]), r[4], float(r[1]) - float(r[0])
        if act in ("fw", "recompute_fw"):
            fw_t[b] += dur
            n_fw[b] += 1
        elif act == "bw":
            bw_t[b] += dur
    kind_ops, kind_t = defaultdict(float), defaultdict(float)
    for b, t in fw_t.items():
        ops = sum(layer_ops[i] for i in blk_layers[b])
        if ops <= 0:
            continue
        # a block's forward time is attributed to its layers' kinds by op share
        for i in blk_layers[b]:
            share = layer_ops[i] / ops
            kind_ops[layer_kind[i]] += layer_ops[i] * n_fw[b]
            kind_t[layer_kind[i]] += t * share
    rate = {k: kind_ops[k] / kind_t[k] for k in kind_ops if kind_t[k] > 0}
    fw_once = sum(fw_t[b] / n_fw[b] for b in bw_t if n_fw[b])
    bw_sum = sum(bw_t.values())
    return {"mac_per_s_by_kind": rate, "backward_multiplier": bw_sum / fw_once if fw_once > 0 else None,
            "forward_s": fw_once, "backward_s": bw_sum}


def calibrate(bundle, trace_csv: str, peaks: dict, pcie: dict, host: dict) -> dict:
    """The measured HardwareSpec fields (see the module docstring)."""
    tr = from_trace(bundle, trace_csv)
    compute_rate = peaks["bf16_tflops_sustained"] * 1e12 / 2.0
    eff = {k: r / compute_rate for k, r in tr["mac_per_s_by_kind"].items()}
    return {
        "compute_rate": compute_rate,
        "efficiency": eff,
        "backward_multiplier": tr["backward_multiplier"],
        "interconnect_bw": pcie["duplex"] * 1e9,
        "near_mem_bw": peaks["hbm_gbs"] * 1e9,
        "host_update_rate": host["elements_per_s"],
        "host_update": host,
        "trace": tr,
        "source": "calibrate.py: MEASURED_PEAKS.json sustained bf16 / 2, executor trace per-kind forward MAC/s "
                  "and backward/forward ratio, duplex PCIe probe, krt_host_update on the runtime's threads",
    }


def capacity_of(hw_text_in: str) -> float:
    for line in hw_text_in.splitlines():
        k, _, v = line.partition("=")
        if k.strip() == "capacity_bytes":
            return float(v)
    raise ValueError("hardware text has no capacity_bytes")


HW_KEYS = ("far_mem_bw", "near_mem_bw", "interconnect_bw", "compute_rate", "host_update_rate",
           "backward_multiplier")


def hw_text(capacity: float, cal: dict, far_mem_bw: float = 200e9) -> str:
    """cost_model.py:308-339 key = value text (repr() keeps the exact doubles)."""
    v = dict(far_mem_bw=far_mem_bw, near_mem_bw=cal["near_mem_bw"], interconnect_bw=cal["interconnect_bw"],
             compute_rate=cal["compute_rate"], host_update_rate=cal["host_update_rate"],
             backward_multiplier=cal["backward_multiplier"])
    lines = [f"capacity_bytes = {float(capacity)!r}"] + [f"{k} = {float(v[k])!r}" for k in HW_KEYS]
    lines.append("duplex = true")
    for kind in sorted(cal["efficiency"]):
        lines.append(f"efficiency.{kind} = {float(cal['efficiency'][kind])!r}")
    return "\n".join(lines) + "\n"
