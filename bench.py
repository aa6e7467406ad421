"""Benchmark: KARMA out-of-core data-parallel training on B200.

Metric (BASELINE.json): samples/sec of a model whose activations exceed HBM,
with the per-iteration roofline (compute / PCIe / NVLink).  Workload (N=1):
cfg1 — ResNet-200, 224x224x3 synthetic N(0,1) images, 1000 classes, bf16,
per-GPU batch 3072 (320 GB of saved activations per iteration = 1.67x the
192 GB of HBM), planned by the UNMODIFIED reference planner into a swap +
recompute schedule (paper_2008_11421_b200/plans/resnet200_b3072.json,
scripts/make_plans.py).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--plan NAME] [--impl reference]

N > 1: one rank per GPU under torchrun (bench.py re-launches itself through
torch.distributed.run when WORLD_SIZE is unset, and fails when the world size
differs from --gpus); the gradient exchange is the runtime's own NCCL
communicator (reduce-scatter per group, all-gather of the updated shards);
weak scaling: every rank trains its own per-GPU batch.  Before the timed
region every rank probes, concurrently, its PCIe link (pinned H2D / D2H /
duplex) and, at N > 1, the NCCL reduce-scatter bus bandwidth at the plan's
group sizes; the iteration roofline uses those measured rates.
`--impl reference` times the CPU reference arm (the in-core fp32 torch CPU
oracle of the same model, oracle/resnet_oracle.py) on all host cores, plus
the reference's own executable CPU path (oocsched plan_model +
simulate_distributed from baseline/_ref).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# unit temporaries come and go in multi-GB sizes next to a 140 GB arena
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

PEAK_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
PCIE_H2D, PCIE_D2H, PCIE_DUPLEX = 55.6e9, 57.3e9, 49.8e9   # scripts/probe_box.py on this pool


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAK_FALLBACK, "fallback"


class Clocks:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def self_launch(args):
    """bench.py --gpus N without torchrun: re-run under torch.distributed.run
    with N ranks on this node (127.0.0.1 rendezvous) and exit with its code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd))


def reference_planner_time(rec, workers):
    """The reference's only executable CPU path for this workload:
    oocsched.plan_model on the committed model/hardware texts, then
    simulate_distributed of the resulting plan at `workers` ranks, timed on
    this host.  The reference is the unmodified package installed in
    baseline/_ref (never /root/reference at run time)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "oocsched").exists():
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, str(ref))
    try:
        from oocsched.cost_model import parse_hardware_text
        from oocsched.distsim import DistConfig, simulate_distributed
        from oocsched.model_ir import parse_model_text
        from oocsched.planner import plan_model
        g, hw = parse_model_text(rec["model"]), parse_hardware_text(rec["hardware"])
        t0 = time.perf_counter()
        plan = plan_model(g, hw, max_blocks=rec.get("max_blocks"))
        t1 = time.perf_counter()
        out = {"plan_model_s": round(t1 - t0, 4), "workers": workers, "cores": 1,
               "max_blocks": rec.get("max_blocks"),
               "same_plan_as_committed": [(b.first_layer, b.last_layer) for b in plan.blocks] ==
                                         [tuple(b["layers"]) for b in rec["plan"]["blocks"]]}
        try:
            dr = simulate_distributed(plan, g, hw, DistConfig(workers=max(1, workers)), iterations=3)
            out["predicted_iteration_s"] = dr.iteration_time
        except Exception as exc:   # the reference's own verdict (e.g. its DP ledger deadlocks)
            out["simulate_distributed_error"] = f"{type(exc).__name__}: {str(exc)[:160]}"
        out["simulate_distributed_s"] = round(time.perf_counter() - t1, 4)
        return out
    except Exception as exc:   # report, do not fail the bench
        return {"error": f"{type(exc).__name__}: {exc}"}
    finally:
        sys.path.remove(str(ref))


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU reference arm / cpu_baseline: in-core fp32 torch CPU training step
# ---------------------------------------------------------------------------
def cpu_sample_batch(rec):
    # bounded CPU sample: ~10-30 s of host work
    m = rec["meta"]
    if m["family"] == "gpt":
        return 1
    return 4 if m["res"] <= 256 else 1


def cpu_sample_note(rec):
    m = rec["meta"]
    if m["family"] == "gpt":
        return " of 256 tokens, scaled to the 1024-token sample by 1/4"
    return "" if m["res"] <= 256 else " at 512x512, scaled by the pixel ratio 1/16"


def cpu_reference(rec, steps, warmup, sample_batch=None):
    """The in-core fp32 torch-CPU oracle of the same model, all host cores."""
    import torch

    from oracle import gpt_oracle, resnet_oracle
    from paper_2008_11421_b200 import units as U
    from paper_2008_11421_b200 import workloads as W

    torch.set_num_threads(os.cpu_count() or 1)
    sample_batch = sample_batch or cpu_sample_batch(rec)
    m = dict(rec["meta"])
    scale = 1.0
    gen = torch.Generator().manual_seed(0)
    if m["family"] == "gpt":
        scale = 256 / m["seq"]
        m["seq"] = 256
        units = U.gpt_units(m["hidden"], m["heads"], m["layers"], 256, m["vocab"], act_dtype=torch.float32)
        x = torch.randint(0, m["vocab"], (sample_batch, 256), generator=gen)
        y = torch.randint(0, m["vocab"], (sample_batch, 256), generator=gen)
        fwd = lambda params: gpt_oracle.forward(units, params, x).reshape(-1, m["vocab"])
        tgt = y.reshape(-1)
    else:
        if m["res"] > 256:
            # in-core fp32 at 2048^2 needs ~314 GB of host RAM per image: time the
            # same network on 512^2 images and scale by the pixel ratio (FLOPs and
            # bytes of these convnets are linear in the pixel count)
            scale = (512 / m["res"]) ** 2
            m["res"] = 512
            units = U.resnet1001_units(512, m["classes"], m["depth"], act_dtype=torch.float32)
        else:
            units = W.units_for(rec)
        x = torch.randn(sample_batch, 3, m["res"], m["res"], generator=gen)
        tgt = torch.randint(0, m["classes"], (sample_batch,), generator=gen)
        fwd = lambda params: resnet_oracle.forward(units, params, x)
    init = {i + 1: [t.float() for t in u.init_params(gen)] for i, u in enumerate(units)}
    params = {k: [t.requires_grad_(True) for t in ts] for k, ts in init.items()}
    flat = [t for k in sorted(params) for t in params[k]]
    opt = torch.optim.SGD(flat, lr=0.1, foreach=False)

    def step():
        opt.zero_grad(set_to_none=True)
        loss = torch.nn.functional.cross_entropy(fwd(params), tgt)
        loss.backward()
        opt.step()

    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = time.perf_counter() - t0
    return sample_batch * steps / dt * scale, torch.get_num_threads(), dt


def model_name(rec):
    m = rec["meta"]
    if m["family"] == "gpt":
        return f"gpt-h{m['hidden']}-l{m['layers']} ({m['heads']} heads, vocab {m['vocab']})"
    return f"resnet{m['depth']}" if "depth" in m else rec["name"]


def metric_name(rec):
    m = rec["meta"]
    if m["family"] == "gpt":
        return (f"samples/sec ({model_name(rec)} seq {m['seq']} training step, per-GPU batch beyond HBM)")
    return (f"samples/sec ({model_name(rec)} {m['res']}x{m['res']} training step, per-GPU batch "
            f"beyond HBM)")


def workload_inputs(rec, dev, gen, batch=None):
    import torch
    m = rec["meta"]
    n = batch or m["batch"]
    if m["family"] == "gpt":
        x = torch.randint(0, m["vocab"], (n, m["seq"]), device=dev, generator=gen, dtype=torch.int32)
        y = torch.randint(0, m["vocab"], (n, m["seq"]), device=dev, generator=gen)
        return x, y
    x = torch.randn(n, 3, m["res"], m["res"], device=dev, generator=gen, dtype=torch.float32).to(
        torch.float32 if m.get("act") == "f32" else torch.bfloat16).contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, m["classes"], (n,), device=dev, generator=gen)
    return x, y


def workload_exec(rec):
    """loss function and optimizer per family: SGD-momentum for the convnets,
    host-side Adam on every block for the transformers."""
    from paper_2008_11421_b200.units import cross_entropy_loss, lm_loss
    if rec["meta"]["family"] == "gpt":
        return lm_loss, dict(optimizer="adam", lr=1e-4, host_path_all=True)
    return cross_entropy_loss, dict(optimizer="sgd", lr=0.1, momentum=0.9)


def run_reference(args, rec):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    value, cores, dt = cpu_reference(rec, steps, warmup)
    m = rec["meta"]
    line = {
        "metric": metric_name(rec),
        "impl": "reference", "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup, "ms_per_step": dt / steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": rec["name"], "model": model_name(rec),
                                         "per_gpu_batch": m["batch"], "image": m["res"]},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": f"in-core fp32 torch-CPU {model_name(rec)} step (oracle/) "
                                   f"on {cpu_sample_batch(rec)} samples per step{cpu_sample_note(rec)}"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_planner": reference_planner_time(rec, args.gpus),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def probe_pcie(dev, world, nbytes=512 << 20, reps=3):
    """Pinned H2D, D2H and duplex copy rates with every rank copying at the
    same time (barrier before each pattern); slowest rank's time."""
    import torch
    import torch.distributed as dist
    h1 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def run(pattern):
        ts = []
        for _ in range(reps + 1):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if pattern in ("h2d", "duplex"):
                with torch.cuda.stream(s1):
                    d1.copy_(h1, non_blocking=True)
            if pattern in ("d2h", "duplex"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize(dev)
            ts.append(time.perf_counter() - t0)
        t = torch.tensor([min(ts[1:])])
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return nbytes / float(t.item())
    out = {"h2d": run("h2d"), "d2h": run("d2h"), "duplex": run("duplex"),
           "bytes": nbytes, "ranks_concurrent": world,
           "note": "pinned cudaMemcpyAsync, all ranks at once, slowest rank (best of 3)"}
    del h1, h2, d1, d2
    return out


def probe_nccl(ex, group_bytes, world):
    """Reduce-scatter seconds on the runtime's own communicator at the plan's
    group sizes (<= 8 distinct sizes probed; others scaled linearly from the
    nearest probed size).  Returns (seconds per iteration for all groups,
    bus GB/s at each probed size)."""
    sizes = sorted(set(group_bytes))
    if len(sizes) > 8:
        sizes = [sizes[round(i * (len(sizes) - 1) / 7)] for i in range(8)]
    t = {b: ex.probe_exchange(b, iters=5) for b in sizes}
    total = 0.0
    for b in group_bytes:
        near = min(sizes, key=lambda x: abs(x - b))
        total += t[near] * b / near
    bus = {str(b): (world - 1) / world * b / t[b] / 1e9 for b in sizes}
    return total, bus


def run_gpu(args, rec):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2008_11421_b200 import workloads as W
    from paper_2008_11421_b200.executor import ExecConfig, Executor
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: world size {world} != --gpus {args.gpus} (launch under torchrun with "
                         f"--nproc-per-node {args.gpus}, or without WORLD_SIZE to self-launch)")
    if os.environ.get("KRT_BENCH_SHARE_GPU") == "1":
        local = 0      # test mode: every rank on cuda:0 (IPC still crosses processes)
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but only {torch.cuda.device_count()} GPUs")
    torch.cuda.set_device(local)
    torch.backends.cudnn.benchmark = True
    nccl_id = None
    if world > 1:
        # control plane (barriers, max-over-ranks, handle exchange) over gloo;
        # the data-path exchange is the runtime's own (IPC) or NCCL
        dist.init_process_group("gloo")
        if args.exchange == "nccl":
            from paper_2008_11421_b200 import _lib
            box = [_lib.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            nccl_id = box[0]
            if rank == 0:
                print(f"bench.py: NCCL exchange communicator, nranks={world}", file=sys.stderr, flush=True)
    m = rec["meta"]
    batch = m["batch"]
    units = W.units_for(rec)
    loss_fn, opt_cfg = workload_exec(rec)
    if args.incore:
        bundle = W.bundle_for(rec, W.incore_plan(rec["plan"])).set_capacity(1e12)
        rec = dict(rec, plan=W.incore_plan(rec["plan"]), name=rec["name"] + "_incore",
                   swapped_bytes=0.0, recompute_bytes=0.0, plan_string="in-core")
    else:
        bundle = W.bundle_for(rec)
    t_setup = time.perf_counter()
    ex = Executor(units, bundle, batch=batch, loss_fn=loss_fn,
                  cfg=ExecConfig(device=local, world_size=world, rank=rank, nccl_id=nccl_id,
                                 ipc_exchange=(world > 1 and args.exchange == "ipc"),
                                 grad_slots=args.grad_slots, exchange_bf16=args.exchange_bf16,
                                 weight_dtype=torch.float32 if m.get("act") == "f32" else torch.bfloat16,
                                 **opt_cfg))
    if world > 1 and args.exchange == "ipc":
        handles = [None] * world
        dist.all_gather_object(handles, ex.ipc_handles())
        ex.ipc_connect(handles)
    ex.init_weights(seed=0)
    setup_s = time.perf_counter() - t_setup
    dev = torch.device("cuda", local)
    import math
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    x, y = workload_inputs(rec, dev, gen)
    cs = ex.compute_stream

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up --------------------------------------------------------------
    for _ in range(args.warmup):
        ex.step(x, y)
    ex.synchronize()
    barrier()
    # ---- link probes (all ranks concurrently, before the timed region) ----------
    from paper_2008_11421_b200 import _lib as _L
    block_params = [sum(sum(math.prod(p) for p in units[i - 1].param_specs())
                        for i in range(b["layers"][0], b["layers"][1] + 1)) for b in rec["plan"]["blocks"]]
    lay = _L.dp_layout(block_params, 0, world)
    group_bytes = [4 * n for n in lay["group_n"]]
    pcie = probe_pcie(dev, world) if not args.no_probe else None
    nccl_rs_s, nccl_bus = (probe_nccl(ex, group_bytes, world)
                           if world > 1 and args.exchange == "nccl" and not args.no_probe else (None, None))
    barrier()
    # ---- timed region: inputs resident in HBM ----------------------------------
    clk = Clocks(local)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ex.stats()["kernel_launches_total"]
    h2d0, d2h0 = ex.stats()["bytes_h2d_total"], ex.stats()["bytes_d2h_total"]
    from paper_2008_11421_b200 import bnfused
    e0.record(cs)
    for k in range(args.steps):
        if k == args.steps - 1:
            bnfused.PROFILE = []      # CUDA events around our kernels in the last timed step
        ex.step(x, y)
    ex.synchronize()
    e1.record(cs)
    barrier()
    prof, bnfused.PROFILE = bnfused.PROFILE, None
    ms = e0.elapsed_time(e1)
    clocks = clk.stop()
    st = ex.stats()
    trace = ex.trace_csv()
    launches = st["kernel_launches_total"] - launches0
    h2d_iter = (st["bytes_h2d_total"] - h2d0) / args.steps
    d2h_iter = (st["bytes_d2h_total"] - d2h0) / args.steps
    t = torch.tensor([ms])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * batch * args.steps / (ms / 1e3)
    # ---- e2e: host (pinned) inputs copied in, loss read back, every step --------
    xh = x.cpu().pin_memory()
    yh = y.cpu().pin_memory()
    e2e_steps = max(1, args.steps)
    # two device input buffers, alternating: step k+2's copy is ordered after
    # step k+1's loss (ex.step makes the caller's stream wait for it), hence
    # after step k's backward, the last reader of step k's input
    xbuf = [torch.empty_like(x), torch.empty_like(x)]
    ybuf = [torch.empty_like(y), torch.empty_like(y)]
    # one untimed step through the same host-input path first, like the warm-up of `value`
    xbuf[1].copy_(xh, non_blocking=True)
    ybuf[1].copy_(yh, non_blocking=True)
    float(ex.step(xbuf[1], ybuf[1]))
    ex.synchronize()
    retries0 = torch.cuda.memory_stats(dev).get("num_alloc_retries", 0)
    barrier()
    t0 = time.perf_counter()
    e2e_marks, issue_marks = [], []
    prev = None
    for k in range(e2e_steps):
        xd, yd = xbuf[k % 2], ybuf[k % 2]
        xd.copy_(xh, non_blocking=True)   # pinned host -> device, every step
        yd.copy_(yh, non_blocking=True)
        loss = ex.step(xd, yd)
        issue_marks.append(time.perf_counter() - t0)
        if prev is not None:
            float(prev)    # D2H of the previous step's loss, read once this step is queued
            e2e_marks.append(time.perf_counter() - t0)
        prev = loss
    float(prev)            # and the last step's
    e2e_marks.append(time.perf_counter() - t0)
    ex.synchronize()
    barrier()
    e2e_s = time.perf_counter() - t0
    e2e_retries = torch.cuda.memory_stats(dev).get("num_alloc_retries", 0) - retries0
    tt = torch.tensor([e2e_s])
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_value = world * batch * e2e_steps / float(tt.item())
    h2d_in = xh.numel() * xh.element_size() + yh.numel() * yh.element_size()

    # ---- roofline ---------------------------------------------------------------
    pk, pk_kind = peaks()
    iter_s = ms / 1e3 / args.steps
    fwd = sum(u.fwd_flops(batch) for u in units)
    plan = rec["plan"]
    rec_fwd = 0.0
    for s in plan["stages"]:
        for a, b in s["ops"]:
            if a == "recompute_fw":
                lo, hi = plan["blocks"][b - 1]["layers"]
                rec_fwd += sum(units[i - 1].fwd_flops(batch) for i in range(lo, hi + 1))
    alg_flops = 3.0 * fwd                     # fwd + bwd (2x) per training step
    exec_flops = alg_flops + rec_fwd          # + recomputed forwards
    sustained = pk["bf16_tflops_sustained"] * 1e12
    # PCIe at the rate measured in this run with every rank copying at once
    # (duplex when both directions move in the iteration); the probe constants
    # only when the probe was skipped
    h2d_rate = (pcie["duplex"] if d2h_iter > 0 else pcie["h2d"]) if pcie else PCIE_H2D
    d2h_rate = (pcie["duplex"] if h2d_iter > 0 else pcie["d2h"]) if pcie else PCIE_D2H
    # HBM: algorithmic bytes of every kernel of the last timed step (own
    # kernels, cuDNN convolutions, cuBLAS GEMMs; each operand read once and
    # each output written once per launch) over the measured copy bandwidth
    terms = {"compute_s": exec_flops / sustained,
             "hbm_s": 0.0,
             "pcie_h2d_s": h2d_iter / h2d_rate,
             "pcie_d2h_s": d2h_iter / d2h_rate,
             "nvlink_s": 0.0}
    nvl = None
    if world > 1:
        # reduce-scatter of the fp32 gradients: measured on the communicator at the
        # plan's group sizes; all-gather of the bf16 weights at the same bus rate
        w_bytes = st["params"] * 2
        if nccl_rs_s is not None:
            best_bus = max(nccl_bus.values()) * 1e9
            terms["nvlink_s"] = nccl_rs_s + (world - 1) / world * w_bytes / best_bus
            nvl = {"reduce_scatter_s": nccl_rs_s, "all_gather_s_est": (world - 1) / world * w_bytes / best_bus,
                   "bus_GBps_by_bytes": nccl_bus, "source": "krt_probe_exchange (ncclReduceScatter, own comm)"}
        else:
            terms["nvlink_s"] = st["params"] * (world - 1) / world * (4 + 2) / 770e9
            nvl = {"source": "B200_PROFILING.md peer copy 770 GB/s (probe skipped / IPC exchange)"}
    rows = [r.split(",") for r in trace.strip().splitlines()[1:]]
    comp = [(float(r[0]), float(r[1])) for r in rows if r[2] == "compute"]
    busy = sum(b - a for a, b in comp)
    span = (max(b for _, b in comp) - min(a for a, _ in comp)) if comp else 0.0
    xin = [(float(r[0]), float(r[1])) for r in rows if r[4] in ("swap_in", "weight_in")]
    xout = [(float(r[0]), float(r[1])) for r in rows if r[4] in ("swap_out", "grad_out")]
    # occupancy of the backward phase against the analytic model (occupancy.py:178-237):
    # steps = the compute ops from the first bw on (bw and recompute_fw), busy =
    # duration, idle = measured stall before it; theta = 0-based index of the
    # first step that waited (None: the backward phase never waited)
    comp_ops = sorted(((float(r[0]), float(r[1]), r[4], float(r[6])) for r in rows if r[2] == "compute"))
    first_bw = next((i for i, o in enumerate(comp_ops) if o[2] == "bw"), None)
    bsteps = comp_ops[first_bw:] if first_bw is not None else []
    theta_meas = next((j for j, o in enumerate(bsteps) if o[3] > 1e-3), None)
    b_busy = sum(o[1] - o[0] for o in bsteps)
    b_idle = sum(o[3] for o in bsteps)
    an = bundle.occupancy()   # analytic_report + find_theta (occupancy.py:178-225) in libkrt
    occupancy = {"theta_predicted": an["theta"], "theta_measured": theta_meas,
                 "backward_steps": len(bsteps), "backward_steps_predicted": len(an["per_step"]),
                 "backward_mean_occupancy_predicted": an["mean_occupancy"],
                 "backward_mean_occupancy_measured": b_busy / (b_busy + b_idle) if bsteps else None,
                 "per_step_predicted_vs_measured": [
                     [row[0], round(row[1], 6),
                      round((o[1] - o[0]) / ((o[1] - o[0]) + o[3]), 6) if (o[1] - o[0]) + o[3] > 0 else 1.0]
                     for row, o in zip(an["per_step"], bsteps)],
                 "note": "theta null = the device never waits on a delivery (occupancy.py:186-190); predicted = "
                         "the plan's own cost model (hardware text of the plan), measured = report_from_steps "
                         "semantics on the executor trace, a step waits when its stall_before > 1 ms"}
    busy_in = sum(b - a for a, b in xin)
    busy_out = sum(b - a for a, b in xout)
    swap_in_bytes = st["iter_bytes_h2d"]
    swap_out_bytes = st["iter_bytes_d2h"]
    # live roofline of our dominant kernel family (CUDA events on the compute stream)
    fam = {}
    for kind, nbytes, a, b, flops in prof or []:
        t = a.elapsed_time(b) * 1e-3
        f = fam.setdefault(kind, [0, 0.0, 0, 0.0, 0.0])
        f[0] += nbytes
        f[1] += t
        f[2] += 1
        f[3] += flops
        # this launch's own roofline time: the slower of its bytes at HBM
        # bandwidth and its flops at the dense bf16 peak
        f[4] += max(nbytes / (pk["hbm_gbs"] * 1e9), flops / (pk["bf16_tflops"] * 1e12))
    kernels = {}
    for k, v in fam.items():
        if v[1] <= 0:
            continue
        kernels[k] = {"launches": v[2], "ms_per_step": v[1] * 1e3, "achieved_GBps": v[0] / v[1] / 1e9,
                      "frac_of_hbm": v[0] / v[1] / 1e9 / pk["hbm_gbs"]}
        if v[3] > 0:   # tensor-core family: also against the dense bf16 peak
            kernels[k]["achieved_TFLOPs"] = v[3] / v[1] / 1e12
            kernels[k]["frac_of_tensor"] = v[3] / v[1] / 1e12 / pk["bf16_tflops"]
            # mixed HBM- and tensor-bound launches: sum of per-launch roofline
            # times (max of the two bounds) over the measured time
            kernels[k]["frac_of_roofline"] = v[4] / v[1]
    # library calls (cuDNN, cuBLAS, aten flash attention) are timed for the step
    # accounting only; the roofline and the launch count are our kernels'
    lib_fam = ("cudnn_", "cublas_", "flash_attn")
    own = {k: v for k, v in fam.items() if not k.startswith(lib_fam)}
    for k in kernels:
        kernels[k]["library"] = k.startswith(lib_fam)
    dom = max(own, key=lambda k: own[k][1]) if own else None
    step_alg_bytes = sum(v[0] for v in fam.values())
    terms["hbm_s"] = step_alg_bytes / (pk["hbm_gbs"] * 1e9)
    bind = max(terms, key=terms.get)

    def dom_roofline(k):
        v = fam[k]
        hbm = {"bound": "hbm", "kernel": k, "achieved": v[0] / v[1] / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
               "frac": v[0] / v[1] / 1e9 / pk["hbm_gbs"], "traffic": None,
               "peak_kind": f"{pk_kind} HBM copy (burst)"}
        if v[3] > 0 and v[3] / v[1] / 1e12 / pk["bf16_tflops"] > hbm["frac"]:
            return {"bound": "tensor", "kernel": k, "achieved": v[3] / v[1] / 1e12, "peak": pk["bf16_tflops"],
                    "unit": "TFLOP/s", "frac": v[3] / v[1] / 1e12 / pk["bf16_tflops"], "traffic": None,
                    "peak_kind": f"{pk_kind} dense bf16 (burst)", "hbm_frac": hbm["frac"]}
        tr = ROOT / "profiles" / "round1_s3_dominant_traffic.json"
        if tr.exists():
            d = json.loads(tr.read_text())
            if d.get("family") == k:   # ncu DRAM bytes of one launch of this family, with its algorithmic bytes
                hbm["traffic"] = d["dram_bytes_per_launch"]
                hbm["traffic_alg_bytes"] = d["alg_bytes_per_launch"]
                hbm["traffic_source"] = f"{d['kernel']}; {d['shape']}; profiles/round1_s3_dominant_traffic.json"
        return hbm
    line = {
        "metric": metric_name(rec),
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if m.get("act") == "f32" else "bf16",
        "data": "synthetic",
        "config": {"workload": rec["name"], "exchange": args.exchange if world > 1 else "none",
                   "exchange_dtype": "bf16" if args.exchange_bf16 else "fp32", "grad_slots": args.grad_slots,
                   **({"conv_math": "fp32" if args.no_tf32 else "tf32 (cuDNN default for fp32 tensors)"}
                      if m.get("act") == "f32" else {}),
                   "model": model_name(rec), "per_gpu_batch": batch,
                   "global_batch": batch * world, "input": m.get("res", m.get("seq")), "parallelism": f"dp{world}",
                   "plan": rec["plan_string"][:160] + " ...",
                   "activations_bytes": rec["total_bytes"], "hbm_bytes": 183359 * 2 ** 20,
                   "swapped_bytes": rec["swapped_bytes"], "recompute_bytes": rec["recompute_bytes"],
                   "l2": f"inputs > L2 (batch tensor {x.numel() * x.element_size() / 1e6:.0f} MB; "
                         f"{rec['total_bytes'] / 1e9:.0f} GB of activations per step)"},
        "roofline": (dict(dom_roofline(dom),
                          note="our dominant kernel family in the step (sum of algorithmic bytes or flops / sum "
                               "of CUDA-event durations over one timed step, on the compute stream)")
                     if dom else None),
        "kernels": kernels,
        "step_roofline": {"bound": "tensor", "achieved": alg_flops / iter_s / 1e12,
                          "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                          "frac": alg_flops / iter_s / sustained,
                          "peak_kind": f"{pk_kind} sustained bf16 (cuBLAS)",
                          "note": "whole training step: algorithmic 3x forward FLOPs / step time; "
                                  "convolutions are cuDNN (sm100 tcgen05 kernels)"},
        "iteration_roofline": dict(terms, binding=bind, bound_s=terms[bind],
                                   frac=terms[bind] / iter_s,
                                   pcie_h2d_GBps=swap_in_bytes / iter_s / 1e9,
                                   pcie_d2h_GBps=swap_out_bytes / iter_s / 1e9,
                                   # while a transfer is in flight, against the probed link rate
                                   pcie_h2d_active_GBps=(swap_in_bytes / busy_in / 1e9) if busy_in else None,
                                   pcie_d2h_active_GBps=(swap_out_bytes / busy_out / 1e9) if busy_out else None,
                                   pcie_h2d_active_frac_of_link=(swap_in_bytes / busy_in / (pcie["h2d"] if pcie else PCIE_H2D))
                                   if busy_in else None,
                                   pcie_d2h_active_frac_of_link=(swap_out_bytes / busy_out / (pcie["d2h"] if pcie else PCIE_D2H))
                                   if busy_out else None,
                                   pcie_link_GBps=({k: (v / 1e9 if k in ("h2d", "d2h", "duplex") else v)
                                                    for k, v in pcie.items()} if pcie else
                                                   {"h2d": PCIE_H2D / 1e9, "d2h": PCIE_D2H / 1e9,
                                                    "source": "scripts/probe_box.py constants (probe skipped)"}),
                                   hbm_step_alg_bytes=step_alg_bytes,
                                   nvlink=nvl),
        "overlap": {"compute_busy_frac": busy / span if span else None,
                    "exposed_stall_frac": 1 - busy / span if span else None,
                    "swap_in_busy_s": sum(b - a for a, b in xin),
                    "swap_out_busy_s": sum(b - a for a, b in xout)},
        "occupancy": occupancy,
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d_in,
                "d2h_bytes_per_step": 4, "steps": e2e_steps,
                "loss_read_s": [round(t, 4) for t in e2e_marks], "issued_s": [round(t, 4) for t in issue_marks],
                "total_s": round(e2e_s, 4),
                "note": "every step: pinned H2D of its inputs, issue, then D2H read of the previous step's loss "
                        "(the last loss read after the loop)",
                "alloc_retries": e2e_retries},
        "gpu_launches": launches + sum(v[2] for v in own.values()) * args.steps,
        "runtime": {k: st[k] for k in ("arena_bytes", "ledger_peak_bytes", "host_swap_bytes",
                                       "swapped_blocks", "ops_per_iteration", "params")},
        "setup_s": setup_s,
        "device_memory": {"torch_max_allocated": torch.cuda.max_memory_allocated(dev),
                          "free_total": list(torch.cuda.mem_get_info(dev))},
        "clocks": clocks,
    }
    if args.trace_out and rank == 0:
        Path(args.trace_out).write_text(trace)
    ex.close()
    del ex
    if rank == 0:
        # HardwareSpec fields measured on this box (calibrate.py):
        # the planner's inputs, from the trace of this run and the probes
        from paper_2008_11421_b200 import calibrate
        host = calibrate.host_update_rate()
        pl = pcie or {"h2d": PCIE_H2D, "d2h": PCIE_D2H, "duplex": PCIE_DUPLEX}
        cal = calibrate.calibrate(bundle, trace, pk, {k: pl[k] / 1e9 for k in ("h2d", "d2h", "duplex")}, host)
        cal["hw_text"] = calibrate.hw_text(calibrate.capacity_of(rec["hardware"]), cal)
        line["calibration"] = cal
    if rank == 0 and not args.no_cpu_baseline:
        line["reference_planner"] = reference_planner_time(rec, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, dt = cpu_reference(rec, steps=2, warmup=1)
        line["cpu_baseline"] = {"value": v, "unit": "samples/s", "cores": cores, "kind": "port",
                                "sample": f"in-core fp32 torch-CPU {model_name(rec)} step "
                                          f"(oracle/), {cpu_sample_batch(rec)} samples x 2 steps"
                                          f"{cpu_sample_note(rec)}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--plan", default="resnet200_b3072")
    ap.add_argument("--impl", default="krt", choices=["krt", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace-out", default=None)
    ap.add_argument("--exchange", default="nccl", choices=["ipc", "nccl"],
                    help="N>1 gradient exchange: NCCL reduce-scatter/all-gather on the runtime's own "
                         "communicator (default), or the runtime's reduce over CUDA IPC peer memory")
    ap.add_argument("--no-probe", action="store_true", help="skip the PCIe / NCCL link probes")
    ap.add_argument("--grad-slots", type=int, default=0,
                    help="gradient ring of R group-sized slots instead of a whole-model region (0: off)")
    ap.add_argument("--exchange-bf16", action="store_true",
                    help="N>1 NCCL exchange: bf16 cast pack before the reduce-scatter (half the NVLink bytes)")
    ap.add_argument("--incore", action="store_true",
                    help="same blocks, everything resident (no swap/recompute): the in-core baseline")
    ap.add_argument("--no-tf32", action="store_true",
                    help="fp32 workloads: cuDNN / cuBLAS in true fp32 (default: their TF32 tensor-core math)")
    args = ap.parse_args()
    if args.no_tf32:
        import torch
        torch.backends.cudnn.allow_tf32 = False
        torch.backends.cuda.matmul.allow_tf32 = False
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    from paper_2008_11421_b200 import workloads as W
    rec = W.load(args.plan)
    if args.impl == "reference":
        run_reference(args, rec)
    else:
        run_gpu(args, rec)


if __name__ == "__main__":
    main()
