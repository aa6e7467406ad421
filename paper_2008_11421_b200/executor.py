"""Per-rank executor: binds a model's units to a KARMA plan and runs training
iterations through libkrt (include/krt.h).

What the runtime (C++/CUDA) owns: the device arena and its static slot
assignment, the pinned-host swap area, the copy-engine transfers
(swap_in/swap_out/grad_out/weight_in), the exchange, the host/device
optimizer and the issue order of every op with its CUDA-event dependencies.
What this module owns: the compute callback — each plan op's forward /
recomputed forward / backward of a block, issued on the runtime's compute
stream with the block's saved tensors living inside its arena slot.

Reference anchors: op vocabulary plan.py:24-29; residency demands
plan.py:129-138 (fw b needs b-1, recompute b needs b-1 and skip sources, bw b
needs b); the 5-stage DP pipeline distsim.py:140-236 / PAPER.md:449-453.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import torch

from . import _lib
from .plan import PlanBundle

ALIGN = 256


def _align(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


class _CudaBuf:
    """Exposes a raw device pointer through __cuda_array_interface__ (zero copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_bytes(ptr: int, nbytes: int, device: torch.device) -> torch.Tensor:
    """uint8 torch view of device memory owned by libkrt."""
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device=device)


def _view(buf: torch.Tensor, off: int, shape, dtype) -> torch.Tensor:
    n = math.prod(shape) * torch.empty((), dtype=dtype).element_size()
    return buf[off:off + n].view(dtype).view(shape)


@dataclass
class SavedSpec:
    shape: tuple
    dtype: torch.dtype

    @property
    def nbytes(self) -> int:
        return math.prod(self.shape) * torch.empty((), dtype=self.dtype).element_size()


class Unit:
    """One executor layer (= one layer of the model IR handed to the planner).

    Subclasses declare their parameters and the tensors they save for
    backward; the first saved tensor is always the unit's input, so a block's
    backward never needs another block (plan.py:136-137) and a recompute can
    regenerate its input from the previous block's last unit (plan.py:133-135).
    """

    name = "unit"

    def param_specs(self) -> list[tuple]:
        return []

    def saved_specs(self, batch: int) -> list[SavedSpec]:
        raise NotImplementedError

    def forward(self, x: torch.Tensor, params: list, saved: Optional[list]) -> torch.Tensor:
        raise NotImplementedError

    def backward(self, dy: torch.Tensor, params: list, saved: list, grads: list) -> torch.Tensor:
        raise NotImplementedError

    def init_params(self, gen: torch.Generator) -> list[torch.Tensor]:
        return []

    def saved_input(self, saved: list) -> torch.Tensor:
        """The unit's input as forward() takes it, rebuilt from its saved tensors."""
        return saved[0]

    def fwd_flops(self, batch: int) -> float:
        return 0.0

    def saved_bytes(self, batch: int) -> int:
        return sum(_align(s.nbytes) for s in self.saved_specs(batch))

    def ir_line(self, lid: int, batch: int) -> str:
        """Model-IR record (model_ir.py:8-25) with measured memory overrides."""
        raise NotImplementedError


@dataclass
class ExecConfig:
    device: int = 0
    world_size: int = 1
    rank: int = 0
    nccl_id: Optional[bytes] = None
    dist_groups: int = 0
    weight_dtype: torch.dtype = torch.float32
    optimizer: str = "sgd"           # "sgd" | "adam"
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    momentum: float = 0.0
    host_threads: int = 0
    arena_slack_bytes: int = 0
    peer_group: Optional[object] = None   # _lib.PeerGroup for in-process ranks
    host_path_all: bool = False           # host update for every block even at world_size 1
    force_dp_path: bool = False           # DP op structure through a 1-rank NCCL communicator
    ipc_exchange: bool = False            # exchange over CUDA IPC peer memory (multi-process)
    grad_slots: int = 0                   # 0: whole-model gradient region; R: ring of R group slots
    exchange_bf16: bool = False           # NCCL reduce-scatter of bf16-packed gradients


class Executor:
    """Runs the plan's iterations for ``units`` grouped by the plan's blocks."""

    def __init__(self, units: Sequence[Unit], bundle: PlanBundle, batch: int,
                 loss_fn: Callable, cfg: ExecConfig = ExecConfig()):
        self.units = list(units)
        for prev, u in zip(self.units, self.units[1:]):
            if hasattr(u, "prev_unit"):   # the unit whose forward output u takes (units.py STATS_HANDOFF)
                u.prev_unit = prev
        self.bundle = bundle
        self.batch = batch
        self.loss_fn = loss_fn
        self.cfg = cfg
        self.dev = torch.device("cuda", cfg.device)
        torch.cuda.set_device(self.dev)
        plan = bundle.to_dict()
        self.plan = plan
        self.blocks = [(b["id"], b["layers"][0], b["layers"][1]) for b in plan["blocks"]]
        self.nb = len(self.blocks)
        if self.blocks[-1][2] != len(self.units):
            raise ValueError(f"plan covers {self.blocks[-1][2]} layers, model has {len(self.units)} units")
        L = _lib.lib()
        wdt = _lib.BF16 if cfg.weight_dtype == torch.bfloat16 else _lib.F32
        self._nccl_id_buf = (C.create_string_buffer(cfg.nccl_id, 128) if cfg.nccl_id else None)
        kc = _lib.Config(cfg.device, cfg.world_size, cfg.rank,
                         C.cast(self._nccl_id_buf, C.c_void_p) if self._nccl_id_buf else None,
                         cfg.dist_groups, wdt, _lib.ADAM if cfg.optimizer == "adam" else _lib.SGD,
                         cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay, cfg.momentum,
                         1.0 / cfg.world_size, cfg.host_threads, cfg.arena_slack_bytes,
                         cfg.peer_group.handle if cfg.peer_group is not None else None,
                         int(cfg.host_path_all), int(cfg.force_dp_path), int(cfg.ipc_exchange),
                         int(cfg.grad_slots), int(cfg.exchange_bf16))
        h = C.c_void_p()
        _lib.check(L.krt_create(C.byref(kc), C.byref(h)))
        self._ctx = h
        # slot layout per block: units' saved tensors back to back, 256-B aligned
        self.layout = {}
        for bid, lo, hi in self.blocks:
            off = 0
            per_unit = []
            numels = []
            for u in self.units[lo - 1:hi]:
                offs = []
                for s in u.saved_specs(batch):
                    offs.append((off, s))
                    off += _align(s.nbytes)
                per_unit.append(offs)
                numels += [math.prod(p) for p in u.param_specs()]
            self.layout[bid] = per_unit
            arr = (C.c_int64 * max(1, len(numels)))(*numels)
            _lib.check(L.krt_register_block(self._ctx, bid, off, arr, len(numels)))
        _lib.check(L.krt_prepare(self._ctx, bundle.handle))
        self._bind_regions()
        self._streams = {}
        s = C.c_void_p()
        _lib.check(L.krt_stream(self._ctx, 0, C.byref(s)))
        self.compute_stream = torch.cuda.ExternalStream(s.value, device=self.dev)
        self._cb = _lib.COMPUTE_CB(self._callback)
        self._loss_ready = torch.cuda.Event()
        self.handoff = None       # (block, activation) between consecutive forwards
        self.grad_handoff = None  # (block, gradient) between backwards
        self.input = None
        self.target = None
        self.loss = None
        self._error = None

    # ------------------------------------------------------------------ memory
    def _region(self, which, block=0):
        p, n = C.c_void_p(), C.c_size_t()
        _lib.check(_lib.lib().krt_region(self._ctx, which, block, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def _bind_regions(self):
        ap, an = self._region(_lib.REGION_ARENA)
        self.arena = device_bytes(ap, an, self.dev)
        self.arena_base = ap
        self.params = {}   # unit index -> list of weight views
        self.grads = {}    # unit index -> list of fp32 grad views
        for bid, lo, hi in self.blocks:
            wp, wn = self._region(_lib.REGION_WEIGHTS, bid)
            gp, gn = self._region(_lib.REGION_GRADS, bid)
            wbuf = device_bytes(wp, wn, self.dev)
            gbuf = device_bytes(gp, gn, self.dev)
            woff = goff = 0
            for ui in range(lo, hi + 1):
                u = self.units[ui - 1]
                pv, gv = [], []
                for shp in u.param_specs():
                    n = math.prod(shp)
                    pv.append(wbuf[woff:woff + n * self._wsize].view(self.cfg.weight_dtype).view(shp))
                    gv.append(gbuf[goff:goff + n * 4].view(torch.float32).view(shp))
                    woff += n * self._wsize
                    goff += n * 4
                self.params[ui] = pv
                self.grads[ui] = gv

    @property
    def _wsize(self):
        return 2 if self.cfg.weight_dtype == torch.bfloat16 else 4

    def load_weights(self, weights: dict):
        """weights: unit index -> list of tensors (any device/dtype)."""
        for ui, ts in weights.items():
            for dst, src in zip(self.params[ui], ts):
                dst.copy_(src.to(device=self.dev, dtype=dst.dtype))
        torch.cuda.synchronize(self.dev)
        _lib.check(_lib.lib().krt_init_master(self._ctx))

    def init_weights(self, seed: int = 0):
        g = torch.Generator().manual_seed(seed)
        self.load_weights({i + 1: u.init_params(g) for i, u in enumerate(self.units)})

    def master(self, block: int) -> torch.Tensor:
        n = sum(math.prod(p) for ui in range(self.blocks[block - 1][1], self.blocks[block - 1][2] + 1)
                for p in self.units[ui - 1].param_specs())
        out = torch.empty(max(n, 1), dtype=torch.float32)
        _lib.check(_lib.lib().krt_read_master(self._ctx, block,
                                              C.cast(out.data_ptr(), C.POINTER(C.c_float)), n))
        return out[:n]

    def ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(256)
        n = C.c_size_t()
        _lib.check(_lib.lib().krt_ipc_export(self._ctx, buf, 256, C.byref(n)))
        return buf.raw[:n.value]

    def ipc_connect(self, all_handles: list):
        """all_handles: every rank's ipc_handles(), in rank order."""
        blob = b"".join(all_handles)
        _lib.check(_lib.lib().krt_ipc_import(self._ctx, blob, len(all_handles)))

    def save_checkpoint(self, path):
        """Write this rank's training state (weights, fp32 masters, optimizer
        moments, iteration counter) to `path` once the last step completed."""
        _lib.check(_lib.lib().krt_checkpoint_save(self._ctx, str(path).encode()))

    def load_checkpoint(self, path):
        """Restore a state saved by save_checkpoint into this prepared executor
        (same units, plan, dtype, world size and rank); the next step continues
        exactly where the saved run stopped."""
        _lib.check(_lib.lib().krt_checkpoint_load(self._ctx, str(path).encode()))

    def flush_weights(self):
        """Return host-updated weights to the device now (krt_flush_weights)."""
        _lib.check(_lib.lib().krt_flush_weights(self._ctx))

    def unit_weights(self) -> dict:
        """Current weights per unit, host-path updates included."""
        self.flush_weights()
        return {ui: [p.detach().clone() for p in ps] for ui, ps in self.params.items()}

    # ------------------------------------------------------------------ compute
    def _slot_views(self, block: int, slot_ptr: int):
        base = slot_ptr - self.arena_base
        out = []
        for offs in self.layout[block]:
            out.append([_view(self.arena, base + o, s.shape, s.dtype) for o, s in offs])
        return out

    def _block_input(self, b: int):
        if b == 1:
            return self.input
        if self.handoff is not None and self.handoff[0] == b - 1:
            return self.handoff[1]
        # regenerate from block b-1's last unit, resident per plan.py:133-135
        p = C.c_void_p()
        _lib.check(_lib.lib().krt_block_slot(self._ctx, b - 1, C.byref(p)))
        prev_views = self._slot_views(b - 1, p.value)
        _, lo, hi = self.blocks[b - 2]
        u = self.units[hi - 1]
        return u.forward(u.saved_input(prev_views[-1]), self.params[hi], None)

    def _callback(self, user, action, block, slot, slot_bytes, stream):
        try:
            with torch.cuda.stream(self.compute_stream):
                self._compute(action, block, slot)
            return 0
        except BaseException as exc:   # never unwind through C
            self._error = exc
            return 1

    def _compute(self, action, b, slot):
        _, lo, hi = self.blocks[b - 1]
        views = self._slot_views(b, slot)
        if action in (_lib.FW, _lib.RECOMPUTE_FW):
            x = self._block_input(b)
            n = hi - lo + 1
            for k, ui in enumerate(range(lo, hi + 1)):
                u = self.units[ui - 1]
                if k + 1 < n and getattr(u, "writes_out", False):
                    # write straight into the next unit's saved-input slot
                    nxt = self.units[ui]
                    x = u.forward(x, self.params[ui], views[k], out=nxt.saved_input(views[k + 1]))
                else:
                    x = u.forward(x, self.params[ui], views[k])
            self.handoff = (b, x)
            if action == _lib.FW and b == self.nb:
                self.loss, dy = self.loss_fn(x, self.target)
                self.grad_handoff = (b, dy)
                self._loss_ready.record(self.compute_stream)
        elif action == _lib.BW:
            if self.grad_handoff is None or self.grad_handoff[0] != b:
                raise RuntimeError(f"backward of block {b} without its output gradient")
            dy = self.grad_handoff[1]
            for k, ui in reversed(list(enumerate(range(lo, hi + 1)))):
                dy = self.units[ui - 1].backward(dy, self.params[ui], views[k], self.grads[ui])
            self.grad_handoff = (b - 1, dy)
        else:
            raise RuntimeError(f"unexpected compute action {action}")

    # ------------------------------------------------------------------ driver
    def step(self, x: torch.Tensor, target=None):
        """One training iteration; returns the (device) loss of this rank."""
        self.input, self.target = x, target
        self.handoff = self.grad_handoff = None
        self._error = None
        # inputs were produced on the caller's stream
        self.compute_stream.wait_stream(torch.cuda.current_stream(self.dev))
        rc = _lib.lib().krt_run_iteration(self._ctx, self._cb, None)
        # the caller's stream waits for the loss only, not for the backward
        # still queued behind it, so the host can issue the next iteration
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_event(self._loss_ready)
        if self.loss is not None:
            self.loss.record_stream(cur)
        if self._error is not None:
            err, self._error = self._error, None
            raise err
        _lib.check(rc)
        return self.loss

    def probe_exchange(self, nbytes: int, iters: int = 5) -> float:
        """Mean seconds of one reduce-scatter of `nbytes` fp32 on this rank's
        NCCL communicator (krt_probe_exchange; collective: call on every rank)."""
        sec = C.c_double()
        _lib.check(_lib.lib().krt_probe_exchange(self._ctx, int(nbytes), iters, C.byref(sec)))
        return sec.value

    def synchronize(self):
        _lib.check(_lib.lib().krt_synchronize(self._ctx))

    def trace_csv(self) -> str:
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_trace_csv(self._ctx, C.byref(out)))
        return _lib.take_string(out)

    def stats(self) -> dict:
        import json
        out = C.c_void_p()
        _lib.check(_lib.lib().krt_stats(self._ctx, C.byref(out)))
        return json.loads(_lib.take_string(out))

    def stream_ptr(self, which: int) -> int:
        s = C.c_void_p()
        _lib.check(_lib.lib().krt_stream(self._ctx, which, C.byref(s)))
        return s.value

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            try:
                torch.cuda.synchronize(self.dev)
            except Exception:
                pass
            self.arena = None
            self.params = self.grads = None
            _lib.lib().krt_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
