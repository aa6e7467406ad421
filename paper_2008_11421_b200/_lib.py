"""ctypes binding of libkrt.so (include/krt.h).

This is the reference-side FFI for the executor path: the reference package is
Python, so its natural binding to a C ABI is ctypes.  The library is built
in-tree by ``__graft_entry__.build()``; importing this module without it
raises immediately — there is no Python fallback for any runtime op.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).with_name("libkrt.so")

KRT_OK, KRT_INFEASIBLE, KRT_USAGE, KRT_INTERNAL = 0, 1, 2, 3
FW, BW, SWAP_IN, SWAP_OUT, RECOMPUTE_FW, WEIGHT_IN, GRAD_OUT, EXCHANGE, HOST_UPDATE = range(9)
ACTION_NAMES = ("fw", "bw", "swap_in", "swap_out", "recompute_fw",
                "weight_in", "grad_out", "exchange", "host_update")
F32, BF16 = 0, 1
SGD, ADAM = 0, 1
REGION_WEIGHTS, REGION_GRADS, REGION_ARENA, REGION_HOST_SWAP = 0, 1, 2, 3


class KrtError(RuntimeError):
    """A non-zero krt status; ``code`` mirrors the reference CLI exit codes."""

    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"krt error {code}: {msg}")


class InfeasiblePlanError(KrtError):
    pass


class DistConfig(C.Structure):
    _fields_ = [("workers", C.c_int), ("ring", C.c_int), ("net_bw", C.c_double),
                ("net_latency", C.c_double), ("groups", C.c_int), ("variant", C.c_int)]


class Config(C.Structure):
    _fields_ = [("device", C.c_int), ("world_size", C.c_int), ("rank", C.c_int),
                ("nccl_id", C.c_void_p), ("dist_groups", C.c_int), ("weight_dtype", C.c_int),
                ("optimizer", C.c_int), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float),
                ("momentum", C.c_float), ("grad_scale", C.c_float), ("host_threads", C.c_int),
                ("arena_slack_bytes", C.c_size_t), ("peer_group", C.c_void_p),
                ("host_path_all", C.c_int), ("force_dp_path", C.c_int), ("ipc_exchange", C.c_int),
                ("grad_slots", C.c_int), ("exchange_bf16", C.c_int)]


COMPUTE_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p)

EXPORTS = {
    "krt_last_error": (C.c_char_p, []),
    "krt_version": (C.c_char_p, []),
    "krt_string_free": (None, [C.c_void_p]),
    "krt_plan_load": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "krt_plan_free": (None, [C.c_void_p]),
    "krt_plan_model": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int,
                                 C.POINTER(C.c_void_p)]),
    "krt_plan_set_capacity": (C.c_int, [C.c_void_p, C.c_double]),
    "krt_plan_string": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "krt_plan_json": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "krt_plan_validate": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int)]),
    "krt_plan_simulate": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "krt_plan_occupancy": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "krt_plan_costs": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "krt_plan_simulate_dist": (C.c_int, [C.c_void_p, C.POINTER(DistConfig), C.c_int,
                                         C.POINTER(C.c_void_p)]),
    "krt_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "krt_dp_layout": (C.c_int, [C.POINTER(C.c_int64), C.c_int, C.c_int, C.c_int,
                                C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "krt_peer_group_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "krt_peer_group_destroy": (C.c_int, [C.c_void_p]),
    "krt_plan_arena": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.c_int, C.POINTER(C.c_void_p)]),
    "krt_probe_exchange": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.POINTER(C.c_double)]),
    "krt_create": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "krt_destroy": (C.c_int, [C.c_void_p]),
    "krt_register_block": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t, C.POINTER(C.c_int64), C.c_int]),
    "krt_prepare": (C.c_int, [C.c_void_p, C.c_void_p]),
    "krt_region": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                             C.POINTER(C.c_size_t)]),
    "krt_stream": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "krt_block_slot": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "krt_init_master": (C.c_int, [C.c_void_p]),
    "krt_run_iteration": (C.c_int, [C.c_void_p, COMPUTE_CB, C.c_void_p]),
    "krt_synchronize": (C.c_int, [C.c_void_p]),
    "krt_flush_weights": (C.c_int, [C.c_void_p]),
    "krt_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "krt_ipc_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "krt_trace_csv": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "krt_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "krt_read_master": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_float), C.c_size_t]),
    "krt_reduce_cast": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_int, C.c_size_t,
                                  C.c_float, C.c_void_p]),
    "krt_device_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int, C.c_size_t, C.c_int, C.c_float, C.c_float, C.c_float,
                                    C.c_float, C.c_float, C.c_float, C.c_int, C.c_void_p]),
    "krt_checkpoint_save": (C.c_int, [C.c_void_p, C.c_char_p]),
    "krt_checkpoint_load": (C.c_int, [C.c_void_p, C.c_char_p]),
    "krt_bn_workspace_bytes": (C.c_size_t, [C.c_int]),
    "krt_bn_stats": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_float, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]),
    "krt_bn_stats_apply": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_float] + [C.c_void_p] * 5
                           + [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "krt_bn_add_relu_backward": (C.c_int, [C.c_void_p] * 12 + [C.c_int64, C.c_int, C.c_void_p, C.c_void_p]),
    "krt_bn_relu_maxpool": (C.c_int, [C.c_void_p] * 6 + [C.c_int] * 7 + [C.c_void_p]),
    "krt_bn_relu_maxpool_bwd_workspace": (C.c_size_t, [C.c_int] * 7),
    "krt_bn_relu_maxpool_bwd": (C.c_int, [C.c_void_p] * 8 + [C.c_int] * 7 + [C.c_void_p]),
    "krt_conv1x1_partials_bytes": (C.c_size_t, [C.c_int]),
    "krt_conv1x1_bn": (C.c_int, [C.c_void_p] * 3 + [C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 6
                       + [C.c_void_p]),
    "krt_conv1x1_bn_res": (C.c_int, [C.c_void_p] * 3 + [C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 8),
    "krt_pad_rgb4": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "krt_conv_gather_bn": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 11 + [C.c_void_p] * 3),
    "krt_conv_im2col_bn": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 10 + [C.c_void_p] * 12),
    "krt_conv_wgrad_workspace_bytes": (C.c_size_t, [C.c_int] * 6),
    "krt_conv3x3_halo_supported": (C.c_int, [C.c_int] * 5),
    "krt_stem_wgrad_workspace": (C.c_size_t, []),
    "krt_stem_wgrad": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 3 + [C.c_void_p, C.c_size_t, C.c_void_p]),
    "krt_wgrad1x1_narrow_supported": (C.c_int, [C.c_int] * 2),
    "krt_wgrad1x1_narrow_workspace": (C.c_size_t, [C.c_int] * 2),
    "krt_wgrad1x1_narrow": (C.c_int, [C.c_void_p] * 3 + [C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 5
                            + [C.c_size_t, C.c_void_p]),
    "krt_wgrad3x3_narrow_supported": (C.c_int, [C.c_int] * 3),
    "krt_wgrad3x3_narrow_workspace": (C.c_size_t, [C.c_int]),
    "krt_wgrad3x3_narrow": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 4 + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p]),
    "krt_mlp_fc1_gelu": (C.c_int, [C.c_void_p] * 5 + [C.c_int64] * 3 + [C.c_void_p]),
    "krt_mlp_fc2_dgelu": (C.c_int, [C.c_void_p] * 4 + [C.c_int64] * 3 + [C.c_void_p]),
    "krt_mlp_fc2_residual": (C.c_int, [C.c_void_p] * 5 + [C.c_int64] * 3 + [C.c_void_p]),
    "krt_linear_wgrad_bgrad": (C.c_int, [C.c_void_p] * 4 + [C.c_int64] * 3 + [C.c_void_p]),
    "krt_conv_wgrad": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 10 + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p]),
    "krt_conv1x1_bn_dgrad": (C.c_int, [C.c_void_p] * 3 + [C.c_int64, C.c_int, C.c_int] + [C.c_void_p] * 8),
    "krt_bn_partials_bwd_finalize": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64] + [C.c_void_p] * 7),
    "krt_bn_backward_elemt": (C.c_int, [C.c_void_p] * 8 + [C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "krt_bn_partials_finalize": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_float, C.c_void_p,
                                           C.c_void_p, C.c_void_p]),
    "krt_ln_fwd": (C.c_int, [C.c_void_p] * 8 + [C.c_int64, C.c_int, C.c_float, C.c_void_p]),
    "krt_ln_bwd_workspace": (C.c_size_t, [C.c_int64, C.c_int]),
    "krt_ln_bwd": (C.c_int, [C.c_void_p] * 10 + [C.c_int64, C.c_int, C.c_void_p]),
    "krt_attn_softmax_bwd": (C.c_int, [C.c_void_p] * 6 + [C.c_int64, C.c_int, C.c_float, C.c_void_p]),
    "krt_lm_xent": (C.c_int, [C.c_void_p] * 4 + [C.c_int64, C.c_int, C.c_float, C.c_void_p]),
    "krt_gelu_bwd_colsum_workspace": (C.c_size_t, [C.c_int64, C.c_int]),
    "krt_gelu_bwd_colsum": (C.c_int, [C.c_void_p] * 5 + [C.c_int64, C.c_int, C.c_void_p]),
    "krt_bn_apply": (C.c_int, [C.c_void_p] * 10 + [C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "krt_bn_add_relu_bwd": (C.c_int, [C.c_void_p] * 13 + [C.c_int64, C.c_int, C.c_void_p]),
    "krt_bn_backward": (C.c_int, [C.c_void_p] * 6 + [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                                   C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "krt_host_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_int, C.c_size_t, C.c_int, C.c_float, C.c_float, C.c_float,
                                  C.c_float, C.c_float, C.c_float, C.c_int, C.c_int]),
}

_lib = None


def lib():
    """Load libkrt.so once; raises if the in-tree build is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the runtime has no Python fallback)")
        # torch first: its bundled libnccl.so.2 (newer than the system one) must
        # be the copy the process resolves; libkrt links NCCL by soname.
        import torch  # noqa: F401
        handle = C.CDLL(os.fspath(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(code: int):
    if code != KRT_OK:
        msg = lib().krt_last_error().decode("utf-8", "replace")
        if code == KRT_INFEASIBLE:
            raise InfeasiblePlanError(code, msg)
        raise KrtError(code, msg)


def take_string(ptr: C.c_void_p) -> str:
    """Copy a malloc'ed C string returned through an out-pointer and free it."""
    try:
        return C.string_at(ptr.value).decode("utf-8")
    finally:
        lib().krt_string_free(ptr)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().krt_nccl_unique_id(buf))
    return buf.raw


class PeerGroup:
    """In-process exchange group (krt_peer_group) for ranks driven by threads."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib().krt_peer_group_create(world, C.byref(h)))
        self.handle = h
        self.world = world

    def close(self):
        if self.handle is not None and self.handle.value:
            lib().krt_peer_group_destroy(self.handle)
            self.handle = None


def dp_layout(block_params, groups: int, world: int) -> dict:
    """krt_dp_layout: the runtime's flat parameter / shard layout."""
    nb = len(block_params)
    bp = (C.c_int64 * nb)(*block_params)
    off = (C.c_int64 * nb)()
    lo, n, sh = (C.c_int64 * nb)(), (C.c_int64 * nb)(), (C.c_int64 * nb)()
    ng = C.c_int()
    check(lib().krt_dp_layout(bp, nb, groups, world, off, C.byref(ng), lo, n, sh))
    k = ng.value
    return {"block_off": list(off), "group_lo": list(lo)[:k], "group_n": list(n)[:k],
            "shard_n": list(sh)[:k]}
