"""World-size-2 data-parallel host logic on CPU (gloo stands in for NCCL).

Each rank runs the executor's DP host path with the product's pieces: the
flat parameter / shard layout (krt_dp_layout) and the host optimizer
(krt_host_update) on its 1/P shard of every group, in reverse group order
(distsim.py:217-236), then all-gathers the updated shards.  Gradients come
from the cfg0 oracle's forward/backward (test infrastructure).  Both ranks
must end bit-identical and match the 2-worker in-core oracle."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fc_chain_oracle as orc
from paper_2008_11421_b200 import _lib


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, optimizer, lr, groups, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ws = [torch.from_numpy(w.copy()) for w in orc.init_weights()]
        n_each = [w.numel() for w in ws]
        lay = _lib.dp_layout(n_each, groups, world)
        total = lay["group_lo"][-1] + lay["group_n"][-1]
        flat_w = torch.zeros(total)
        for b, w in enumerate(ws):
            flat_w[lay["block_off"][b]:lay["block_off"][b] + w.numel()] = w.flatten()
        # host state: this rank's shard of every group
        shards = []
        for lo, n, sh in zip(lay["group_lo"], lay["group_n"], lay["shard_n"]):
            s0 = lo + rank * sh
            shards.append(dict(lo=lo, n=n, sh=sh, s0=s0, p=flat_w[s0:s0 + sh].clone(),
                               m=torch.zeros(sh), v=torch.zeros(sh), w=torch.zeros(sh)))
        L = _lib.lib()
        losses = []
        for it in range(1, 4):
            cur = [flat_w[lay["block_off"][b]:lay["block_off"][b] + n_each[b]].view(64, 64).numpy()
                   for b in range(6)]
            loss, grads = orc.forward_backward(cur, orc.inputs(rank, it))
            losses.append(loss)
            flat_g = torch.zeros(total)
            for b, g in enumerate(grads):
                flat_g[lay["block_off"][b]:lay["block_off"][b] + g.size] = torch.from_numpy(g).flatten()
            for gi in reversed(range(len(shards))):          # end of the model first
                s = shards[gi]
                recv = torch.zeros(s["sh"])
                dist.all_reduce(gsum := flat_g[s["lo"]:s["lo"] + s["n"]].clone())
                recv.copy_(gsum[rank * s["sh"]:(rank + 1) * s["sh"]])
                recv.mul_(1.0 / world)                       # grad_scale, as the runtime applies it
                _lib.check(L.krt_host_update(s["p"].data_ptr(), s["m"].data_ptr(), s["v"].data_ptr(),
                                             recv.data_ptr(), s["w"].data_ptr(), _lib.F32, s["sh"],
                                             _lib.ADAM if optimizer == "adam" else _lib.SGD, lr, 0.9,
                                             0.999, 1e-8, 0.0, 0.0, it, 2))
                parts = [torch.zeros(s["sh"]) for _ in range(world)]
                dist.all_gather(parts, s["w"])
                flat_w[s["lo"]:s["lo"] + s["n"]] = torch.cat(parts)
        final = [flat_w[lay["block_off"][b]:lay["block_off"][b] + n_each[b]].view(64, 64).numpy().copy()
                 for b in range(6)]
        out_q.put((rank, losses, final))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("optimizer,lr,groups", [("sgd", 1e-2, 0), ("adam", 1e-3, 2)])
def test_two_rank_dp_host_path(optimizer, lr, groups):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, optimizer, lr, groups, q)) for r in range(2)]
    [p.start() for p in procs]
    res = dict()
    for _ in range(2):
        r, losses, final = q.get(timeout=240)
        res[r] = (losses, final)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    ref_losses, ref_w = orc.train(workers=2, iterations=3, optimizer=optimizer, lr=lr)
    for r in (0, 1):
        np.testing.assert_allclose(res[r][0], [l[r] for l in ref_losses], rtol=1e-5)
    atol = 1e-6 if optimizer == "sgd" else 1e-5
    for a, b, ref in zip(res[0][1], res[1][1], ref_w):
        assert np.array_equal(a, b)
        np.testing.assert_allclose(a, ref, rtol=1e-5, atol=atol)


def test_layout_shards_are_aligned_and_cover():
    lay = _lib.dp_layout([4096, 100, 7, 0, 5000], 2, 8)
    for lo, n, sh in zip(lay["group_lo"], lay["group_n"], lay["shard_n"]):
        assert n % (8 * 64) == 0 and sh * 8 == n and lo % 64 == 0
    assert lay["block_off"][:3] == [0, 4096, 4224]   # blocks 64-element aligned
    assert all(o % 64 == 0 for o in lay["block_off"])
