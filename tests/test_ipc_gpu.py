"""Multi-process data parallelism over CUDA IPC peer memory (ipc_exchange):
two processes, one rank each, exchange gradients with the runtime's own
reduce kernel reading the peer's gradient region and gather weight shards
with device-to-device copies, ordered by stream-memory-op flags.  Both
processes share cuda:0 here (one GPU per gpurun); across GPUs the same
pointers are NVLink peer mappings.  cfg0 with 2 workers vs the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, optimizer, lr, q):
    import json
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    from oracle import fc_chain_oracle as orc
    from paper_2008_11421_b200.executor import ExecConfig, Executor
    from paper_2008_11421_b200.plan import PlanBundle
    from paper_2008_11421_b200.units import FCUnit, mse_zero_loss
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cases = json.loads((root / "tests" / "golden" / "sched_cases.json").read_text())["cases"]
        c = next(x for x in cases if x["name"] == "cfg0_fc_chain")
        ex = Executor([FCUnit(64, 64) for _ in range(6)], PlanBundle(c["model"], c["hardware"], c["plan"]),
                      batch=2, loss_fn=mse_zero_loss,
                      cfg=ExecConfig(world_size=world, rank=rank, ipc_exchange=True, optimizer=optimizer,
                                     lr=lr, dist_groups=3))
        w0 = orc.init_weights()
        ex.load_weights({i + 1: [torch.from_numpy(w)] for i, w in enumerate(w0)})
        handles = [None] * world
        dist.all_gather_object(handles, ex.ipc_handles())
        ex.ipc_connect(handles)
        losses = [float(ex.step(torch.from_numpy(orc.inputs(rank, it)).cuda())) for it in range(1, 4)]
        w = ex.unit_weights()
        st = ex.stats()
        dist.barrier()
        q.put((rank, losses, [w[i + 1][0].cpu().numpy() for i in range(6)], st["bytes_net_total"]))
        ex.close()
    except BaseException as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("optimizer,lr", [("sgd", 1e-2), ("adam", 1e-3)])
def test_two_process_ipc_dp_matches_oracle(optimizer, lr):
    from oracle import fc_chain_oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, optimizer, lr, q)) for r in range(2)]
    [p.start() for p in ps]
    res = {}
    try:
        for _ in range(2):
            r, losses, ws, net = q.get(timeout=180)
            assert ws is not None, losses
            res[r] = (losses, ws, net)
    finally:
        [p.join(timeout=60) for p in ps]
        for p in ps:
            if p.is_alive():
                p.kill()
    ref_losses, ref_w = orc.train(workers=2, iterations=3, optimizer=optimizer, lr=lr)
    for r in (0, 1):
        np.testing.assert_allclose(res[r][0], [l[r] for l in ref_losses], rtol=1e-5)
        assert res[r][2] > 0
    atol = 1e-6 if optimizer == "sgd" else 1e-5
    for a, b, ref in zip(res[0][1], res[1][1], ref_w):
        assert np.array_equal(a, b)
        np.testing.assert_allclose(a, ref, rtol=1e-5, atol=atol)
