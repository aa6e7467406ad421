"""Data parallelism across GPUs through the runtime's own NCCL communicator
(the default exchange of bench.py): one process per GPU, rank 0's
ncclUniqueId broadcast over gloo, per-group ncclReduceScatter of the fp32
gradients -> D2H of this rank's shard -> host SGD/Adam on the shard -> H2D ->
ncclAllGather (distsim.py:205-236 with the reduce moved in front of the
shard-sized grad_out).  cfg0 (BASELINE configs[0]) with 2 workers
vs the CPU oracle (oracle/fc_chain_oracle.py) at the DP tolerances of
DESIGN 6; and bench.py --gpus 2 self-launching 2 ranks.  Both need >= 2 GPUs
and skip with the reason otherwise (gpurun boxes have one)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs (NCCL cannot put two ranks on one device)")]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, optimizer, lr, q):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle import fc_chain_oracle as orc
    from paper_2008_11421_b200 import _lib
    from paper_2008_11421_b200.executor import ExecConfig, Executor
    from paper_2008_11421_b200.plan import PlanBundle
    from paper_2008_11421_b200.units import FCUnit, mse_zero_loss
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank)
        box = [_lib.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        cases = json.loads((ROOT / "tests" / "golden" / "sched_cases.json").read_text())["cases"]
        c = next(x for x in cases if x["name"] == "cfg0_fc_chain")
        ex = Executor([FCUnit(64, 64) for _ in range(6)], PlanBundle(c["model"], c["hardware"], c["plan"]),
                      batch=2, loss_fn=mse_zero_loss,
                      cfg=ExecConfig(device=rank, world_size=world, rank=rank, nccl_id=box[0],
                                     optimizer=optimizer, lr=lr, dist_groups=3))
        w0 = orc.init_weights()
        ex.load_weights({i + 1: [torch.from_numpy(w)] for i, w in enumerate(w0)})
        losses = [float(ex.step(torch.from_numpy(orc.inputs(rank, it)).cuda(rank))) for it in range(1, 4)]
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
def test_two_gpu_nccl_dp_matches_oracle(optimizer, lr):
    from oracle import fc_chain_oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, optimizer, lr, q)) for r in range(2)]
    [p.start() for p in ps]
    res = {}
    try:
        for _ in range(2):
            r, losses, ws, net = q.get(timeout=300)
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
        assert np.array_equal(a, b)        # replicas identical after the all-gather
        np.testing.assert_allclose(a, ref, rtol=1e-5, atol=atol)


def test_bench_self_launches_two_ranks():
    """`bench.py --gpus 2` without torchrun spawns 2 NCCL ranks and reports the
    whole-job value with n_gpus 2 and a measured NVLink term."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                          "--plan", "resnet_small_bf16", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["exchange"] == "nccl"
    nv = line["iteration_roofline"]["nvlink"]
    assert nv["reduce_scatter_s"] > 0 and "krt_probe_exchange" in nv["source"]
