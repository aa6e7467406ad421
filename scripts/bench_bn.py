"""CUDA-event timing of the fused BN kernels at the ResNet-200 layer shapes
(batch 512 slices of the b3072 bench workload), algorithmic bytes / time.

    python scripts/bench_bn.py [--batch 512] [--json out.json]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--json", default=None)
ap.add_argument("--preact", action="store_true", help="ResNet-1001 @ 2048^2 widths (batch 2 unless --batch)")
args = ap.parse_args()

# (C, H): bottleneck widths and outputs of the four ResNet-200 stages
SHAPES = [(64, 56), (256, 56), (128, 28), (512, 28), (256, 14), (1024, 14), (512, 7), (2048, 7)]
if args.preact:   # pre-activation ResNet-1001 at 2048^2: unit input 4w and width w per stage
    SHAPES = [(64, 2048), (16, 2048), (128, 1024), (32, 1024), (256, 512), (64, 512)]
if args.batch is None:
    args.batch = 2 if args.preact else 512


def t(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


rows_out = []
for c, hw in SHAPES:
    n = args.batch
    mk = lambda: torch.randn(n, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    x, r, dy = mk(), mk(), mk()
    g = torch.ones(c, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(c, device="cuda", dtype=torch.bfloat16)
    m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    dg, db = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    bnfused.stats(x, m, i)
    nb = x.numel() * 2
    cases = [("stats", lambda: bnfused.stats(x, m, i), nb),
             ("stats_apply", lambda: bnfused.stats_apply(x, m, i, g, b, relu=True), 3 * nb),
             ("stats_apply_res", lambda: bnfused.stats_apply(x, m, i, g, b, relu=True, res=r), 4 * nb),
             ("apply", lambda: bnfused.apply(x, m, i, g, b, relu=True), 2 * nb),
             ("apply_res", lambda: bnfused.apply(x, m, i, g, b, relu=True, res=r), 3 * nb),
             ("add_relu_bwd", lambda: bnfused.add_relu_bwd(dy, x, m, i, g, b, r), 4 * nb),
             ("backward_relu", lambda: bnfused.backward(dy, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db), 5 * nb),
             ("add_relu_backward", lambda: bnfused.add_relu_backward(dy, x, m, i, g, b, r, dgamma=dg, dbeta=db),
              7 * nb)]
    for name, fn, traffic in cases:
        sec = t(fn)
        rows_out.append({"C": c, "HW": hw, "batch": n, "kernel": name, "us": sec * 1e6,
                         "GBps": traffic / sec / 1e9})
        print(f"C={c:5d} {hw:3d}x{hw:<3d} {name:18s} {sec*1e6:9.1f} us {traffic/sec/1e9:8.1f} GB/s")
    del x, r, dy
    torch.cuda.empty_cache()
# ResNet stem: relu(bn(c)) -> maxpool 3x3/s2 fused vs apply + aten max-pool (fwd and bwd)
n, c, hw = args.batch, 64, 112
x = torch.randn(n, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
g = torch.ones(c, device="cuda", dtype=torch.bfloat16)
b = torch.zeros(c, device="cuda", dtype=torch.bfloat16)
m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
bnfused.stats(x, m, i)
y = bnfused.relu_maxpool(x, m, i, g, b)
dy = torch.randn_like(y).contiguous(memory_format=torch.channels_last)


def aten_fw():
    a = bnfused.apply(x, m, i, g, b, relu=True)
    return torch.ops.aten.max_pool2d_with_indices(a, [3, 3], [2, 2], [1, 1])


def aten_bw():
    a = bnfused.apply(x, m, i, g, b, relu=True)
    _, idx = torch.ops.aten.max_pool2d_with_indices(a, [3, 3], [2, 2], [1, 1])
    return torch.ops.aten.max_pool2d_with_indices_backward(dy, a, [3, 3], [2, 2], [1, 1], [1, 1], False, idx)


nb_in, nb_out = x.numel() * 2, y.numel() * 2
for name, fn, traffic in [("relu_maxpool", lambda: bnfused.relu_maxpool(x, m, i, g, b), nb_in + nb_out),
                          ("apply+aten_maxpool", aten_fw, nb_in + nb_out),
                          ("relu_maxpool_bwd", lambda: bnfused.relu_maxpool_backward(dy, x, m, i, g, b),
                           2 * nb_in + nb_out),
                          ("apply+aten_maxpool_bwd", aten_bw, 2 * nb_in + nb_out)]:
    sec = t(fn)
    rows_out.append({"C": c, "HW": hw, "batch": n, "kernel": name, "us": sec * 1e6, "GBps": traffic / sec / 1e9})
    print(f"C={c:5d} {hw:3d}x{hw:<3d} {name:22s} {sec*1e6:9.1f} us {traffic/sec/1e9:8.1f} GB/s (vs fused-min bytes)")
if args.json:
    json.dump(rows_out, open(args.json, "w"), indent=1)
