"""ResNet-1001 (cfg2, 2048x2048, batch 2) pre-activation bottleneck 1x1
convolutions on the tcgen05 GEMM: conv1 = relu(bn0(x)) . W1 + BN1 stats,
conv3 = relu(bn2(c2)) . W3 + shortcut; GB/s of algorithmic bytes (A read,
residual read, C written) from CUDA events, vs the measured HBM copy peak.

    python scripts/bench_preact_gemm.py [--batch 2] [--res 2048] [--json out.json]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--res", type=int, default=2048)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--json", default=None)
ap.add_argument("--only", default=None, help="stage:conv, e.g. 1:conv3 (profiling)")
args = ap.parse_args()


def t(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def cl(x):
    return x.contiguous(memory_format=torch.channels_last)


out = []
for si, (w, side) in enumerate(((16, args.res), (32, args.res // 2), (64, args.res // 4))):
    n = args.batch
    for name, cin, cout, resid in (("conv1", 4 * w, w, False), ("conv3", w, 4 * w, True)):
        if args.only and args.only != f"{si + 1}:{name}":
            continue
        x = cl(torch.randn(n, cin, side, side, device="cuda", dtype=torch.bfloat16))
        wt = cl(torch.randn(cout, cin, 1, 1, device="cuda", dtype=torch.bfloat16) * cin ** -0.5)
        g = torch.ones(cin, device="cuda", dtype=torch.bfloat16)
        b = torch.zeros(cin, device="cuda", dtype=torch.bfloat16)
        m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
        bnfused.stats(x, m, i)
        y = cl(torch.empty(n, cout, side, side, device="cuda", dtype=torch.bfloat16))
        r = cl(torch.randn(n, cout, side, side, device="cuda", dtype=torch.bfloat16)) if resid else None
        so = (torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda"))
        M = n * side * side
        nbytes = M * (cin + cout * (2 if resid else 1)) * 2
        fn = (lambda: bnfused.conv1x1(x, wt, out=y, pre=(m, i, g, b), res=r)) if resid else \
             (lambda: bnfused.conv1x1(x, wt, out=y, pre=(m, i, g, b), stats=so))
        sec = t(fn, args.reps)
        apply_sec = t(lambda: bnfused.apply(x, m, i, g, b, relu=True), args.reps)
        res = {"stage": si + 1, "conv": name, "M": M, "K": cin, "N": cout, "us": sec * 1e6,
               "GBps": nbytes / sec / 1e9, "bn_apply_same_input_GBps": 2 * M * cin * 2 / apply_sec / 1e9}
        print(json.dumps(res), flush=True)
        out.append(res)
        del x, y, r
        torch.cuda.empty_cache()
if args.json:
    json.dump(out, open(args.json, "w"), indent=1)
