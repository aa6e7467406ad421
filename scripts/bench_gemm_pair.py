"""Own tcgen05 convolutions vs cuDNN at the ResNet-200 bottleneck shapes
(batch from argv, default 1024: every operand beyond L2), for the CTA-pair
A/B comparison: run once with KRT_GEMM_PAIR=0 and once with it unset.
CUDA events, median of 10; one JSON line per (stage, conv).

    KRT_GEMM_PAIR=0 python scripts/bench_gemm_pair.py 1024
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

aten = torch.ops.aten
torch.backends.cudnn.benchmark = True


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return round(ts[len(ts) // 2], 4)


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pair = os.environ.get("KRT_GEMM_PAIR", "1")
for (w, side) in [(64, 56), (128, 28), (256, 14), (512, 7)]:
    dev = "cuda"
    for name, cin, cout, k in (("conv1", 4 * w, w, 1), ("conv2", w, w, 3), ("conv3", w, 4 * w, 1)):
        x = cl(torch.randn(n, cin, side, side, device=dev).to(torch.bfloat16))
        g = torch.ones(cin, device=dev, dtype=torch.bfloat16)
        b = torch.zeros(cin, device=dev, dtype=torch.bfloat16)
        m, i = torch.empty(cin, device=dev), torch.empty(cin, device=dev)
        bnfused.stats(x, m, i)
        sm, si = torch.empty(cout, device=dev), torch.empty(cout, device=dev)
        fl = 2.0 * n * side * side * k * k * cin * cout
        r = {"pair": pair, "w": w, "side": side, "conv": name, "cin": cin, "cout": cout, "batch": n}
        if k == 1:
            wt = (torch.randn(cout, cin, device=dev) * cin ** -0.5).to(torch.bfloat16)
            wn = wt.view(cout, cin, 1, 1)
            if bnfused.conv1x1_supported(cin, cout):
                r["own_plain"] = timeit(lambda: bnfused.conv1x1(x, wn))
                r["own_stats"] = timeit(lambda: bnfused.conv1x1(x, wn, stats=(sm, si)))
            if bnfused.conv1x1_supported(cin, cout, pre=True):
                r["own_pre_stats"] = timeit(lambda: bnfused.conv1x1(x, wn, pre=(m, i, g, b), stats=(sm, si)))
            r["cudnn"] = timeit(lambda: aten.convolution(x, wn, None, [1, 1], [0, 0], [1, 1], False, [0, 0], 1))
        else:
            wt = (torch.randn(cout, 3, 3, cin, device=dev) * (9 * cin) ** -0.5).to(torch.bfloat16)
            wn = wt.permute(0, 3, 1, 2)
            r["own_plain"] = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1))
            r["own_stats"] = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1, stats=(sm, si)))
            r["own_pre_stats"] = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1, pre=(m, i, g, b), stats=(sm, si)))
            r["cudnn"] = timeit(lambda: aten.convolution(x, wn, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1))
        r["bn_apply"] = timeit(lambda: bnfused.apply(x, m, i, g, b, relu=True))
        r["TFLOPs"] = {kk: round(fl / v / 1e9) for kk, v in r.items() if kk.startswith(("own", "cudnn"))}
        print(json.dumps(r), flush=True)
