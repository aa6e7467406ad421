"""cuDNN 1x1 weight gradients at the ResNet-1001 2048x2048 widths (batch 2):
conv1 (4w -> w) and conv3 (w -> 4w) per stage, against the HBM floor (x and
dy read once) and the bn_apply that rebuilds their input."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

aten = torch.ops.aten
torch.backends.cudnn.benchmark = True
hbm = 6548.8e9


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
    return ts[len(ts) // 2]


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


for w, side in ((16, 2048), (32, 1024), (64, 512)):
    for name, cin, cout in (("conv1", 4 * w, w), ("conv3", w, 4 * w)):
        x = cl(torch.randn(2, cin, side, side, device="cuda").to(torch.bfloat16))
        dy = cl(torch.randn(2, cout, side, side, device="cuda").to(torch.bfloat16))
        wt = cl((torch.randn(cout, cin, 1, 1, device="cuda") * 0.1).to(torch.bfloat16))
        r = {"w": w, "side": side, "conv": name, "cin": cin, "cout": cout,
             "floor_ms": (x.numel() + dy.numel()) * 2 / hbm * 1e3}
        r["cudnn_wgrad_ms"] = timeit(lambda: aten.convolution_backward(dy, x, wt, None, [1, 1], [0, 0], [1, 1], False,
                                                                       [0, 0], 1, [False, True, False]))
        m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
        bnfused.stats(x, m, i)
        g = torch.ones(cin, device="cuda", dtype=torch.bfloat16)
        b = torch.zeros(cin, device="cuda", dtype=torch.bfloat16)
        r["bn_apply_ms"] = timeit(lambda: bnfused.apply(x, m, i, g, b, relu=True))
        dwo = torch.empty(cout, 1, 1, cin, device="cuda")
        r["own_wgrad_ms"] = timeit(lambda: bnfused.wgrad1x1_narrow(dy, x, dwo))
        r["own_wgrad_pre_ms"] = timeit(lambda: bnfused.wgrad1x1_narrow(dy, x, dwo, pre=(m, i, g, b)))
        print(json.dumps(r), flush=True)
