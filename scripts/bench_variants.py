"""Own convolution variants vs cuDNN (conv only) at ResNet-200 stage shapes,
batch from argv (default 1024: beyond L2).  Isolates what the BN prologue,
the statistics epilogue and the im2col path cost.  CUDA events, median of 10."""
import json
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
for (w, side) in [(128, 28), (256, 14), (512, 7)]:
    x = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
    dy = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
    wt = (torch.randn(w, 3, 3, w, device="cuda") * (9 * w) ** -0.5).to(torch.bfloat16)
    wn = wt.permute(0, 3, 1, 2)
    g = torch.ones(w, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(w, device="cuda", dtype=torch.bfloat16)
    m, i = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
    bnfused.stats(x, m, i)
    sm, si = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
    dw = torch.empty(w, 3, 3, w, device="cuda")
    fl = 2.0 * n * side * side * 9 * w * w
    r = {"w": w, "side": side, "batch": n, "GFLOP": fl / 1e9}
    r["fprop_plain"] = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1))
    r["fprop_stats"] = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1, stats=(sm, si)))
    r["fprop_pre"] = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1, pre=(m, i, g, b)))
    r["fprop_pre_stats"] = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1, pre=(m, i, g, b), stats=(sm, si)))
    r["cudnn_fprop"] = timeit(lambda: aten.convolution(x, wn, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1))
    r["bn_apply"] = timeit(lambda: bnfused.apply(x, m, i, g, b, relu=True))
    r["bn_stats"] = timeit(lambda: bnfused.stats(x, sm, si))
    r["wgrad_plain"] = timeit(lambda: bnfused.conv_wgrad(dy, x, dw, 3, 1, 1))
    r["wgrad_pre"] = timeit(lambda: bnfused.conv_wgrad(dy, x, dw, 3, 1, 1, pre=(m, i, g, b)))
    r["cudnn_wgrad"] = timeit(lambda: aten.convolution_backward(dy, x, wn, None, [1, 1], [1, 1], [1, 1], False,
                                                                [0, 0], 1, [False, True, False]))
    r["dgrad_bn"] = timeit(lambda: bnfused.conv_im2col_dgrad_bn_backward(dy, wt, x, m, i, g, b))
    r["cudnn_dgrad"] = timeit(lambda: aten.convolution_backward(dy, x, wn, None, [1, 1], [1, 1], [1, 1], False,
                                                                [0, 0], 1, [True, False, False]))
    r["bn_backward"] = timeit(lambda: bnfused.backward(dy, x, m, i, g, b, relu=True))
    r["TFLOPs"] = {k: round(fl / v / 1e9) for k, v in r.items() if k.startswith(("fprop", "wgrad", "cudnn"))}
    print(json.dumps(r), flush=True)
