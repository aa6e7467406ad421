"""ResNet-200 bottleneck convolutions at batch 512 (a 1/6 slice of the bench
batch): cuDNN (what units.py calls) vs a plain cuBLAS GEMM on the NHWC view
for the 1x1 convolutions, fprop / dgrad / wgrad, TFLOP/s from CUDA events.

    python scripts/bench_conv.py [--batch 512] [--json out.json]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
torch.backends.cudnn.benchmark = True
ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=512)
ap.add_argument("--json", default=None)
args = ap.parse_args()
aten = torch.ops.aten


def t(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def cl(t_):
    return t_.contiguous(memory_format=torch.channels_last)


out = []
n = args.batch
for w, hw in ((64, 56), (128, 28), (256, 14), (512, 7)):
    for name, cin, cout, k in (("conv1_1x1", 4 * w, w, 1), ("conv2_3x3", w, w, 3), ("conv3_1x1", w, 4 * w, 1)):
        x = cl(torch.randn(n, cin, hw, hw, device="cuda", dtype=torch.bfloat16))
        wt = cl(torch.randn(cout, cin, k, k, device="cuda", dtype=torch.bfloat16) * 0.05)
        pad = k // 2
        y = aten.convolution(x, wt, None, [1, 1], [pad, pad], [1, 1], False, [0, 0], 1)
        dy = cl(torch.randn_like(y))
        flops = 2.0 * n * hw * hw * cin * cout * k * k
        res = {"stage_w": w, "hw": hw, "conv": name, "cin": cin, "cout": cout}
        res["cudnn_fprop_us"] = t(lambda: aten.convolution(x, wt, None, [1, 1], [pad, pad], [1, 1], False,
                                                            [0, 0], 1)) * 1e6
        res["cudnn_dgrad_us"] = t(lambda: aten.convolution_backward(dy, x, wt, None, [1, 1], [pad, pad], [1, 1],
                                                                     False, [0, 0], 1, [True, False, False])) * 1e6
        res["cudnn_wgrad_us"] = t(lambda: aten.convolution_backward(dy, x, wt, None, [1, 1], [pad, pad], [1, 1],
                                                                     False, [0, 0], 1, [False, True, False])) * 1e6
        if k == 1:
            from paper_2008_11421_b200 import bnfused
            mo, io = torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda")
            mi, ii = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda")
            gi = torch.ones(cin, device="cuda", dtype=torch.bfloat16)
            bi = torch.zeros(cin, device="cuda", dtype=torch.bfloat16)
            bnfused.stats(x, mi, ii)
            res["tc_gemm_us"] = t(lambda: bnfused.conv1x1(x, wt, out=y)) * 1e6
            res["tc_gemm_stats_us"] = t(lambda: bnfused.conv1x1(x, wt, out=y, stats=(mo, io))) * 1e6
            if cin <= 1024:
                res["tc_gemm_pre_stats_us"] = t(lambda: bnfused.conv1x1(x, wt, out=y, pre=(mi, ii, gi, bi),
                                                                        stats=(mo, io))) * 1e6

            def cudnn_stats():
                aten.convolution(x, wt, None, [1, 1], [0, 0], [1, 1], False, [0, 0], 1)
                bnfused.stats(y, mo, io)

            def cudnn_pre_stats():
                a = bnfused.apply(x, mi, ii, gi, bi, relu=True)
                aten.convolution(a, wt, None, [1, 1], [0, 0], [1, 1], False, [0, 0], 1)
                bnfused.stats(y, mo, io)
            res["cudnn_stats_us"] = t(cudnn_stats) * 1e6
            res["cudnn_pre_stats_us"] = t(cudnn_pre_stats) * 1e6
            xm = x.permute(0, 2, 3, 1).reshape(-1, cin)      # NHWC view, no copy
            dym = dy.permute(0, 2, 3, 1).reshape(-1, cout)
            wm = wt.reshape(cout, cin)
            res["gemm_fprop_us"] = t(lambda: torch.mm(xm, wm.t())) * 1e6
            res["gemm_dgrad_us"] = t(lambda: torch.mm(dym, wm)) * 1e6
            res["gemm_wgrad_us"] = t(lambda: torch.mm(dym.t(), xm)) * 1e6
        for kk in list(res):
            if kk.endswith("_us"):
                res[kk.replace("_us", "_tflops")] = flops / (res[kk] * 1e-6) / 1e12
        out.append(res)
        print(" ".join(f"{k_}={v:.1f}" if isinstance(v, float) else f"{k_}={v}" for k_, v in res.items()
                       if not k_.endswith("_us")), flush=True)
        del x, wt, y, dy
        torch.cuda.empty_cache()
if args.json:
    json.dump(out, open(args.json, "w"), indent=1)
