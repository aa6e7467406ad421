"""ResNet stem convolution (7x7/2, 3 -> 64, 224^2) forward and weight
gradient under different input layouts (cuDNN picks a legacy sm80 kernel for
3-channel NHWC), CUDA-event timing, TFLOP/s.

    python scripts/bench_stem.py [--batch 512]
"""
import argparse
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
torch.backends.cudnn.benchmark = True
ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=512)
args = ap.parse_args()
aten = torch.ops.aten
n = args.batch


def t(fn, reps=5):
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


flops = 2.0 * n * 112 * 112 * 64 * 3 * 49
x0 = torch.randn(n, 3, 224, 224, device="cuda", dtype=torch.bfloat16)
w0 = torch.randn(64, 3, 7, 7, device="cuda", dtype=torch.bfloat16) * 0.1
for name, cpad, fmt in (("nhwc_c3", 3, torch.channels_last), ("nchw_c3", 3, torch.contiguous_format),
                        ("nhwc_c4", 4, torch.channels_last), ("nhwc_c8", 8, torch.channels_last)):
    x = torch.zeros(n, cpad, 224, 224, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=fmt)
    x[:, :3] = x0
    w = torch.zeros(64, cpad, 7, 7, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=fmt)
    w[:, :3] = w0
    y = aten.convolution(x, w, None, [2, 2], [3, 3], [1, 1], False, [0, 0], 1)
    dy = torch.randn_like(y)
    f = t(lambda: aten.convolution(x, w, None, [2, 2], [3, 3], [1, 1], False, [0, 0], 1))
    g = t(lambda: aten.convolution_backward(dy, x, w, None, [2, 2], [3, 3], [1, 1], False, [0, 0], 1,
                                            [False, True, False]))
    print(f"{name}: fprop {f * 1e3:.2f} ms ({flops / f / 1e12:.0f} TFLOP/s)  wgrad {g * 1e3:.2f} ms "
          f"({flops / g / 1e12:.0f} TFLOP/s)", flush=True)
    del x, w, y, dy
    torch.cuda.empty_cache()

# the tcgen05 implicit GEMM (csrc/gemm_sm100.cu GATHER mode) with the BN statistics
from paper_2008_11421_b200 import bnfused  # noqa: E402
x = x0.contiguous(memory_format=torch.channels_last)
w = w0.contiguous(memory_format=torch.channels_last)
y = torch.empty(n, 64, 112, 112, device="cuda", dtype=torch.bfloat16, memory_format=torch.channels_last)
m, i = torch.empty(64, device="cuda"), torch.empty(64, device="cuda")
f = t(lambda: bnfused.conv_gather(x, w, 2, 3, out=y))
fs = t(lambda: bnfused.conv_gather(x, w, 2, 3, out=y, stats=(m, i)))
nbytes = x.numel() * 2 + y.numel() * 2
print(f"tc_gather: fprop {f * 1e3:.2f} ms ({flops / f / 1e12:.0f} TFLOP/s, {nbytes / f / 1e9:.0f} GB/s)  "
      f"+stats {fs * 1e3:.2f} ms", flush=True)
x4 = torch.zeros(n, 4, 224, 224, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
x4[:, :3] = x0
w4 = torch.zeros(64, 4, 7, 7, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
w4[:, :3] = w0
f4 = t(lambda: bnfused.conv_gather(x4, w4, 2, 3, out=y, stats=(m, i)))
print(f"tc_gather on a 4-channel input (no pad pass): {f4 * 1e3:.2f} ms ({flops / f4 / 1e12:.0f} TFLOP/s)", flush=True)
