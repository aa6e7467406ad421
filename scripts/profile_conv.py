"""cuDNN convolutions of the ResNet-200 bottleneck at batch 512 (stage 1-3
shapes), fprop / dgrad / wgrad, after cudnn.benchmark's algorithm search,
inside cudaProfilerStart/Stop for an ncu capture of the steady-state kernels:

    ncu --profile-from-start off --set full -o prof python scripts/profile_conv.py
"""
import sys

import torch

sys.path.insert(0, ".")
torch.backends.cudnn.benchmark = True
aten = torch.ops.aten


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


cases = []
for w, hw in ((64, 56), (128, 28), (256, 14)):
    for cin, cout, k in ((4 * w, w, 1), (w, w, 3), (w, 4 * w, 1)):
        x = cl(torch.randn(512, cin, hw, hw, device="cuda", dtype=torch.bfloat16))
        wt = cl(torch.randn(cout, cin, k, k, device="cuda", dtype=torch.bfloat16) * 0.05)
        y = aten.convolution(x, wt, None, [1, 1], [k // 2, k // 2], [1, 1], False, [0, 0], 1)
        cases.append((x, wt, cl(torch.randn_like(y)), k // 2))


def run_all():
    for x, wt, dy, pad in cases:
        aten.convolution(x, wt, None, [1, 1], [pad, pad], [1, 1], False, [0, 0], 1)
        aten.convolution_backward(dy, x, wt, None, [1, 1], [pad, pad], [1, 1], False, [0, 0], 1, [True, True, False])


for _ in range(3):
    run_all()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run_all()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
