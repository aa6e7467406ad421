"""Runs the tcgen05 1x1-conv GEMM at ResNet-200 stage-2 / stage-1 shapes
(batch 512) for an ncu capture:

    ncu --set full -k regex:conv1x1_kernel -o prof python scripts/profile_conv1x1.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused  # noqa: E402


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


for w, hw in ((128, 28), (64, 56)):
    x = cl(torch.randn(512, 4 * w, hw, hw, device="cuda", dtype=torch.bfloat16))
    c2 = cl(torch.randn(512, w, hw, hw, device="cuda", dtype=torch.bfloat16))
    w1 = cl(torch.randn(w, 4 * w, 1, 1, device="cuda", dtype=torch.bfloat16) * 0.05)
    w3 = cl(torch.randn(4 * w, w, 1, 1, device="cuda", dtype=torch.bfloat16) * 0.05)
    m, i = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
    m3, i3 = torch.empty(4 * w, device="cuda"), torch.empty(4 * w, device="cuda")
    g = torch.ones(w, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(w, device="cuda", dtype=torch.bfloat16)
    bnfused.stats(c2, m, i)
    for _ in range(2):
        bnfused.conv1x1(x, w1, stats=(m, i))                    # conv1 + BN1 statistics
        bnfused.conv1x1(c2, w3, pre=(m, i, g, b), stats=(m3, i3))  # relu(bn2) prologue + BN3 statistics
torch.cuda.synchronize()
