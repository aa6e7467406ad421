"""ncu target: the own 3x3 conv (halo path for 64/128 output channels) on one
ResNet-200 stage shape, plain and with the BN prologue + statistics.

    python scripts/profile_halo.py [batch] [w] [side]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w, side = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (64, 56)
x = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
wt = (torch.randn(w, 3, 3, w, device="cuda") * (9 * w) ** -0.5).to(torch.bfloat16)
g = torch.ones(w, device="cuda", dtype=torch.bfloat16)
b = torch.zeros(w, device="cuda", dtype=torch.bfloat16)
m, i = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
bnfused.stats(x, m, i)
sm, si = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
for _ in range(2):
    bnfused.conv_im2col(x, wt, 1, 1)
    bnfused.conv_im2col(x, wt, 1, 1, pre=(m, i, g, b), stats=(sm, si))
torch.cuda.synchronize()
