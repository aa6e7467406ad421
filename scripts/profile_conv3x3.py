"""ncu target: the own 3x3 im2col fprop (plain) and cuDNN's 3x3 fprop on one
ResNet-200 stage shape, two launches each (the second is the warm one).

    python scripts/profile_conv3x3.py [batch] [w] [side]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

aten = torch.ops.aten
torch.backends.cudnn.benchmark = True


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w, side = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (64, 56)
x = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
wt = (torch.randn(w, 3, 3, w, device="cuda") * (9 * w) ** -0.5).to(torch.bfloat16)
wn = wt.permute(0, 3, 1, 2)
for _ in range(3):  # cuDNN benchmark mode settles its algorithm on the first call
    aten.convolution(x, wn, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1)
for _ in range(2):
    bnfused.conv_im2col(x, wt, 1, 1)
torch.cuda.synchronize()
