"""ncu target: one launch each of the own im2col 3x3 fprop (with / without
the BN prologue and statistics), the wgrad GEMM, and cuDNN's 3x3 fprop on the
same ResNet-200 stage-2 shape (batch given on the command line)."""
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
w, side = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (128, 28)
x = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
dy = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
wt = (torch.randn(w, 3, 3, w, device="cuda") * (9 * w) ** -0.5).to(torch.bfloat16)
g = torch.ones(w, device="cuda", dtype=torch.bfloat16)
b = torch.zeros(w, device="cuda", dtype=torch.bfloat16)
m, i = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
bnfused.stats(x, m, i)
sm, si = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
dw = torch.empty(w, 3, 3, w, device="cuda")
wn = wt.permute(0, 3, 1, 2)
for _ in range(2):
    bnfused.conv_im2col(x, wt, 1, 1, pre=(m, i, g, b), stats=(sm, si))
    bnfused.conv_im2col(x, wt, 1, 1)
    bnfused.conv_wgrad(dy, x, dw, 3, 1, 1, pre=(m, i, g, b))
    aten.convolution(x, wn, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1)
torch.cuda.synchronize()
