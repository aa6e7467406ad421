"""tcgen05 1x1 dgrad + BN-backward-reduce GEMM at ResNet-200 stage-2 shape
(batch 512, 28x28, 512 -> 128 channels) for an ncu capture."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused  # noqa: E402


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


n, w, hw = 512, 128, 28
x = cl(torch.randn(n, w, hw, hw, device="cuda", dtype=torch.bfloat16))
dy = cl(torch.randn(n, 4 * w, hw, hw, device="cuda", dtype=torch.bfloat16))
wt = cl(torch.randn(4 * w, w, 1, 1, device="cuda", dtype=torch.bfloat16) * 0.05)
g = torch.ones(w, device="cuda", dtype=torch.bfloat16)
b = torch.zeros(w, device="cuda", dtype=torch.bfloat16)
m, i = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
bnfused.stats(x, m, i)
for _ in range(3):
    bnfused.conv1x1_dgrad_bn_backward(dy, wt, x, m, i, g, b)
    bnfused.conv1x1(dy, wt.reshape(4 * w, w).t().contiguous().reshape(w, 4 * w, 1, 1))  # same GEMM, store only
torch.cuda.synchronize()
