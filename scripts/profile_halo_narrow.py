"""ncu target: the halo 3x3 kernel at the ResNet-1001 stage-1 shape (16
channels, 2048x2048, batch 2), plain, two launches."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

w, side = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (16, 2048)
x = torch.randn(2, w, side, side, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
wt = (torch.randn(w, 3, 3, w, device="cuda") * 0.1).to(torch.bfloat16)
for _ in range(2):
    bnfused.conv_im2col(x, wt, 1, 1)
torch.cuda.synchronize()
