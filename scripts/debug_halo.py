"""Debug: own halo 3x3 conv vs torch, per single tap (weights zero elsewhere)."""
import os
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

torch.manual_seed(0)
n, cin, cout, h = 2, 64, 64, 8
x = torch.randn(n, cin, h, h, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
print("baseoff", os.environ.get("KRT_HALO_BASEOFF"))
for tap in list(range(9)) + [None]:
    w = (torch.randn(cout, 3, 3, cin, device="cuda") * 0.1)
    if tap is not None:
        m = torch.zeros(3, 3, device="cuda")
        m[tap // 3, tap % 3] = 1
        w = w * m.view(1, 3, 3, 1)
    w = w.to(torch.bfloat16).contiguous()
    y = bnfused.conv_im2col(x, w, 1, 1)
    ref = F.conv2d(x.float(), w.permute(0, 3, 1, 2).float(), padding=1)
    err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
    bad = ((y.float() - ref).abs() > 0.05 * ref.abs().max()).nonzero()
    print("tap", tap, "err", round(err, 4), "bad", bad.shape[0], bad[:4].tolist() if bad.shape[0] else "")
