"""ncu target: the stem weight-gradient kernel at batch 256 (224x224)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
x = torch.randn(n, 3, 224, 224, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
dc = torch.randn(n, 64, 112, 112, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
dw = torch.empty(64, 7, 7, 3, device="cuda")
for _ in range(2):
    bnfused.stem_wgrad(dc, x, dw)
torch.cuda.synchronize()
