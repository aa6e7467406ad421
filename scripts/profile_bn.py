"""Runs each fused BN kernel twice at ResNet-200 stage-1 size (batch 512,
56x56, C=256 -> 411M elements, 822 MB bf16 per tensor) for an ncu capture:

    ncu --set full --clock-control none --import-source on -k regex:"stats_kernel|apply_kernel|bwd_kernel|add_relu" -o prof \
        python scripts/profile_bn.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused  # noqa: E402

n, c, h, w = 512, int(sys.argv[1]) if len(sys.argv) > 1 else 256, 56, 56
mk = lambda: torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
x, r, dy = mk(), mk(), mk()
g = torch.ones(c, device="cuda", dtype=torch.bfloat16)
b = torch.zeros(c, device="cuda", dtype=torch.bfloat16)
m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
dg, db = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
for _ in range(2):
    bnfused.stats(x, m, i)
    y = bnfused.stats_apply(x, m, i, g, b, relu=True)
    y = bnfused.apply(x, m, i, g, b, relu=True)
    dz = bnfused.add_relu_bwd(dy, x, m, i, g, b, r)
    dx = bnfused.backward(dz, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db)
    dz, dx = bnfused.add_relu_backward(dy, x, m, i, g, b, r, dgamma=dg, dbeta=db)
torch.cuda.synchronize()
