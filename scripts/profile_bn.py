"""Runs the fused BN kernels once each at ResNet-200 stage-1 size
(batch 512, 56x56, C=256 -> 411M elements, 822 MB bf16) for ncu capture."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused

n, c, h, w = 512, 256, 56, 56
x = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
r = torch.randn_like(x, memory_format=torch.channels_last)
dy = torch.randn_like(x, memory_format=torch.channels_last)
g = torch.ones(c, device="cuda", dtype=torch.bfloat16)
b = torch.zeros(c, device="cuda", dtype=torch.bfloat16)
m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
dg, db = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
for _ in range(2):
    bnfused.stats(x, m, i)
    y = bnfused.apply(x, m, i, g, b, relu=True, res=r)
    dz = bnfused.add_relu_bwd(dy, x, m, i, g, b, r)
    dx = bnfused.backward(dz, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db)
torch.cuda.synchronize()
# CUDA-event timing of each kernel (the bench.py roofline uses the same numbers)
def t(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3
nb = x.numel() * 2
for name, fn, traffic in [("stats", lambda: bnfused.stats(x, m, i), nb),
                          ("apply+res+relu", lambda: bnfused.apply(x, m, i, g, b, relu=True, res=r), 3 * nb),
                          ("add_relu_bwd", lambda: bnfused.add_relu_bwd(dy, x, m, i, g, b, r), 4 * nb),
                          ("bwd(reduce+elemt)", lambda: bnfused.backward(dz, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db), 5 * nb)]:
    sec = t(fn)
    print(f"{name:20s} {sec*1e3:8.3f} ms  {traffic/sec/1e9:8.1f} GB/s algorithmic")
