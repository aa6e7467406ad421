"""ln_bwd (own one-pass LayerNorm backward + residual add) vs aten's
native_layer_norm_backward + add at the GPT shapes: time and HBM fraction."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2008_11421_b200 import lnfused

for T, H in [(147456, 1920), (131072, 3072), (180224, 4256)]:
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    dy = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    a = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    g = (torch.randn(H, device="cuda") * 0.1 + 1).to(torch.bfloat16)
    b = torch.zeros(H, device="cuda", dtype=torch.bfloat16)
    m, s = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
    lnfused.ln_fwd(x, g, b, 1e-5, m, s)
    dg, db = torch.empty(H, device="cuda"), torch.empty(H, device="cuda")

    def own():
        lnfused.ln_bwd(dy, x, g, m, s, dg, db, addend=a)

    def aten():
        dx, dgg, dbb = torch.ops.aten.native_layer_norm_backward(dy, x, [H], m.view(-1, 1), s.view(-1, 1), g, b,
                                                                 [True, True, True])
        return dx + a

    def own_fwd():
        lnfused.ln_fwd(x, g, b, 1e-5, m, s, residual=a, x2_out=dy)

    def own_fwd_plain():
        lnfused.ln_fwd(x, g, b, 1e-5, m, s)

    for name, fn in (("own ln_bwd", own), ("aten ln_bwd + add", aten), ("own ln_fwd + residual", own_fwd),
                     ("own ln_fwd (no residual; 4 B/elem, figure below counts 8)", own_fwd_plain)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        nb = T * H * 2 * 4   # bwd: dy, x, addend read, dx written; fwd: x, r read, x2, h written
        print(f"T{T} H{H} {name}: {ms:.3f} ms, {nb / ms / 1e6:.0f} GB/s (algorithmic 8 B/elem)", flush=True)
