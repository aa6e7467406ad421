"""lm_xent (fused LM cross-entropy, csrc/ln_kernels.cu) vs the chunked fp32
torch loss at the GPT shapes: time and HBM fraction (4 B per logit)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2008_11421_b200 import lnfused  # noqa: E402


def chunked(z, y, chunk_rows=8192):
    n = z.shape[0]
    dl = torch.empty_like(z)
    for r0 in range(0, n, chunk_rows):
        lf = z[r0:r0 + chunk_rows].float()
        tc = y[r0:r0 + chunk_rows]
        lse = torch.logsumexp(lf, dim=1)
        p = torch.exp(lf - lse.view(-1, 1))
        p[torch.arange(p.shape[0], device=p.device), tc] -= 1.0
        dl[r0:r0 + chunk_rows] = (p / n).to(z.dtype)
    return dl


for T, V in [(147456, 51200), (131072, 51200)]:
    z = torch.randn(T, V, device="cuda").mul_(3).to(torch.bfloat16)
    y = torch.randint(0, V, (T,), device="cuda")
    for name, fn in (("own lm_xent", lambda: lnfused.lm_xent(z, y, 1.0 / T)), ("torch chunked fp32", lambda: chunked(z, y))):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"T{T} V{V} {name}: {ms:.2f} ms, {T * V * 4 / ms / 1e6:.0f} GB/s (4 B/logit)", flush=True)
    del z
