"""Determinism and speed of the attention backends (forward alone, backward)
with torch.use_deterministic_algorithms(True, warn_only=False) (the setting
under which flash / cuDNN pick their deterministic backward)."""
import torch

from probe_attention import run

aten = torch.ops.aten
for (n, h, s, d) in [(16, 32, 1024, 96), (144, 20, 1024, 96)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(n, s, h, d, device="cuda", generator=g, dtype=torch.bfloat16).transpose(1, 2)
                   for _ in range(4))
    flops_f = 2.0 * n * h * s * s * d
    for det_mode in (False, True):
        torch.use_deterministic_algorithms(det_mode, warn_only=False)
        for kind in ("flash", "cudnn"):
            try:
                o = [run(kind, q, k, v, do) for _ in range(4)]
                fdet = all(torch.equal(o[0][0], x[0]) for x in o)
                bdet = all(all(torch.equal(a, b) for a, b in zip(o[0][1], x[1])) for x in o)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(5):
                    run(kind, q, k, v, do)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 5
                print(f"n{n} h{h} det_algos={det_mode} {kind}: fwd repeatable {fdet}, bwd {bdet}, fwd+bwd {ms:.2f} ms "
                      f"({3.5 * flops_f / ms / 1e9:.0f} TF)", flush=True)
            except Exception as ex:
                print(f"n{n} det_algos={det_mode} {kind}: failed {repr(ex)[:200]}", flush=True)
