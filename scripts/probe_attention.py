"""Attention backends on B200 at the GPT shapes (causal, bf16): aten flash
(FA2 code) vs cuDNN SDPA (sm100 kernels): time fwd/bwd and check that two
runs are bitwise identical (the executor's recompute-forward and the
out-of-core == in-core tests need determinism)."""
import sys
import torch

aten = torch.ops.aten


def run(kind, q, k, v, do):
    if kind == "flash":
        o, lse = aten._scaled_dot_product_flash_attention(q, k, v, 0.0, True, False)[:2]
        z = torch.zeros((), dtype=torch.int64, device=q.device)
        s = q.shape[2]
        g = aten._scaled_dot_product_flash_attention_backward(do, q, k, v, o, lse, None, None, s, s, 0.0, True, z, z)
        return o, g
    r = aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
    o, lse, _, _, _, _, seed, off, _ = r
    s = q.shape[2]
    g = aten._scaled_dot_product_cudnn_attention_backward(do, q, k, v, o, lse, seed, off, None, None, None, s, s,
                                                          0.0, True)
    return o, g


def main():
    for (n, h, s, d) in [(144, 20, 1024, 96), (128, 32, 1024, 96), (16, 32, 1024, 128)]:
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v, do = (torch.randn(n, s, h, d, device="cuda", generator=g, dtype=torch.bfloat16).transpose(1, 2)
                       for _ in range(4))
        flops_f = 2.0 * n * h * s * s * d  # causal: half of 4 s^2 d
        for kind in ("flash", "cudnn"):
            try:
                o1, g1 = run(kind, q, k, v, do)
                o2, g2 = run(kind, q, k, v, do)
                det = torch.equal(o1, o2) and all(torch.equal(a, b) for a, b in zip(g1, g2))
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                torch.cuda.synchronize()
                e0.record()
                for _ in range(5):
                    o, lse = (run(kind, q, k, v, do)[0], None)
                e1.record()
                torch.cuda.synchronize()
                ms_total = e0.elapsed_time(e1) / 5
                # fwd alone
                e0.record()
                for _ in range(5):
                    if kind == "flash":
                        aten._scaled_dot_product_flash_attention(q, k, v, 0.0, True, False)
                    else:
                        aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
                e2.record()
                torch.cuda.synchronize()
                ms_f = e0.elapsed_time(e2) / 5
                ms_b = ms_total - ms_f
                ref = run("flash", q, k, v, do)[0]
                err = ((o1.float() - ref.float()).norm() / ref.float().norm()).item()
                print(f"{kind:6s} n{n} h{h} s{s} d{d}: fwd {ms_f:.2f} ms ({flops_f / ms_f / 1e9:.0f} TF), "
                      f"bwd {ms_b:.2f} ms ({2.5 * flops_f / ms_b / 1e9:.0f} TF), deterministic {det}, "
                      f"rel diff vs flash {err:.2e}", flush=True)
            except Exception as ex:
                print(kind, "failed:", repr(ex)[:300], flush=True)


if __name__ == "__main__":
    main()
