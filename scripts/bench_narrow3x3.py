"""cuDNN 3x3 / stride-1 convolutions at the ResNet-1001 2048x2048 widths
(batch 2): fprop, dgrad, wgrad times against the HBM floor of each (operands
read once, result written once; measured HBM copy bandwidth from argv)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

aten = torch.ops.aten
torch.backends.cudnn.benchmark = True
hbm = float(sys.argv[1]) if len(sys.argv) > 1 else 6548.8e9


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for w, side in ((16, 2048), (32, 1024), (64, 512)):
    x = torch.randn(2, w, side, side, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    dy = torch.randn_like(x)
    wt = (torch.randn(w, w, 3, 3, device="cuda") * 0.1).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    nb = x.numel() * 2
    r = {"w": w, "side": side, "floor_ms": 2 * nb / hbm * 1e3}
    r["fprop_ms"] = timeit(lambda: aten.convolution(x, wt, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1))
    r["dgrad_ms"] = timeit(lambda: aten.convolution_backward(dy, x, wt, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1,
                                                             [True, False, False]))
    r["wgrad_ms"] = timeit(lambda: aten.convolution_backward(dy, x, wt, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1,
                                                             [False, True, False]))
    wo = wt.permute(0, 2, 3, 1).contiguous()   # OHWI
    g = torch.ones(w, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(w, device="cuda", dtype=torch.bfloat16)
    m, i = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
    bnfused.stats(x, m, i)
    sm, si = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
    r["halo"] = bnfused.conv3x3_halo_supported(side, side, w, w, True)
    r["own_fprop_ms"] = timeit(lambda: bnfused.conv_im2col(x, wo, 1, 1))
    r["own_fprop_pre_stats_ms"] = timeit(lambda: bnfused.conv_im2col(x, wo, 1, 1, pre=(m, i, g, b), stats=(sm, si)))
    r["own_dgrad_ms"] = timeit(lambda: bnfused.conv3x3_dgrad(dy, wo))
    dwo = torch.empty(w, 3, 3, w, device="cuda")
    r["own_wgrad_ms"] = timeit(lambda: bnfused.wgrad3x3_narrow(dy, x, dwo))
    r["own_wgrad_pre_ms"] = timeit(lambda: bnfused.wgrad3x3_narrow(dy, x, dwo, pre=(m, i, g, b)))
    r["bn_apply_ms"] = timeit(lambda: bnfused.apply(x, m, i, g, b, relu=True))
    r["bn_stats_ms"] = timeit(lambda: bnfused.stats(x, sm, si))
    r["frac_of_floor"] = {k: round(r["floor_ms"] / r[k], 3) for k in r if k.endswith("_ms") and k != "floor_ms"
                          and not k.startswith("bn_")}
    print(json.dumps(r), flush=True)
