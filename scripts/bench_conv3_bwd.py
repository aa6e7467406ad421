"""Backward of a bottleneck's conv3 (1x1, w -> 4w) at ResNet-200 stage
shapes, batch from argv: the current path (bn_apply of a2 = relu(bn2(c2)),
cuDNN dgrad+wgrad in one call, BN2 backward) vs own tcgen05 kernels (1x1
dgrad GEMM with BN2's backward reduce in its epilogue + elementwise pass, 1x1
wgrad GEMM with relu(bn2(.)) applied to c2 in shared memory: a2 never
exists).  Also conv1's backward (x -> w, no prologue on x).  Median of 10."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

aten = torch.ops.aten
torch.backends.cudnn.benchmark = True


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
    return round(ts[len(ts) // 2], 4)


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
for (w, side) in [(64, 56), (128, 28), (256, 14), (512, 7)]:
    c2 = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
    dc3 = cl(torch.randn(n, 4 * w, side, side, device="cuda").to(torch.bfloat16))
    w3 = (torch.randn(4 * w, 1, 1, w, device="cuda") * w ** -0.5).to(torch.bfloat16)   # OHWI
    g = torch.ones(w, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(w, device="cuda", dtype=torch.bfloat16)
    m, i = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
    bnfused.stats(c2, m, i)
    dg, db = torch.empty(w, device="cuda"), torch.empty(w, device="cuda")
    gw3 = torch.empty(4 * w, 1, 1, w, device="cuda")
    w3n = w3.permute(0, 3, 1, 2)

    def cur():
        a2 = bnfused.apply(c2, m, i, g, b, relu=True)
        da2, dw3, _ = aten.convolution_backward(dc3, a2, w3n, None, [1, 1], [0, 0], [1, 1], False, [0, 0], 1,
                                                [True, True, False])
        gw3.copy_(dw3.permute(0, 2, 3, 1))
        bnfused.backward(da2, c2, m, i, g, b, relu=True, dgamma=dg, dbeta=db)

    def own():
        bnfused.conv_wgrad(dc3, c2, gw3, 1, 1, 0, pre=(m, i, g, b))
        bnfused.conv1x1_dgrad_bn_backward(dc3, w3n, c2, m, i, g, b, dgamma=dg, dbeta=db)

    def mixed():   # own wgrad (no a2), cuDNN dgrad + BN backward
        bnfused.conv_wgrad(dc3, c2, gw3, 1, 1, 0, pre=(m, i, g, b))
        da2, _, _ = aten.convolution_backward(dc3, c2, w3n, None, [1, 1], [0, 0], [1, 1], False, [0, 0], 1,
                                              [True, False, False])
        bnfused.backward(da2, c2, m, i, g, b, relu=True, dgamma=dg, dbeta=db)
    r = {"w": w, "side": side, "batch": n, "conv3_bwd_current": timeit(cur)}
    if w >= 64 and 4 * w % 128 == 0:
        r["conv3_bwd_own"] = timeit(own)
        r["conv3_bwd_ownwgrad_cudnn_dgrad"] = timeit(mixed)
    # conv1 (4w -> w): wgrad without prologue (x is the unit input)
    x = cl(torch.randn(n, 4 * w, side, side, device="cuda").to(torch.bfloat16))
    dc1 = cl(torch.randn(n, w, side, side, device="cuda").to(torch.bfloat16))
    w1n = (torch.randn(w, 4 * w, 1, 1, device="cuda") * (4 * w) ** -0.5).to(torch.bfloat16)
    gw1 = torch.empty(w, 1, 1, 4 * w, device="cuda")
    r["conv1_wgrad_cudnn"] = timeit(lambda: aten.convolution_backward(dc1, x, w1n, None, [1, 1], [0, 0], [1, 1], False,
                                                                      [0, 0], 1, [False, True, False]))
    if w % 128 == 0:
        r["conv1_wgrad_own"] = timeit(lambda: bnfused.conv_wgrad(dc1, x, gw1, 1, 1, 0))
    print(json.dumps(r), flush=True)
