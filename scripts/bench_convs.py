"""Own tcgen05 convolutions vs cuDNN at ResNet-200 shapes (batch 256 per
launch, bf16): 3x3 fprop with relu(bn) prologue + statistics epilogue vs
bn_apply + cuDNN + bn_stats; 3x3 dgrad with the BN-backward reduce vs cuDNN
dgrad + bn_backward; wgrad (1x1 and 3x3, BN prologue) vs bn_apply + cuDNN
wgrad.  CUDA events, median of 20 after 5 warm-ups.  Prints one JSON line
per shape."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_11421_b200 import bnfused  # noqa: E402

aten = torch.ops.aten
torch.backends.cudnn.benchmark = True


def timeit(fn, reps=20, warm=5):
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


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    dev = "cuda"
    for (w, side) in [(64, 56), (128, 28), (256, 14), (512, 7)]:
        x = cl(torch.randn(n, w, side, side, device=dev).to(torch.bfloat16))
        dy = cl(torch.randn(n, w, side, side, device=dev).to(torch.bfloat16))
        wt = (torch.randn(w, 3, 3, w, device=dev) * (9 * w) ** -0.5).to(torch.bfloat16)
        g = torch.ones(w, device=dev, dtype=torch.bfloat16)
        b = torch.zeros(w, device=dev, dtype=torch.bfloat16)
        m, i = torch.empty(w, device=dev), torch.empty(w, device=dev)
        bnfused.stats(x, m, i)
        wn = wt.permute(0, 3, 1, 2)
        fl3 = 2.0 * n * side * side * 9 * w * w
        sm, si = torch.empty(w, device=dev), torch.empty(w, device=dev)
        own_f = timeit(lambda: bnfused.conv_im2col(x, wt, 1, 1, pre=(m, i, g, b), stats=(sm, si)))

        def cudnn_f():
            a = bnfused.apply(x, m, i, g, b, relu=True)
            c = aten.convolution(a, wn, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1)
            bnfused.stats(c, sm, si)
        ref_f = timeit(cudnn_f)
        dg, db = torch.empty(w, device=dev), torch.empty(w, device=dev)
        own_d = timeit(lambda: bnfused.conv_im2col_dgrad_bn_backward(dy, wt, x, m, i, g, b, dgamma=dg, dbeta=db))

        def cudnn_d():
            a = bnfused.apply(x, m, i, g, b, relu=True)
            da, _, _ = aten.convolution_backward(dy, a, wn, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1,
                                                 [True, False, False])
            bnfused.backward(da, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db)
        ref_d = timeit(cudnn_d)
        dw = torch.empty(w, 3, 3, w, device=dev)
        own_w = timeit(lambda: bnfused.conv_wgrad(dy, x, dw, 3, 1, 1, pre=(m, i, g, b))) if w >= 128 else None

        def cudnn_w():
            a = bnfused.apply(x, m, i, g, b, relu=True)
            _, gw, _ = aten.convolution_backward(dy, a, wn, None, [1, 1], [1, 1], [1, 1], False, [0, 0], 1,
                                                 [False, True, False])
            dw.copy_(gw.permute(0, 2, 3, 1))
        ref_w = timeit(cudnn_w)
        # 1x1 wgrads of the same stage: conv3 (w -> 4w, prologue on c2), conv1 (4w -> w, no prologue)
        x4 = cl(torch.randn(n, 4 * w, side, side, device=dev).to(torch.bfloat16))
        dy4 = cl(torch.randn(n, 4 * w, side, side, device=dev).to(torch.bfloat16))
        dw3 = torch.empty(4 * w, 1, 1, w, device=dev)
        own_w3 = timeit(lambda: bnfused.conv_wgrad(dy4, x, dw3, 1, 1, 0, pre=(m, i, g, b)))

        def cudnn_w3():
            a = bnfused.apply(x, m, i, g, b, relu=True)
            _, gw, _ = aten.convolution_backward(dy4, a, dw3.new_empty(4 * w, w, 1, 1).to(torch.bfloat16), None,
                                                 [1, 1], [0, 0], [1, 1], False, [0, 0], 1, [False, True, False])
        ref_w3 = timeit(cudnn_w3)
        dw1 = torch.empty(w, 1, 1, 4 * w, device=dev)
        own_w1 = timeit(lambda: bnfused.conv_wgrad(dy, x4, dw1, 1, 1, 0)) if w >= 128 else None

        def cudnn_w1():
            _, gw, _ = aten.convolution_backward(dy, x4, dw1.new_empty(w, 4 * w, 1, 1).to(torch.bfloat16), None,
                                                 [1, 1], [0, 0], [1, 1], False, [0, 0], 1, [False, True, False])
        ref_w1 = timeit(cudnn_w1) if w >= 128 else None
        fl1 = 2.0 * n * side * side * 4 * w * w
        print(json.dumps({
            "stage_width": w, "side": side, "batch": n,
            "fprop3x3_ms": [own_f, ref_f], "fprop3x3_own_TFLOPs": fl3 / own_f / 1e9,
            "dgrad3x3_ms": [own_d, ref_d], "dgrad3x3_own_TFLOPs": fl3 / own_d / 1e9,
            "wgrad3x3_ms": [own_w, ref_w], "wgrad3x3_own_TFLOPs": fl3 / own_w / 1e9 if own_w else None,
            "wgrad1x1_conv3_ms": [own_w3, ref_w3], "wgrad1x1_conv3_own_TFLOPs": fl1 / own_w3 / 1e9,
            "wgrad1x1_conv1_ms": [own_w1, ref_w1], "wgrad1x1_conv1_own_TFLOPs": fl1 / own_w1 / 1e9 if own_w1 else None,
            "note": "[own, cudnn incl. the bn passes it needs]"}), flush=True)


if __name__ == "__main__":
    main()
