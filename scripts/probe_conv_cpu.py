import time, torch
torch.backends.cudnn.benchmark = True
aten = torch.ops.aten
cl = lambda t: t.contiguous(memory_format=torch.channels_last)
for (n, c, hw, k) in ((2, 16, 256, 3), (2, 64, 128, 1)):
    x = cl(torch.randn(n, c, hw, hw, device="cuda", dtype=torch.bfloat16))
    w = cl(torch.randn(c, c, k, k, device="cuda", dtype=torch.bfloat16))
    y = aten.convolution(x, w, None, [1, 1], [k // 2] * 2, [1, 1], False, [0, 0], 1)
    dy = cl(torch.randn_like(y))
    for mask in ([True, True, False], [False, True, False]):
        for _ in range(3):
            aten.convolution_backward(dy, x, w, None, [1, 1], [k // 2] * 2, [1, 1], False, [0, 0], 1, mask)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            aten.convolution_backward(dy, x, w, None, [1, 1], [k // 2] * 2, [1, 1], False, [0, 0], 1, mask)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"n{n} c{c} hw{hw} k{k} mask{mask}: cpu issue {(t1-t0)/50*1e6:.0f} us/call, wall {(t2-t0)/50*1e6:.0f} us/call", flush=True)
    t0 = time.perf_counter()
    for _ in range(50):
        aten.convolution(x, w, None, [1, 1], [k // 2] * 2, [1, 1], False, [0, 0], 1)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"  fprop: cpu issue {(t1-t0)/50*1e6:.0f} us/call, wall {(t2-t0)/50*1e6:.0f}", flush=True)
