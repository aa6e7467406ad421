import sys, torch
sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused
def t(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps * 1e-3
cl = lambda z: z.contiguous(memory_format=torch.channels_last)
n, side = 2, 2048
for cin, cout in ((16, 64), (64, 16), (32, 128)):
    x = cl(torch.randn(n, cin, side, side, device="cuda", dtype=torch.bfloat16))
    w = cl(torch.randn(cout, cin, 1, 1, device="cuda", dtype=torch.bfloat16) * 0.1)
    r = cl(torch.randn(n, cout, side, side, device="cuda", dtype=torch.bfloat16))
    y = cl(torch.empty(n, cout, side, side, device="cuda", dtype=torch.bfloat16))
    g = torch.ones(cin, device="cuda", dtype=torch.bfloat16); b = torch.zeros(cin, device="cuda", dtype=torch.bfloat16)
    m, i = torch.empty(cin, device="cuda"), torch.empty(cin, device="cuda"); bnfused.stats(x, m, i)
    so = (torch.empty(cout, device="cuda"), torch.empty(cout, device="cuda"))
    M = n * side * side
    for name, fn, nb in (("plain", lambda: bnfused.conv1x1(x, w, out=y), M * (cin + cout) * 2),
                         ("pre", lambda: bnfused.conv1x1(x, w, out=y, pre=(m, i, g, b)), M * (cin + cout) * 2),
                         ("stats", lambda: bnfused.conv1x1(x, w, out=y, stats=so), M * (cin + cout) * 2),
                         ("res", lambda: bnfused.conv1x1(x, w, out=y, res=r), M * (cin + 2 * cout) * 2),
                         ("pre_res", lambda: bnfused.conv1x1(x, w, out=y, pre=(m, i, g, b), res=r), M * (cin + 2 * cout) * 2)):
        sec = t(fn)
        print(f"K={cin} N={cout} {name:8s} {sec*1e6:7.1f} us {nb/sec/1e9:6.0f} GB/s", flush=True)
