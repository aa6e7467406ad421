import sys, torch
sys.path.insert(0, ".")
from paper_2008_11421_b200 import bnfused, _lib
def t(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps * 1e-3
for c, hw in ((64, 56), (256, 14), (128, 28), (512, 7)):
    n = 3072
    mk = lambda: torch.randn(n, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    x, dy = mk(), mk()
    g = torch.ones(c, device="cuda", dtype=torch.bfloat16); b = torch.zeros(c, device="cuda", dtype=torch.bfloat16)
    m, i = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    dg, db = torch.empty(c, device="cuda"), torch.empty(c, device="cuda")
    bnfused.stats(x, m, i)
    coef = torch.randn(3 * c, device="cuda")
    dx = torch.empty_like(x)
    rows = n * hw * hw
    full = t(lambda: bnfused.backward(dy, x, m, i, g, b, relu=True, dgamma=dg, dbeta=db))
    el = t(lambda: _lib.lib().krt_bn_backward_elemt(dy.data_ptr(), x.data_ptr(), m.data_ptr(), i.data_ptr(), g.data_ptr(), b.data_ptr(), coef.data_ptr(), None, 1, dx.data_ptr(), rows, c, None))
    nb = x.numel() * 2
    red = full - el
    print(f"C={c} hw={hw}: full {full*1e6:.0f}us ({5*nb/full/1e9:.0f} GB/s)  elemt {el*1e6:.0f}us ({3*nb/el/1e9:.0f} GB/s)  reduce {red*1e6:.0f}us ({2*nb/red/1e9:.0f} GB/s)")
    del x, dy, dx; torch.cuda.empty_cache()
