"""CPU-side checks: the C ABI loads and exports every symbol of
include/krt.h; the host optimizer matches torch/numpy; the oracle is sane."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import torch

from oracle import fc_chain_oracle as orc
from paper_2008_11421_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def test_every_header_symbol_exported():
    hdr = (ROOT / "include" / "krt.h").read_text()
    names = set(re.findall(r"\b(krt_[a-z_0-9]+)\s*\(", hdr))
    names -= {"krt_compute_cb"}
    so = C.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in sorted(names) if not hasattr(so, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) >= names
    assert b"sm_100a" in _lib.lib().krt_version()


def test_host_adam_matches_torch():
    n = 4099
    g = torch.Generator().manual_seed(1)
    p = torch.randn(n, generator=g)
    grad = torch.randn(n, generator=g)
    hp, hm, hv = p.clone(), torch.zeros(n), torch.zeros(n)
    w32 = torch.empty(n)
    L = _lib.lib()
    ref = p.clone().requires_grad_(True)
    opt = torch.optim.Adam([ref], lr=1e-3, weight_decay=0.01, foreach=False)
    for step in range(1, 6):
        _lib.check(L.krt_host_update(hp.data_ptr(), hm.data_ptr(), hv.data_ptr(), grad.data_ptr(),
                                     w32.data_ptr(), _lib.F32, n, _lib.ADAM, 1e-3, 0.9, 0.999, 1e-8,
                                     0.01, 0.0, step, 3))
        ref.grad = grad.clone()
        opt.step()
    torch.testing.assert_close(hp, ref.detach(), rtol=1e-6, atol=1e-7)
    assert torch.equal(w32, hp)


def test_host_sgd_momentum_matches_torch():
    n = 1000
    g = torch.Generator().manual_seed(2)
    p = torch.randn(n, generator=g)
    hp, hm = p.clone(), torch.zeros(n)
    ref = p.clone().requires_grad_(True)
    opt = torch.optim.SGD([ref], lr=0.1, momentum=0.9, foreach=False)
    L = _lib.lib()
    for step in range(1, 4):
        grad = torch.randn(n, generator=g)
        _lib.check(L.krt_host_update(hp.data_ptr(), hm.data_ptr(), None, grad.data_ptr(), None,
                                     _lib.F32, n, _lib.SGD, 0.1, 0.9, 0.999, 1e-8, 0.0, 0.9, step, 1))
        ref.grad = grad.clone()
        opt.step()
    torch.testing.assert_close(hp, ref.detach(), rtol=1e-6, atol=1e-6)


def test_host_bf16_rounding_is_rne():
    n = 64
    p = torch.tensor([1.0 + k * 2 ** -9 for k in range(n)], dtype=torch.float32)
    grad = torch.zeros(n)
    hw = torch.empty(n, dtype=torch.bfloat16)
    hm = torch.zeros(n)
    _lib.check(_lib.lib().krt_host_update(p.data_ptr(), hm.data_ptr(), None, grad.data_ptr(),
                                          hw.data_ptr(), _lib.BF16, n, _lib.SGD, 0.0, 0.9, 0.999,
                                          1e-8, 0.0, 0.0, 1, 1))
    assert torch.equal(hw, p.to(torch.bfloat16))


def test_oracle_gradients_match_torch_autograd():
    ws = orc.init_weights()
    x = orc.inputs(0, 1)
    loss, grads = orc.forward_backward(ws, x)
    tw = [torch.tensor(w, requires_grad=True) for w in ws]
    y = torch.tensor(x)
    for w in tw:
        y = y @ w.T
    tl = (y * y).mean()
    tl.backward()
    assert abs(float(tl) - float(loss)) <= 1e-6 * abs(float(loss))
    for g, w in zip(grads, tw):
        np.testing.assert_allclose(g, w.grad.numpy(), rtol=1e-5, atol=1e-8)


def test_oracle_dp_mean_equals_concatenated_batch():
    # 2 workers x batch 2 with mean exchange == 1 worker on the batch of 4
    ws = orc.init_weights()
    _, g0 = orc.forward_backward(ws, orc.inputs(0, 1))
    _, g1 = orc.forward_backward(ws, orc.inputs(1, 1))
    _, gc = orc.forward_backward(ws, np.concatenate([orc.inputs(0, 1), orc.inputs(1, 1)]))
    for a, b, c in zip(g0, g1, gc):
        np.testing.assert_allclose((a + b) / 2, c, rtol=1e-5, atol=1e-7)
