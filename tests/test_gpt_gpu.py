"""GPT decoder units (cfg3/cfg4 model family) under reference-planner plans
vs the CPU fp32 in-core oracle, and out-of-core vs in-core bitwise."""
import pytest
import torch

from oracle import gpt_oracle
from paper_2008_11421_b200 import workloads as W
from paper_2008_11421_b200.executor import ExecConfig, Executor
from paper_2008_11421_b200.units import lm_loss

pytestmark = pytest.mark.gpu


def batches(rec, iters, seed=0):
    g = torch.Generator().manual_seed(seed)
    m = rec["meta"]
    xs = [torch.randint(0, m["vocab"], (m["batch"], m["seq"]), generator=g) for _ in range(iters)]
    ys = [torch.randint(0, m["vocab"], (m["batch"], m["seq"]), generator=g) for _ in range(iters)]
    return xs, ys


def run(rec, plan=None, iters=3, lr=0.1, capacity=None, optimizer="sgd"):
    units = W.units_for(rec)
    b = W.bundle_for(rec, plan)
    if capacity:
        b.set_capacity(capacity)
    act = units[1].act
    ex = Executor(units, b, batch=rec["meta"]["batch"], loss_fn=lm_loss,
                  cfg=ExecConfig(optimizer=optimizer, lr=lr, weight_dtype=act))
    gen = torch.Generator().manual_seed(5)
    init = {i + 1: u.init_params(gen) for i, u in enumerate(units)}
    ex.load_weights(init)
    xs, ys = batches(rec, iters)
    losses = [float(ex.step(x.cuda().int(), y.cuda())) for x, y in zip(xs, ys)]
    w = ex.unit_weights()
    st = ex.stats()
    ex.close()
    return units, init, losses, w, st


@pytest.fixture(autouse=True)
def strict():
    old = (torch.backends.cuda.matmul.allow_tf32, torch.are_deterministic_algorithms_enabled())
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.use_deterministic_algorithms(True, warn_only=True)
    yield
    torch.backends.cuda.matmul.allow_tf32 = old[0]
    torch.use_deterministic_algorithms(old[1])


def test_gpt_plan_matches_cpu_oracle():
    rec = W.load("gpt_small_f32")
    assert any(b["recompute"] for b in rec["plan"]["blocks"]) and "in" in rec["plan_string"]
    units, init, losses, w, st = run(rec)
    assert st["iter_bytes_h2d"] > 0
    xs, ys = batches(rec, 3)
    ref_losses, ref_w = gpt_oracle.train(units, init, xs, ys, lr=0.1)
    torch.testing.assert_close(torch.tensor(losses), torch.tensor(ref_losses), rtol=1e-4, atol=1e-5)
    for k in ref_w:
        for got, ref in zip(w[k], ref_w[k]):
            torch.testing.assert_close(got.cpu().float(), ref, rtol=1e-3, atol=1e-5)


def test_gpt_bf16_out_of_core_equals_in_core_and_tracks_oracle():
    rec = W.load("gpt_small_bf16")
    units, init, l_ooc, w_ooc, s_ooc = run(rec, lr=0.05)
    _, _, l_inc, w_inc, _ = run(rec, plan=W.incore_plan(rec["plan"]), lr=0.05, capacity=1e12)
    assert s_ooc["iter_bytes_h2d"] > 0 and l_ooc == l_inc
    for k in w_inc:
        for a, b in zip(w_ooc[k], w_inc[k]):
            assert torch.equal(a, b), k
    xs, ys = batches(rec, 3)
    ref_losses, _ = gpt_oracle.train(units, init, xs, ys, lr=0.05)
    torch.testing.assert_close(torch.tensor(l_ooc), torch.tensor(ref_losses), rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("hidden,heads", [(256, 4), (608, 4)])
def test_cudnn_attention_matches_flash(monkeypatch, hidden, heads):
    """The decoder layer's attention on cuDNN's sm100 kernels (the bench
    path) vs aten's flash kernel (the deterministic path): output and every
    gradient agree to bf16 resolution.  Head dim 152 (Turing-NLG's 4256 / 28):
    cuDNN forward, its logsumexp handed to the flash backward."""
    from paper_2008_11421_b200 import units as U
    torch.use_deterministic_algorithms(False)
    u = U.TransformerLayerUnit(hidden, heads, 128)
    gen = torch.Generator().manual_seed(3)
    params = [p.to("cuda", torch.bfloat16) for p in u.init_params(gen)]
    x = (torch.randn(4 * 128, hidden, generator=gen)).to("cuda", torch.bfloat16)
    dy = (torch.randn(4 * 128, hidden, generator=gen)).to("cuda", torch.bfloat16)
    res = {}
    for flag in (False, True):
        monkeypatch.setattr(U, "ATTN_CUDNN", flag)
        saved = [torch.zeros(s.shape, dtype=s.dtype, device="cuda") for s in u.saved_specs(4)]
        grads = [torch.zeros(p.shape, dtype=torch.float32, device="cuda") for p in params]
        y = u.forward(x, params, saved)
        dx = u.backward(dy, params, saved, grads)
        res[flag] = [y.float(), dx.float()] + grads
    for a, b in zip(res[False], res[True]):
        assert ((a - b).norm() / b.norm()).item() <= 2e-2


@pytest.mark.parametrize("n,nh,s,hd,chunk", [(3, 2, 64, 152, 2), (1, 4, 256, 152, 8)])
def test_unfused_attention_backward_vs_fp32(n, nh, s, hd, chunk):
    """The unfused causal attention backward (head dims > 128: TF32 / bf16
    cuBLAS GEMMs + the own softmax-gradient pass) vs fp32 autograd of causal
    attention on the same bf16 q, k, v, dO: dQ, dK, dV within bf16 resolution."""
    import math
    from paper_2008_11421_b200 import units as U
    torch.use_deterministic_algorithms(False)
    u = U.TransformerLayerUnit(nh * hd, nh, s)
    g = torch.Generator(device="cuda").manual_seed(5)
    qkv = torch.randn(n * s, 3 * nh * hd, device="cuda", generator=g).to(torch.bfloat16)
    do = torch.randn(n * s, nh * hd, device="cuda", generator=g).to(torch.bfloat16)
    q, k, v = (t.float().requires_grad_(True) for t in u._heads(qkv))
    sc = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
    mask = torch.ones(s, s, dtype=torch.bool, device="cuda").triu(1)
    sc = sc.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(sc, dim=-1)
    o = torch.softmax(sc, dim=-1) @ v
    dO = do.view(n, s, nh, hd).transpose(1, 2)
    o.backward(dO.float())
    ob = o.detach().to(torch.bfloat16)
    qb, kb, vb = u._heads(qkv)
    d = u._attn_bw_unfused(dO, qb, kb, vb, ob, lse.detach().float(), n, chunk=chunk)
    got = d.view(n, s, 3, nh, hd)
    for i, ref in enumerate((q.grad, k.grad, v.grad)):
        x = got[:, :, i].transpose(1, 2).float()
        assert ((x - ref).norm() / ref.norm()).item() <= 1e-2, i
