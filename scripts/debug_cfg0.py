import json, sys
import numpy as np, torch
sys.path.insert(0, '.')
torch.backends.cuda.matmul.allow_tf32 = False
from oracle import fc_chain_oracle as orc
from paper_2008_11421_b200.executor import ExecConfig, Executor
from paper_2008_11421_b200.plan import PlanBundle
from paper_2008_11421_b200.units import FCUnit, mse_zero_loss
cases = json.load(open('tests/golden/sched_cases.json'))['cases']
c = next(x for x in cases if x['name'] == 'cfg0_fc_chain')
w0 = orc.init_weights()
# torch CUDA in-core autograd reference, fp64 reference too
def torch_ref(dev, dt, its=3, lr=1e-2):
    ws = [torch.tensor(w, dtype=dt, device=dev, requires_grad=True) for w in w0]
    for it in range(1, its + 1):
        y = torch.tensor(orc.inputs(0, it), dtype=dt, device=dev)
        for w in ws: y = y @ w.T
        l = (y * y).mean(); l.backward()
        with torch.no_grad():
            for w in ws: w -= lr * w.grad; w.grad = None
    return [w.detach().cpu().double().numpy() for w in ws]
r64 = torch_ref('cpu', torch.float64)
rcu = torch_ref('cuda', torch.float32)
_, rnp = orc.train(workers=1, iterations=3, optimizer='sgd', lr=1e-2, weights=w0)
for plan_name in ('gold',):
    b = PlanBundle(c['model'], c['hardware'], c['plan'])
    ex = Executor([FCUnit(64, 64) for _ in range(6)], b, batch=2, loss_fn=mse_zero_loss, cfg=ExecConfig(optimizer='sgd', lr=1e-2))
    ex.load_weights({i + 1: [torch.from_numpy(w)] for i, w in enumerate(w0)})
    for it in range(1, 4):
        ex.step(torch.from_numpy(orc.inputs(0, it)).cuda())
    ex.synchronize()
    got = ex.unit_weights()
    for i in range(6):
        g = got[i + 1][0].cpu().double().numpy()
        print(i + 1, 'exec-vs-f64 %.3e' % np.abs(g - r64[i]).max(), 'np-vs-f64 %.3e' % np.abs(rnp[i] - r64[i]).max(),
              'cuda-vs-f64 %.3e' % np.abs(rcu[i] - r64[i]).max(), 'update mag %.3e' % np.abs(r64[i] - w0[i]).max())
    print(ex.trace_csv())
    print(ex.stats())
