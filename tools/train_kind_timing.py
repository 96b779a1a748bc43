"""Time of one device-resident training step (config-5 shape) per loss kind:
plain, element L1, group LASSO, sparse-group LASSO (loss.cpp:35-91)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
K, N, L, n = 20, 30, 40, 5000
ctx = eng.Context(0)
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 2))
ctx.generate(base, 0, n, N, K, 7.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
out = {}
for name, kw in (("plain", dict(kind=0)), ("element_l1", dict(kind=1, lam=1e-5)),
                 ("group", dict(kind=2, lam1=1e-4)), ("sparse_group", dict(kind=2, lam1=1e-4, lam2=1e-5))):
    m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
    raw = m.new_raw()
    for _ in range(3):
        m.train_grad(n, H, y, x, raw, want_eval=False); m.train_apply(raw, n, lr0=1e-3, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        m.train_grad(n, H, y, x, raw, want_eval=False); m.train_apply(raw, n, lr0=1e-3, **kw)
    e1.record(); torch.cuda.synchronize()
    obj, reg = m.train_status()
    out[name] = {"ms_per_step": e0.elapsed_time(e1) / 20, "objective": obj, "regularizer": reg}
    m.close()
print(json.dumps(out))
