import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200 import workload as wl
K, N, L, n = 20, 30, 40, 5000
ctx = eng.Context(0)
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 2))
ctx.generate(base, 0, n, N, K, 7.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
out = {}
params = wl.xavier_params(K, L, seed=9)
gm = wl.group_masks(K, L, seed=31)
sp, sm = wl.sparse_group_model(params, gm, K)
for name, (p, m_, fr) in (("dense", (params, None, 0)), ("group_masked", (params, gm, 0)), ("sparse_group_masked", (sp, sm, 0)),
                      ("dense_frozen30", (params, None, 30))):
    m = ctx.model(K, N, 160, 40, p, masks=m_, frozen_prefix=fr)
    raw = m.new_raw()
    to = fr > 0
    for _ in range(3):
        m.train_grad(n, H, y, x, raw, trainable_only=to, want_eval=False); m.train_apply(raw, n, lr0=1e-3, kind=2, lam1=1e-4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        m.train_grad(n, H, y, x, raw, trainable_only=to, want_eval=False); m.train_apply(raw, n, lr0=1e-3, kind=2, lam1=1e-4)
    e1.record(); torch.cuda.synchronize()
    ev = m.batch_evaluate_device(n, H, y, x)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(5): ev = m.batch_evaluate_device(n, H, y, x)
    t1.record(); torch.cuda.synchronize()
    out[name] = {"train_ms_per_step": e0.elapsed_time(e1) / 20, "eval_ms": t0.elapsed_time(t1)/5, "eval_path": m.path_name, "loss": ev.data_loss}
    m.close()
print(json.dumps(out))
