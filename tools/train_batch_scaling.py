"""Device-resident training step time vs batch size (L=40, group LASSO)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
K, N, L = 20, 30, 40
ctx = eng.Context(0)
out = {}
for n in (500, 1000, 5000, 20000, 50000, 100000):
    H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
    y = torch.empty((n, N), dtype=torch.float32, device="cuda")
    x = torch.empty((n, K), dtype=torch.int8, device="cuda")
    base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 2))
    ctx.generate(base, 0, n, N, K, 7.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
    m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
    raw = m.new_raw()
    for _ in range(3):
        m.train_grad(n, H, y, x, raw, want_eval=False); m.train_apply(raw, n, lr0=1e-3, kind=2, lam1=1e-4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        m.train_grad(n, H, y, x, raw, want_eval=False); m.train_apply(raw, n, lr0=1e-3, kind=2, lam1=1e-4)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[n] = {"ms_per_step": round(ms, 4), "samples_per_s": round(n / ms * 1e3)}
    m.close(); del H, y, x
print(json.dumps(out))
