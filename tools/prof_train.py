"""Profiling driver for the training kernels: config-5 training steps (L=40,
batch 5000, sparse-group LASSO, Adam) through detnet_train_grad /
detnet_train_apply after warm-up steps. Used under ncu (-k regex:k_bwd_tc /
k_dw_tc / k_stack_h16). argv: steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_09446_b200 as eng  # noqa: E402
from paper_2003_09446_b200.workload import xavier_params  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K, N, L, n = 20, 30, 40, 5000
ctx = eng.Context(0)
m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
raw = m.new_raw()
base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 2))
ctx.generate(base, 0, n, N, K, 7.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
for _ in range(steps):
    m.train_grad(n, H, y, x, raw, want_eval=False)
    m.train_apply(raw, n, kind=2, lam1=1e-4, lr0=1e-3)
torch.cuda.synchronize()
obj, _ = m.train_status()
print("objective", obj)
