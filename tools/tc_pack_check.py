"""Debug: tcgen05 images packed on the device after a training step vs the host packing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
from oracle.oracle import Oracle
K, N, L, n = 20, 30, 6, 192
orc = Oracle()
H, x, y, _ = orc.generate_batch(orc.rng(1, 2), N, K, n, 7.0, 14.0)
H32 = (H / np.sqrt(N)).astype(np.float32); y32 = (y / np.sqrt(N)).astype(np.float32)
ctx = eng.Context(0)
m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
raw = m.new_raw()
Hd, yd, xd = (torch.from_numpy(a).cuda() for a in (H32, y32, x.astype(np.int8)))
for step in range(3):
    ev = m.train_grad(n, Hd, yd, xd, raw)
    m.train_apply(raw, n, lr0=1e-3)
    e_dev, xh_dev = m.batch_evaluate(H32, y32, x.astype(np.int8), want_xhat=True)
    fresh = ctx.model(K, N, 160, 40, m.get_params())
    e_host, xh_host = fresh.batch_evaluate(H32, y32, x.astype(np.int8), want_xhat=True)
    print(step, "train-fwd loss", ev.data_loss, "dev-packed", e_dev.data_loss, "host-packed",
          e_host.data_loss, "max|dx|", np.abs(xh_dev - xh_host).max())
