"""Per-layer / per-tensor comparison of the GPU batch gradient with the oracle (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import Model as OModel, Oracle, record_slices
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
K, N, L, n = [int(a) for a in sys.argv[1:5]] if len(sys.argv) > 4 else (4, 8, 3, 64)
orc = Oracle()
params = xavier_params(K, L, seed=5)
r = orc.rng(2, 0)
H, x, y, _ = orc.generate_batch(r, N, K, n, 7.0, 14.0)
H32 = (H / np.sqrt(N)).astype(np.float32); y32 = (y / np.sqrt(N)).astype(np.float32)
ctx = eng.Context(0)
m = ctx.model(K, N, 8 * K, 2 * K, params)
ev, g = m.batch_gradient(H32, y32, x.astype(np.int8))
om = OModel(K, N, 8 * K, 2 * K, L, params)
ref = orc.batch_gradient(om, H32.astype(np.float64), y32.astype(np.float64), x)
print("loss", ev.data_loss, ref["data_loss"])
sl = record_slices(K, 8 * K, 2 * K)
for l in range(L):
    for name, s in sl.items():
        a, b = g[l, s], ref["grads"][l, s]
        print(l, name, f"max|ref|={np.max(np.abs(b)):.3e} maxerr={np.max(np.abs(a-b)):.3e}", a[:3], b[:3])
