"""Compare the tcgen05 path with the SIMT path on small inputs (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params

K, N = 20, 30
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
rs = np.random.default_rng(0)
H = (rs.standard_normal((n, N, K)) / np.sqrt(N)).astype(np.float32)
x = np.where(rs.random((n, K)) > 0.5, 1, -1).astype(np.int8)
y = (np.einsum("snk,sk->sn", H.astype(np.float64), x) + 0.3 * rs.standard_normal((n, N)) / np.sqrt(N)).astype(np.float32)
params = xavier_params(K, L, seed=9)
ctx = eng.Context(0)
m = ctx.model(K, N, 160, 40, params)
ctx.set_path(1)
ev1, xh1 = m.batch_evaluate(H, y, x, want_xhat=True)
ctx.set_path(2)
print("tc path:", m.path_name)
ev2, xh2 = m.batch_evaluate(H, y, x, want_xhat=True)
d = np.abs(xh1 - xh2)
print("max |dx| per layer:", d.max(axis=(0, 2)))
print("simt", ev1, "\ntc  ", ev2)
print("sample 0 layer 0 simt:", xh1[0, 0, :6], "\n                  tc:", xh2[0, 0, :6])
