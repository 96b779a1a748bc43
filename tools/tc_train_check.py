"""Debug: batch_gradient through the tcgen05 training forward vs the SIMT one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
from oracle.oracle import Oracle
K, N, L, n = 20, 30, int(sys.argv[1]) if len(sys.argv) > 1 else 6, 192
orc = Oracle()
H, x, y, _ = orc.generate_batch(orc.rng(1, 2), N, K, n, 7.0, 14.0)
H32 = (H / np.sqrt(N)).astype(np.float32); y32 = (y / np.sqrt(N)).astype(np.float32)
p = xavier_params(K, L, seed=9)
res = {}
for path in (0, 1):
    ctx = eng.Context(0, path=path)
    m = ctx.model(K, N, 160, 40, p)
    ev, g = m.batch_gradient(H32, y32, x.astype(np.int8), kind=0)
    res[path] = (ev, g)
    print(path, m.path_name, ev)
g0, g1 = res[0][1], res[1][1]
d = np.abs(g0 - g1)
print("max |dg|", d.max(), "max|g|", np.abs(g1).max(), "argmax", np.unravel_index(d.argmax(), d.shape))
from paper_2003_09446_b200.workload import record_layout
sl, P = record_layout(K, 160, 40)
for name, s_ in sl.items():
    dd = d[:, s_]
    print(name, dd.max() if dd.size else 0, np.abs(g1[:, s_]).max() if dd.size else 0)
