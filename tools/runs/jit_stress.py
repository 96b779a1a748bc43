import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from test_sparse_jit_gpu import _sparse_model
from test_parity_gpu import _inputs, _omodel, _e2e_ok
from oracle.oracle import Oracle
from paper_2003_09446_b200 import Context
orc = Oracle()
c = Context(0)
for K, L, keep in ((20, 90, 0.02), (32, 4, 0.02)):
    p, m = _sparse_model(K, L, seed=3, keep=keep)
    H, y, x = _inputs(orc, 300, K=K, N=2 * K, seed=1)
    t = time.perf_counter()
    mod = c.model(K, 2 * K, 8 * K, 2 * K, p, masks=m)
    ev, xh = mod.batch_evaluate(H, y, x, want_xhat=True)
    dt = time.perf_counter() - t
    ref = orc.evaluate(_omodel(p, K=K, N=2 * K, masks=m), H.astype(np.float64), y.astype(np.float64), x.astype(np.float64), want_xhat=True)
    print(K, L, mod.path_name, "first eval s", round(dt, 1), "e2e", _e2e_ok(xh, ref["xhat"]), ev.symbol_errors, int(ref["errors"].sum()))
