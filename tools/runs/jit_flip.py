import sys, os, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_parity_gpu import _inputs, _omodel, K, N
from oracle.oracle import Oracle
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import group_masks, sparse_group_model, xavier_params
orc = Oracle()
params = xavier_params(K, 8, seed=9)
ps, ms = sparse_group_model(params, group_masks(K, 8, seed=31), K)
H, y, x = _inputs(orc, 512)
ctx = eng.Context(0)
for env in (None, "DETNET_NO_JIT"):
    if env: os.environ[env] = "1"
    m = ctx.model(K, N, 160, 40, ps, masks=ms)
    ev, xh = m.batch_evaluate(H, y, x, want_xhat=True)
    ref = orc.evaluate(_omodel(ps, masks=ms), H.astype(np.float64), y.astype(np.float64), x.astype(np.float64), want_xhat=True)
    xl = xh.reshape(512, 8, K)[:, -1]; rl = ref["xhat"].reshape(512, 8, K)[:, -1]
    d = (xl >= 0) != (rl >= 0)
    print(m.path_name, ev.symbol_errors, int(ref["errors"].sum()), "flips", d.sum(), "x at flips", xl[d][:10], "ref", rl[d][:10])
    print("max abs diff all layers", np.abs(xh - ref["xhat"].reshape(xh.shape)).max())
