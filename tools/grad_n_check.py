"""Debug: batch_gradient vs the FP64 oracle at several batch sizes (dW splits)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
from oracle.oracle import Oracle, Model as OModel
K, N, L = 20, 30, 6
orc = Oracle()
ctx = eng.Context(0)
p = xavier_params(K, L, seed=9)
for n in (192, 256, 300, 1000, 4000):
    H, x, y, _ = orc.generate_batch(orc.rng(1, 2), N, K, n, 7.0, 14.0)
    H32 = (H / np.sqrt(N)).astype(np.float32); y32 = (y / np.sqrt(N)).astype(np.float32)
    m = ctx.model(K, N, 160, 40, p)
    ev, g = m.batch_gradient(H32, y32, x.astype(np.int8), kind=2, lam1=1e-4)
    ref = orc.batch_gradient(OModel(K, N, 160, 40, L, p), H32.astype(np.float64), y32.astype(np.float64), x, kind=2, lam1=1e-4)
    gr = ref["grads"]
    d = np.abs(g - gr)
    print(n, "loss rel", abs(ev.data_loss - ref["data_loss"]) / ref["data_loss"], "max|dg|/max|g|", d.max() / np.abs(gr).max(),
          "median rel", np.median(d / (np.abs(gr) + 1e-30)))
