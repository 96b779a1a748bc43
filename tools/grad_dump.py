"""Writes batch_gradient of a fixed seeded workload to argv[1] (.npy), for
bit-identity checks between kernel variants (DETNET_LIB / environment
switches read once per process). argv: out K N L n."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import Oracle
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
out, K, N, L, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
orc = Oracle()
H, x, y, _ = orc.generate_batch(orc.rng(2, 0), N, K, n, 7.0, 14.0)
H32 = (H / np.sqrt(N)).astype(np.float32)
y32 = (y / np.sqrt(N)).astype(np.float32)
ctx = eng.Context(0)
m = ctx.model(K, N, 8 * K, 2 * K, xavier_params(K, L, seed=9))
ev, g = m.batch_gradient(H32, y32, x.astype(np.int8), kind=2, lam=0.0, lam1=1e-4, lam2=0.0)
np.save(out, np.concatenate([g.ravel(), [ev.loss_sum]]))
