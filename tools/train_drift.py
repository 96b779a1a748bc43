"""Per-step loss drift of the GPU training loop vs the oracle (debug aid)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import Model as OModel, Oracle
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
K, N, L, n, steps = 20, 30, int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
orc = Oracle()
params = xavier_params(K, L, seed=9)
ctx = eng.Context(0)
m = ctx.model(K, N, 8 * K, 2 * K, params)
om = OModel(K, N, 8 * K, 2 * K, L, params.copy())
mo1 = np.zeros_like(params); mo2 = np.zeros_like(params)
raw = m.new_raw()
train_rng = orc.lib.or_stream(C.byref(orc.rng(1, 0)), 2)
val_rng = orc.lib.or_stream(C.byref(orc.rng(1, 0)), 3)
Hv, xv, yv, _ = orc.generate_batch(val_rng, N, K, 2000, 12.0, 12.0)
Hv32 = (Hv / np.sqrt(N)).astype(np.float32); yv32 = (yv / np.sqrt(N)).astype(np.float32)
s_or = 0
for step in range(steps):
    H, x, y, _ = orc.generate_batch(train_rng, N, K, n, 7.0, 14.0)
    H32 = (H / np.sqrt(N)).astype(np.float32); y32 = (y / np.sqrt(N)).astype(np.float32)
    Hd, yd, xd = (torch.from_numpy(a).cuda() for a in (H32, y32, x.astype(np.int8)))
    ev = m.train_grad(n, Hd, yd, xd, raw)
    m.train_apply(raw, n, kind=2, lam1=1e-4, lr0=1e-3)
    ref = orc.batch_gradient(om, H32.astype(np.float64), y32.astype(np.float64), x, kind=2, lam1=1e-4)
    s_or = orc.adam_step(om, ref["grads"], mo1, mo2, s_or, lr0=1e-3)
    rel = abs(ev.data_loss - ref["data_loss"]) / abs(ref["data_loss"])
    if step % 10 == 0 or step == steps - 1:
        dp = np.max(np.abs(m.get_params() - om.params))
        print(f"step {step}: loss gpu {ev.data_loss:.6e} oracle {ref['data_loss']:.6e} rel {rel:.2e} max|dparam| {dp:.2e}")
# final models on a fixed validation set
mg = ctx.model(K, N, 8 * K, 2 * K, m.get_params())
evg = mg.batch_evaluate(Hv32, yv32, xv.astype(np.int8))
evo = orc.batch_evaluate(om, Hv32.astype(np.float64), yv32.astype(np.float64), xv)
print("final val loss gpu", evg.data_loss, "oracle", evo["data_loss"], "rel", abs(evg.data_loss - evo["data_loss"]) / evo["data_loss"],
      "ber", evg.ber(), evo["symbol_errors"] / evo["symbols"])
