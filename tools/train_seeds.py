"""Debug: distribution of the 100-step FP32-vs-FP64 training drift over seeds
(final validation loss relative difference, as in test_train_gpu)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import Model as OModel, Oracle
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
K, N, L, steps = 20, 30, 6, 100
n = int(sys.argv[1]) if len(sys.argv) > 1 else 192
L = int(sys.argv[2]) if len(sys.argv) > 2 else L
orc = Oracle()
ctx = eng.Context(0)
if os.environ.get("TC_FWD"): ctx.set_train_forward(True)
ctx.set_path(int(os.environ.get("TC_PATH", "0")))  # 0 split-FP16, 2 3xTF32 (tensor-core forward)
pairs = [(9, 1), (9, 2), (10, 1), (11, 3), (12, 4)]
pairs += [(20 + i, 30 + i) for i in range(int(os.environ.get("EXTRA_SEEDS", "0")))]
finals, tracked = [], []
for pseed, dseed in pairs:
    params = xavier_params(K, L, seed=pseed)
    m = ctx.model(K, N, 8 * K, 2 * K, params)
    om = OModel(K, N, 8 * K, 2 * K, L, params.copy())
    mo1 = np.zeros_like(params); mo2 = np.zeros_like(params)
    raw = m.new_raw()
    train_rng = orc.lib.or_stream(C.byref(orc.rng(dseed, 0)), 2)
    val_rng = orc.lib.or_stream(C.byref(orc.rng(dseed, 0)), 3)
    Hv, xv, yv, _ = orc.generate_batch(val_rng, N, K, 2000, 12.0, 12.0)
    Hv32 = (Hv / np.sqrt(N)).astype(np.float32); yv32 = (yv / np.sqrt(N)).astype(np.float32)
    s_or = 0
    rels = []
    for step in range(steps):
        H, x, y, _ = orc.generate_batch(train_rng, N, K, n, 7.0, 14.0)
        H32 = (H / np.sqrt(N)).astype(np.float32); y32 = (y / np.sqrt(N)).astype(np.float32)
        Hd, yd, xd = (torch.from_numpy(a).cuda() for a in (H32, y32, x.astype(np.int8)))
        ev = m.train_grad(n, Hd, yd, xd, raw)
        m.train_apply(raw, n, kind=2, lam1=1e-4, lr0=1e-3)
        ref = orc.batch_gradient(om, H32.astype(np.float64), y32.astype(np.float64), x, kind=2, lam1=1e-4)
        s_or = orc.adam_step(om, ref["grads"], mo1, mo2, s_or, lr0=1e-3)
        rels.append(abs(ev.data_loss - ref["data_loss"]) / abs(ref["data_loss"]))
    mg = ctx.model(K, N, 8 * K, 2 * K, m.get_params())
    evg = mg.batch_evaluate(Hv32, yv32, xv.astype(np.int8))
    evo = orc.batch_evaluate(om, Hv32.astype(np.float64), yv32.astype(np.float64), xv)
    fr = abs(evg.data_loss - evo['data_loss']) / evo['data_loss']
    finals.append(fr)
    tracked.append(next((i for i, r in enumerate(rels) if r > 1e-5), len(rels)))
    print(f"seeds {pseed},{dseed}: tracked {tracked[-1]} max rel first10 {max(rels[:10]):.2e} first50 {max(rels[:50]):.2e} final val rel "
          f"{abs(evg.data_loss - evo['data_loss']) / evo['data_loss']:.2e}", flush=True)
print(f"SUMMARY fwd={'tc' if os.environ.get('TC_FWD') else 'simt'} path={os.environ.get('TC_PATH', '0')} "
      f"n={len(finals)} median final {np.median(finals):.2e} mean {np.mean(finals):.2e} "
      f"max {np.max(finals):.2e} median tracked {np.median(tracked)}", flush=True)
