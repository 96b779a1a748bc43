import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_2003_09446_b200 import Context
c = Context(0)
for nb in (4, 12, 36, 4, 12, 36):
    t = time.perf_counter()
    recs, res, _ = c.train_incremental(20, 30, 40, 10, 40, nb, 5000, 2000, 3, halt_epsilon=0.0,
                                       val_snr_db=10.0, snr_lo_db=7.0, snr_hi_db=14.0, lr0=1e-3,
                                       kind=2, lam1=1e-4)
    print(nb, "host", round((time.perf_counter() - t) * 1e3, 2), "ms; res", round(res["seconds"] * 1e3, 2),
          "ms; steps", res["optimizer_steps"], "wall_ms", [round(r["wall_ms"], 2) for r in recs])
