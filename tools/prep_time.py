"""Times K1 (preprocess class) alone via the context's kernel timers for
n samples of the config-2 workload; prints ms per 2^20 samples."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
K, N, L = 20, 30, 40
ctx = eng.Context(0)
m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
for snr in (0.0, 10.0, 14.0):
    base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131 + 5))
    ctx.generate(base, 0, n, N, K, snr, snr, 1.0 / np.sqrt(N), H, y, x)
    m.batch_evaluate_device(n, H, y, x)
    ctx.set_profiling(True)
    ctx.kernel_times(reset=True)
    for _ in range(3):
        ev = m.batch_evaluate_device(n, H, y, x)
    t = ctx.kernel_times(reset=True)
    ctx.set_profiling(False)
    scale = (1 << 20) / n / 3
    print(f"snr {snr}: preprocess {t['preprocess'][0]*scale:.3f} ms/2^20, fallback(other) "
          f"{t['other'][0]*scale:.3f}, stack {t['stack'][0]*scale:.3f}  {ev}")
