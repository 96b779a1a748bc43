"""Stack-kernel time (ms per 2^20 detections, config-2 workload, L=40) of the
library DETNET_LIB points at -- for A/B runs of kernel variants."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
path = int(sys.argv[2]) if len(sys.argv) > 2 else 0
K, N, L = 20, 30, 40
ctx = eng.Context(0, path=path)
m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131 + 5))
ctx.generate(base, 0, n, N, K, 10.0, 10.0, 1.0 / np.sqrt(N), H, y, x)
for _ in range(2):
    m.batch_evaluate_device(n, H, y, x)
ctx.kernel_times(reset=True)
ctx.set_profiling(True)
for _ in range(5):
    ev = m.batch_evaluate_device(n, H, y, x)
ctx.set_profiling(False)
kt = ctx.kernel_times(reset=True)
print(f"{os.environ.get('DETNET_LIB', 'default')}: {m.path_name} stack {kt['stack'][0] / kt['stack'][1]:.3f} ms "
      f"loss {ev.data_loss:.6f} errors {ev.symbol_errors}")
