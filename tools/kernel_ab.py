"""A/B timing of kernel variants: per-launch event times of the engine's
kernels (ctx.kernel_times) over repeated config-2 (or config-3) evaluations
of n samples at 10 dB. Select the library with DETNET_LIB. argv: n [config] [reps]."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
config = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
K, N = 20, 30
L = 90 if config == 1 else 40
ctx = eng.Context(0)
params = xavier_params(K, L, seed=9)
masks = None
if config in (3, 4):
    from paper_2003_09446_b200 import workload as wl
    masks = wl.group_masks(K, L, seed=31)
    if config == 4:
        params, masks = wl.sparse_group_model(params, masks, K)
m = ctx.model(K, N, 160, 40, params, masks=masks)
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131 + 5))
ctx.generate(base, 0, n, N, K, 10.0, 10.0, 1.0 / np.sqrt(N), H, y, x)
for _ in range(3):
    ev = m.batch_evaluate_device(n, H, y, x)
torch.cuda.synchronize()
ctx.set_profiling(True)
ctx.kernel_times(reset=True)
for _ in range(reps):
    ev = m.batch_evaluate_device(n, H, y, x)
torch.cuda.synchronize()
kt = ctx.kernel_times(reset=True)
print(json.dumps({"lib": os.environ.get("DETNET_LIB", "default"), "n": n, "config": config,
                  "path": m.path_name, "ms_per_call": {k: v[0] / reps for k, v in kt.items() if v[1]},
                  "errors": ev.symbol_errors, "loss": ev.data_loss}))
