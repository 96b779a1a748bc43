"""Profiling driver: one detnet_batch_evaluate_device over n samples of the
config-2 workload (L=40; argv[3] = 3: config-3 group masks) after a warm-up
call. Used under ncu. argv: n [path [config]]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
path = int(sys.argv[2]) if len(sys.argv) > 2 else 0
config = int(sys.argv[3]) if len(sys.argv) > 3 else 2
K, N, L = 20, 30, 40
if config == 4 and path == 0:
    path = 3  # the sparse-group model's kernel (model-specialised, opt-in path)
ctx = eng.Context(0, path=path)
params = xavier_params(K, L, seed=9)
masks = None
if config in (3, 4):  # group-pruned (compacted tcgen05 kernel) / sparse group (JIT kernel)
    from paper_2003_09446_b200.workload import group_masks, sparse_group_model
    masks = group_masks(K, L, seed=31)
    if config == 4:
        params, masks = sparse_group_model(params, masks, K)
m = ctx.model(K, N, 160, 40, params, masks=masks)
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131 + 5))
ctx.generate(base, 0, n, N, K, 10.0, 10.0, 1.0 / np.sqrt(N), H, y, x)
import time
for _ in range(2):
    ev = m.batch_evaluate_device(n, H, y, x)
print(m.path_name, ev)
if os.environ.get("PROF_TIME"):  # per-kernel event times over a few calls
    ctx.set_profiling(True)
    ctx.kernel_times(reset=True)
    for _ in range(5):
        ev = m.batch_evaluate_device(n, H, y, x)
    kt = ctx.kernel_times(reset=True)
    print("kernel ms per call:", {k: round(v[0] / 5, 4) for k, v in kt.items() if v[1]})
