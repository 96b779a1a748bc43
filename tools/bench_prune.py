"""SURVEY 8f row 3 measurement: sparse-group pruning of an L=40 DetNet
(1.03 M parameters) on the device master weights (detnet_model_prune, which
also rebuilds the packed layouts) vs the reference's prune on the host."""
import json
import os

# the in-process reference (OpenMP) must not spin its workers while the GPU
# side is timed on the same host cores (read when libgomp loads)
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2003_09446_b200 as eng  # noqa: E402
from oracle.oracle import Model as OModel, RefLib  # noqa: E402
from paper_2003_09446_b200.workload import xavier_params  # noqa: E402


def main():
    K, N, Z, V, L = 20, 30, 160, 40, 40
    p = xavier_params(K, L, seed=9)
    ctx, ref = eng.Context(0), RefLib()
    out = {}
    for eta1, eta2 in ((0.5, 0.3), (0.8, 0.2)):
        ts = []
        for _ in range(3):
            m = ctx.model(K, N, Z, V, p)
            t0 = time.perf_counter()
            m.prune(2, 0.0, eta1, eta2)
            ts.append(time.perf_counter() - t0)
            masks = m.get_masks()
        t0 = time.perf_counter()
        want = ref.prune(OModel(K, N, Z, V, L, p), 2, 0.0, eta1, eta2)
        tr = time.perf_counter() - t0
        rep, _ = m.cost_report()
        out[f"eta1={eta1},eta2={eta2}"] = {
            "b200_ms_incl_repack": 1e3 * min(ts), "reference_ms": 1e3 * tr,
            "masks_identical": bool(np.array_equal(masks, want)),
            "params_nonzero": rep["params_nonzero"], "flops": rep["flops"],
            "flops_dense": rep["flops_dense"], "compacted_tcgen05": m.path_name}
    print(json.dumps({"model": "L=40 K=20 z=160 v=40", **out}))


if __name__ == "__main__":
    main()
