#!/usr/bin/env python3
"""FP32 gradient noise of the engine's training paths against the FP64
reference, next to O32's (the FP32 restatement): prints the relative L2
error of batch_gradient for each forward / sweep combination (run the sweep
variants with DETNET_BWD_SIMT=1 / DETNET_DW_SIMT=1)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from oracle.oracle import Model, Oracle, RefLib
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    K, N, L, n = 20, 30, int(sys.argv[1]) if len(sys.argv) > 1 else 6, 2000
    orc, ref = Oracle(), RefLib()
    out = {}
    for scaled in (True, False):
        r = orc.rng(200, 0)
        H, x, y, _ = orc.generate_batch(r, N, K, n, 4.0, 12.0)
        s = 1 / np.sqrt(N) if scaled else 1.0
        H32, y32 = (H * s).astype(np.float32), (y * s).astype(np.float32)
        params = xavier_params(K, L, seed=5)
        om = Model(K, N, 8 * K, 2 * K, L, params, frozen_prefix=1)
        g64 = ref.batch_gradient(om, H32.astype(np.float64), y32.astype(np.float64), x, kind=2,
                                 lam1=0.04, lam2=0.04)["grads"]
        nrm = np.linalg.norm(g64)
        o32 = orc.batch_gradient_f32(om, H32.astype(np.float64), y32.astype(np.float64), x, kind=2,
                                     lam1=0.04, lam2=0.04)["grads"]
        row = {"o32": np.linalg.norm(o32 - g64) / nrm}
        for fwd in ("simt", "tc", "tc-tf32"):
            c = Context(0, path=2 if fwd == "tc-tf32" else 0)
            c.set_train_forward(fwd != "simt")
            m = c.model(K, N, 8 * K, 2 * K, params, frozen_prefix=1)
            _, g = m.batch_gradient(H32, y32, x.astype(np.int8), 2, 0.0, 0.04, 0.04)
            row[fwd] = np.linalg.norm(g - g64) / nrm
        out["scaled" if scaled else "unscaled"] = row
    print(json.dumps(out))


if __name__ == "__main__":
    main()
