#!/usr/bin/env python3
"""One pass over every kernel family through the C-ABI, printing a JSON
digest of the results: run with DETNET_LIB=build/debug/libdetnet_b200.so
(device-side bounds checks, -DDETNET_DEBUG_ASSERT) and with the product
library; tests/test_debug_build_gpu.py asserts both succeed with equal
digests. TEST INFRASTRUCTURE (uses the oracle's host generator)."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    import torch

    from oracle.oracle import Oracle
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import group_masks, sparse_group_model, xavier_params
    orc = Oracle()
    K, N, L, n = 20, 30, 6, 1000
    r = orc.rng(3, 0)
    H, x, y, _ = orc.generate_batch(r, N, K, n, 7.0, 14.0)
    H = (H / np.sqrt(N)).astype(np.float32)
    y = (y / np.sqrt(N)).astype(np.float32)
    x = x.astype(np.int8)
    params = xavier_params(K, L, seed=9)
    gm = group_masks(K, L, seed=31)
    sp, sm = sparse_group_model(params, gm, K)
    out = {}
    for path in (1, 2, 4, 3):
        c = Context(0, path=path)
        for name, (p, m) in (("dense", (params, None)), ("group", (params, gm)), ("sgl", (sp, sm))):
            if path == 3 and name != "sgl":
                continue
            ev, xh = c.model(K, N, 160, 40, p, masks=m).batch_evaluate(H, y, x, want_xhat=True)
            out[f"eval_p{path}_{name}"] = [ev.data_loss, ev.symbol_errors, digest(xh)]
    for fp64 in (False, True):
        c = Context(0)
        c.set_train_precision(fp64)
        m = c.model(K, N, 160, 40, params, masks=gm, frozen_prefix=1)
        ev, g = m.batch_gradient(H, y, x, 2, 0.0, 1e-4, 0.0)
        out[f"grad_fp64_{fp64}"] = [ev.data_loss, digest(g)]
        raw = m.new_raw()
        Hd, yd, xd = (torch.from_numpy(a).cuda() for a in (H, y, x))
        for _ in range(2):
            m.train_grad(n, Hd, yd, xd, raw)
            m.train_apply(raw, n, kind=2, lam1=1e-4, lr0=1e-3)
        out[f"train_fp64_{fp64}"] = [m.train_status()[0], digest(m.get_params())]
    g = Context(devices=[0, 0, 0])
    ev = g.model(K, N, 160, 40, params).batch_evaluate(np.tile(H, (20, 1, 1)), np.tile(y, (20, 1)),
                                                       np.tile(x, (20, 1)))
    out["group"] = [ev.data_loss, ev.symbol_errors]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
