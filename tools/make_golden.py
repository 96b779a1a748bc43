"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle` has built
oracle/_ref/libunfold_ref.so):  python tools/make_golden.py
The fixtures pin the C restatement and the GPU path on machines without the
reference (e.g. the GPU box). Every array is produced by the reference's own
public API (Rng, generate_batch, forward, batch_evaluate, batch_gradient,
adam_step); the workload builders only fill ModelParams fields.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Model, Oracle, RefLib, record_size, record_slices, xavier_model  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def gauss_model(ref, K, N, L, seed):
    """init_params(Rng(seed), K, N, L) draw order (model.cpp:140-159)."""
    Z, V = 8 * K, 2 * K
    IN = 3 * K + V
    sl = record_slices(K, Z, V)
    r = ref.lib.ref_rng_new(seed, 0)
    params = np.zeros((L, record_size(K, Z, V)))
    for l in range(L):
        for name, (rows, cols) in (("W1", (Z, IN)), ("W2", (K, Z)), ("W3", (V, Z))):
            std = 1.0 / np.sqrt(cols)
            params[l, sl[name]] = [std * ref.lib.ref_rng_next_gaussian(r) for _ in range(rows * cols)]
        params[l, sl["t"]] = 0.5
    ref.lib.ref_rng_free(r)
    return Model(K, N, Z, V, L, params)


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = RefLib()
    orc = Oracle()

    # 1. rng streams
    np.savez_compressed(os.path.join(OUT, "rng.npz"),
                        u64=np.array(ref.draws(123, 7, 64, "u64"), np.uint64),
                        gauss=np.array(ref.draws(123, 7, 64, "gaussian")),
                        uniform=np.array(ref.draws(9, 0, 64, "uniform")))

    # 2. generate_batch, ranged and fixed SNR (K=20, N=30)
    r = ref.lib.ref_rng_new(2, 0)
    H, x, y, s2 = ref.generate_batch(r, 30, 20, 8, 7.0, 14.0)
    H2, x2, y2, s22 = ref.generate_batch(r, 30, 20, 4, 10.0, 10.0)
    ref.lib.ref_rng_free(r)
    np.savez_compressed(os.path.join(OUT, "generate_batch.npz"), H=H, x=x, y=y, sigma2=s2,
                        H_fixed=H2, x_fixed=x2, y_fixed=y2, sigma2_fixed=s22)

    # 3. dense forward at the config shape (K=20, N=30), L=4, scaled FP32 inputs
    m = xavier_model(orc, n_tx=20, n_rx=30, depth=4, seed=9)
    Hs = (H / np.sqrt(30)).astype(np.float32).astype(np.float64)
    ys = (y / np.sqrt(30)).astype(np.float32).astype(np.float64)
    xh = np.stack([ref.forward(m, Hs[s], ys[s])["x_hat"] for s in range(8)])
    vv = np.stack([ref.forward(m, Hs[s], ys[s])["v"] for s in range(8)])
    ev = ref.batch_evaluate(m, Hs, ys, x)
    np.savez_compressed(os.path.join(OUT, "forward_k20.npz"), params=m.params.astype(np.float32),
                        H=Hs.astype(np.float32), y=ys.astype(np.float32), x=x.astype(np.int8),
                        x_hat=xh, v=vv, data_loss=ev["data_loss"],
                        symbol_errors=ev["symbol_errors"], flagged=ev["flagged"])

    # 4. masked + frozen gradient (K=3, N=5, L=4), SGL loss, then two Adam steps
    gm = gauss_model(ref, 3, 5, 4, seed=100)
    rs = np.random.default_rng(2)
    masks = (rs.random(gm.params.shape) > 0.3).astype(np.float64)
    masks[:, record_slices(3, 24, 6)["t"]] = 1.0
    gm.masks = masks
    gm.frozen_prefix = 1
    r = ref.lib.ref_rng_new(200, 0)
    Hg, xg, yg, _ = ref.generate_batch(r, 5, 3, 157, 4.0, 12.0)
    ref.lib.ref_rng_free(r)
    gr = ref.batch_gradient(gm, Hg, yg, xg, kind=2, lam1=0.04, lam2=0.04)
    p0 = gm.params.copy()
    mo = np.zeros_like(gm.params); vo = np.zeros_like(gm.params)
    step = ref.adam_step(gm, gr["grads"], mo, vo, 0, lr0=1e-3)
    step = ref.adam_step(gm, gr["grads"], mo, vo, step, lr0=1e-3)
    np.savez_compressed(os.path.join(OUT, "gradient_k3.npz"), params=p0, masks=masks,
                        H=Hg, x=xg, y=yg, grads=gr["grads"], data_loss=gr["data_loss"],
                        symbol_errors=gr["symbol_errors"], flagged=gr["flagged"],
                        adam_params=gm.params, adam_m=mo, adam_v=vo, adam_step=step)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
