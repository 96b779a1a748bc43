"""Seeded synthetic workloads of BASELINE.json / SURVEY 8d, built without the
oracle (product side).

* Xavier-uniform weights drawn with the reference Rng (rng.cpp:12-46) as
  U(-a, a) = -a + 2a * next_uniform(), a = sqrt(6 / (fan_in + fan_out)),
  layer by layer in W1, W2, W3 order, rounded to FP32; zero biases; t = 0.5.
  The splitmix64 stream is random access (draw d = mix64(s0 + (d+1) gamma)),
  so the draws are vectorised with numpy uint64 arithmetic.
* Masks for the group-pruned (config 3) and sparse-group (config 4) models.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9e3779b97f4a7c15)
_M1 = np.uint64(0xbf58476d1ce4e5b9)
_M2 = np.uint64(0x94d049bb133111eb)


def mix64(z):
    z = np.asarray(z, np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def rng_state(seed, stream_id=0):
    """Rng(seed, stream_id) state (rng.cpp:18-19)."""
    with np.errstate(over="ignore"):
        return np.uint64(mix64(mix64(np.uint64(seed) ^ np.uint64(0x853c49e6748fea9b))
                               + np.uint64(stream_id)))


def uniform_draws(state, first, count):
    """next_uniform() draws [first, first+count) of a stream with state `state`."""
    d = np.arange(first + 1, first + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = mix64(np.uint64(state) + d * GAMMA)
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def record_layout(K, Z, V):
    IN = 3 * K + V
    out, off = {}, 0
    for name, size in (("W1", Z * IN), ("b1", Z), ("W2", K * Z), ("b2", K), ("W3", V * Z),
                       ("b3", V), ("t", 1)):
        out[name] = slice(off, off + size)
        off += size
    return out, off


def xavier_params(n_tx=20, depth=40, seed=9, z_dim=None, v_dim=None, t0=0.5):
    """[depth, P] float64 layer records with FP32-representable values."""
    K = n_tx
    Z = z_dim or 8 * K
    V = v_dim or 2 * K
    IN = 3 * K + V
    sl, P = record_layout(K, Z, V)
    st = rng_state(seed, 0)
    params = np.zeros((depth, P))
    d = 0
    for l in range(depth):
        for name, (rows, cols) in (("W1", (Z, IN)), ("W2", (K, Z)), ("W3", (V, Z))):
            a = (6.0 / (rows + cols)) ** 0.5
            u = uniform_draws(st, d, rows * cols)
            d += rows * cols
            params[l, sl[name]] = -a + (a - -a) * u
        params[l, sl["t"]] = t0
    return params.astype(np.float32).astype(np.float64)


def group_masks(n_tx=20, depth=40, seed=31, dead_units=112, dead_cols=30, z_dim=None, v_dim=None):
    """Config 3 masks: per layer a seeded Fisher-Yates choice of
    `dead_units` hidden units (W1 row, mb1, W2/W3 column zeroed) and
    `dead_cols` W1 input columns."""
    K = n_tx
    Z = z_dim or 8 * K
    V = v_dim or 2 * K
    IN = 3 * K + V
    sl, P = record_layout(K, Z, V)
    rs = np.random.default_rng(seed)
    masks = np.ones((depth, P))
    for l in range(depth):
        units = rs.permutation(Z)[:dead_units]
        cols = rs.permutation(IN)[:dead_cols]
        M1 = np.ones((Z, IN)); mb1 = np.ones(Z); M2 = np.ones((K, Z)); M3 = np.ones((V, Z))
        M1[units, :] = 0.0
        mb1[units] = 0.0
        M2[:, units] = 0.0
        M3[:, units] = 0.0
        M1[:, cols] = 0.0
        masks[l, sl["W1"]] = M1.ravel()
        masks[l, sl["b1"]] = mb1
        masks[l, sl["W2"]] = M2.ravel()
        masks[l, sl["W3"]] = M3.ravel()
    return masks


def sparse_group_model(params, masks, n_tx=20, seed=47, keep=0.05, std=0.05, z_dim=None,
                       v_dim=None):
    """Config 4: inside the surviving groups keep each weight with
    Bernoulli(keep); surviving values N(0, std^2) (BASELINE 'N(0,0.05)' read
    as std 0.05), rounded to FP32. Returns (params, masks)."""
    K = n_tx
    Z = z_dim or 8 * K
    V = v_dim or 2 * K
    sl, P = record_layout(K, Z, V)
    rs = np.random.default_rng(seed)
    p = params.copy()
    mk = masks.copy()
    for l in range(p.shape[0]):
        for name in ("W1", "W2", "W3"):
            keepm = (rs.random(sl[name].stop - sl[name].start) < keep).astype(np.float64)
            mk[l, sl[name]] *= keepm
            vals = rs.normal(0.0, std, sl[name].stop - sl[name].start)
            p[l, sl[name]] = np.where(mk[l, sl[name]] != 0, vals, 0.0)
    return p.astype(np.float32).astype(np.float64), mk
