"""The C restatement against golden vectors produced by the reference itself
(tools/make_golden.py). Runs without /root/reference (e.g. on the GPU box)."""
import os

import numpy as np

from oracle.oracle import Model

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name))


def test_golden_rng(oracle):
    g = _load("rng.npz")
    assert np.array_equal(np.array(oracle.draws(123, 7, 64, "u64"), np.uint64), g["u64"])
    assert np.array_equal(np.array(oracle.draws(123, 7, 64, "gaussian")), g["gauss"])
    assert np.array_equal(np.array(oracle.draws(9, 0, 64, "uniform")), g["uniform"])


def test_golden_generate_batch(oracle):
    g = _load("generate_batch.npz")
    r = oracle.rng(2, 0)
    H, x, y, s2 = oracle.generate_batch(r, 30, 20, 8, 7.0, 14.0)
    assert np.array_equal(H, g["H"]) and np.array_equal(x, g["x"]) and np.array_equal(y, g["y"])
    assert np.array_equal(s2, g["sigma2"])
    H, x, y, s2 = oracle.generate_batch(r, 30, 20, 4, 10.0, 10.0)
    assert np.array_equal(H, g["H_fixed"]) and np.array_equal(y, g["y_fixed"])


def test_golden_forward(oracle):
    g = _load("forward_k20.npz")
    m = Model(20, 30, 160, 40, 4, g["params"].astype(np.float64))
    H, y, x = (g[k].astype(np.float64) for k in ("H", "y", "x"))
    ev = oracle.evaluate(m, H, y, x, want_xhat=True)
    assert np.array_equal(ev["xhat"], g["x_hat"][:, 1:])
    be = oracle.batch_evaluate(m, H, y, x)
    assert be["data_loss"] == float(g["data_loss"])
    assert be["symbol_errors"] == int(g["symbol_errors"]) and be["flagged"] == int(g["flagged"])


def test_golden_gradient_and_adam(oracle):
    g = _load("gradient_k3.npz")
    m = Model(3, 5, 24, 6, 4, g["params"].copy(), masks=g["masks"], frozen_prefix=1)
    gr = oracle.batch_gradient(m, g["H"], g["y"], g["x"], kind=2, lam1=0.04, lam2=0.04)
    assert np.array_equal(gr["grads"], g["grads"])
    assert gr["data_loss"] == float(g["data_loss"])
    mo = np.zeros_like(m.params); vo = np.zeros_like(m.params)
    step = oracle.adam_step(m, gr["grads"], mo, vo, 0, lr0=1e-3)
    step = oracle.adam_step(m, gr["grads"], mo, vo, step, lr0=1e-3)
    assert step == int(g["adam_step"])
    assert np.array_equal(m.params, g["adam_params"])
    assert np.array_equal(mo, g["adam_m"]) and np.array_equal(vo, g["adam_v"])
