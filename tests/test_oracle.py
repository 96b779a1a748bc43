"""Pin the C restatement (oracle/detnet_oracle.c) to the reference itself.

Every check is bit-exact: the restatement follows the reference loop orders
(linalg.cpp, model.cpp, loss.cpp, backward.cpp, adam.cpp, kernels.cpp) and
both are compiled with -ffp-contract=off. The reference side is the
unmodified library compiled from /root/reference/proj/src (oracle/_ref).
"""
import numpy as np
import pytest

from oracle.oracle import Model, record_size, record_slices, xavier_model


def _gauss_model(oracle, K, N, L, seed, Z=None, V=None, t0=0.5, scale=1.0):
    """init_params-style model (model.cpp:140-159 draw order) from the oracle Rng."""
    import ctypes as C
    Z = Z or 8 * K
    V = V or 2 * K
    IN = 3 * K + V
    P = record_size(K, Z, V)
    sl = record_slices(K, Z, V)
    r = oracle.rng(seed, 0)
    params = np.zeros((L, P))
    for l in range(L):
        for name, (rows, cols) in (("W1", (Z, IN)), ("W2", (K, Z)), ("W3", (V, Z))):
            std = scale / np.sqrt(cols)
            params[l, sl[name]] = [std * oracle.lib.or_next_gaussian(C.byref(r))
                                   for _ in range(rows * cols)]
        params[l, sl["t"]] = t0
    return Model(K, N, Z, V, L, params)


def _masks(m, seed, p_zero=0.3):
    rng = np.random.default_rng(seed)
    masks = (rng.random(m.params.shape) > p_zero).astype(np.float64)
    sl = record_slices(m.n_tx, m.z_dim, m.v_dim)
    masks[:, sl["t"]] = 1.0
    return masks


def test_rng_draws_bit_exact(oracle, ref):
    for kind in ("u64", "uniform", "gaussian"):
        a = oracle.draws(123, 7, 500, kind)
        b = ref.draws(123, 7, 500, kind)
        assert a == b, kind


def test_rng_random_access_formula(oracle):
    """Draw d of a stream equals mix64(s0 + (d+1) * gamma)."""
    r = oracle.rng(5, 3)
    s0 = r.s
    draws = oracle.draws(5, 3, 64)
    g = 0x9e3779b97f4a7c15
    for d, v in enumerate(draws):
        assert v == oracle.lib.or_mix64((s0 + (d + 1) * g) % 2**64)


@pytest.mark.parametrize("snr", [(7.0, 14.0), (10.0, 10.0)])
def test_generate_batch_bit_exact(oracle, ref, snr):
    rr = ref.lib.ref_rng_new(2, 0)
    Hr, xr, yr, sr = ref.generate_batch(rr, 30, 20, 37, *snr)
    Hr2, *_ = ref.generate_batch(rr, 30, 20, 5, *snr)  # second call: rng advanced by one
    ref.lib.ref_rng_free(rr)
    ro = oracle.rng(2, 0)
    Ho, xo, yo, so = oracle.generate_batch(ro, 30, 20, 37, *snr)
    Ho2, *_ = oracle.generate_batch(ro, 30, 20, 5, *snr)
    assert np.array_equal(Hr, Ho) and np.array_equal(xr, xo) and np.array_equal(yr, yo)
    assert np.array_equal(sr, so) and np.array_equal(Hr2, Ho2)


def test_forward_trace_bit_exact(oracle, ref):
    m = _gauss_model(oracle, 4, 8, 5, seed=10)
    r = oracle.rng(11, 0)
    H, x, y, _ = oracle.generate_batch(r, 8, 4, 6, 0.0, 15.0)
    for s in range(6):
        tr = ref.forward(m, H[s], y[s])
        ev = oracle.evaluate(m, H[s:s + 1], y[s:s + 1], x[s:s + 1], want_xhat=True)
        assert np.array_equal(ev["xhat"][0], tr["x_hat"][1:])
        st, q, G, xt = oracle.preprocess(H[s], y[s])
        assert st == 0
        assert np.array_equal(xt, ref.zf_decode(H[s], y[s]))
        # single-layer restatement on the reference trajectory
        for l in range(m.depth):
            xo, vo, aux = oracle.layer(m, l, q, G, tr["x_hat"][l], tr["v"][l])
            assert np.array_equal(xo, tr["x_hat"][l + 1]) and np.array_equal(vo, tr["v"][l + 1])
            assert np.array_equal(aux["u1"], tr["u1"][l]) and np.array_equal(aux["u2"], tr["u2"][l])


@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("trainable_only,frozen", [(False, 0), (True, 2)])
def test_batch_evaluate_bit_exact(oracle, ref, masked, trainable_only, frozen):
    m = xavier_model(oracle, n_tx=6, n_rx=9, depth=5, seed=3)
    m.frozen_prefix = frozen
    if masked:
        m.masks = _masks(m, 1)
    r = oracle.rng(4, 0)
    H, x, y, _ = oracle.generate_batch(r, 9, 6, 57, 4.0, 12.0)
    a = oracle.batch_evaluate(m, H, y, x, trainable_only)
    for parallel in (False, True):
        b = ref.batch_evaluate(m, H, y, x, trainable_only, parallel=parallel)
        assert a == b


@pytest.mark.parametrize("kind,lam,lam1,lam2", [(0, 0, 0, 0), (1, 0.03, 0, 0), (2, 0, 0.04, 0.04),
                                                (2, 0, 1e-4, 0.0)])
@pytest.mark.parametrize("masked,frozen", [(False, 0), (True, 1)])
def test_batch_gradient_bit_exact(oracle, ref, kind, lam, lam1, lam2, masked, frozen):
    m = _gauss_model(oracle, 3, 5, 4, seed=100)
    m.frozen_prefix = frozen
    if masked:
        m.masks = _masks(m, 2)
    r = oracle.rng(200, 0)
    H, x, y, _ = oracle.generate_batch(r, 5, 3, 157, 4.0, 12.0)
    a = oracle.batch_gradient(m, H, y, x, kind, lam, lam1, lam2)
    b = ref.batch_gradient(m, H, y, x, kind, lam, lam1, lam2, parallel=True)
    c = ref.batch_gradient(m, H, y, x, kind, lam, lam1, lam2, parallel=False)
    assert np.array_equal(a["grads"], b["grads"]) and np.array_equal(b["grads"], c["grads"])
    assert a["data_loss"] == b["data_loss"] and a["symbol_errors"] == b["symbol_errors"]
    assert oracle.regularizer(m, kind, lam, lam1, lam2) == ref.regularizer(m, kind, lam, lam1, lam2)


def test_adam_bit_exact(oracle, ref):
    m = _gauss_model(oracle, 3, 5, 3, seed=7)
    m.masks = _masks(m, 3)
    m.frozen_prefix = 1
    r = oracle.rng(8, 0)
    H, x, y, _ = oracle.generate_batch(r, 5, 3, 40, 0.0, 15.0)
    g = oracle.batch_gradient(m, H, y, x, 2, 0, 0.01, 0.01)["grads"]
    import dataclasses
    m1, m2 = m, dataclasses.replace(m, params=m.params.copy())
    mo1 = np.zeros_like(m.params); vo1 = np.zeros_like(m.params)
    mo2 = np.zeros_like(m.params); vo2 = np.zeros_like(m.params)
    s1 = s2 = 999
    for _ in range(3):
        s1 = oracle.adam_step(m1, g, mo1, vo1, s1, lr0=1e-3, decay_step=1000)
        s2 = ref.adam_step(m2, g, mo2, vo2, s2, lr0=1e-3, decay_step=1000)
    assert s1 == s2 == 1002
    assert np.array_equal(m1.params, m2.params)
    assert np.array_equal(mo1, mo2) and np.array_equal(vo1, vo2)


def test_flops_census(oracle, ref):
    """compression.cpp:120-129; literals from test_compression.cpp:235-258."""
    m = xavier_model(oracle, n_tx=20, n_rx=30, depth=2, seed=1)
    m90 = Model(20, 30, 160, 40, 90, np.repeat(m.params[:1], 90, axis=0))
    assert oracle.flops_per_detection(m90) == 4_705_200 == ref.flops_per_detection(m90)
    m40 = Model(20, 30, 160, 40, 40, np.repeat(m.params[:1], 40, axis=0))
    assert oracle.flops_per_detection(m40) == 2_105_200
    mm = xavier_model(oracle, n_tx=4, n_rx=8, depth=3, seed=2)
    mm.masks = _masks(mm, 5)
    assert oracle.flops_per_detection(mm) == ref.flops_per_detection(mm)


def test_loss_literals(oracle):
    """L=1 -> loss exactly 0 (log 1 = 0, acceptance.cpp:326-339)."""
    m = xavier_model(oracle, n_tx=4, n_rx=8, depth=1, seed=2)
    r = oracle.rng(1, 0)
    H, x, y, _ = oracle.generate_batch(r, 8, 4, 20, 0.0, 15.0)
    ev = oracle.evaluate(m, H, y, x)
    assert np.all(ev["loss"] == 0.0)


def test_f32_restatement_close(oracle):
    m = xavier_model(oracle, n_tx=20, n_rx=30, depth=10, seed=9)
    r = oracle.rng(2, 0)
    H, x, y, _ = oracle.generate_batch(r, 30, 20, 16, 7.0, 14.0)
    H = (H / np.sqrt(30)).astype(np.float32).astype(np.float64)
    y = (y / np.sqrt(30)).astype(np.float32).astype(np.float64)
    a = oracle.evaluate(m, H, y, x, want_xhat=True)
    b = oracle.evaluate_f32(m, H, y, x)
    assert np.max(np.abs(a["xhat"] - b["xhat"])) < 1e-3


def test_o32_batch_gradient_tracks_reference(oracle, ref):
    """O32 (the FP32 restatement used to calibrate FP32's own training
    spread) stays within FP32 noise of the reference's FP64 batch_gradient."""
    from oracle.oracle import scaled_inputs
    m = xavier_model(oracle, depth=4, seed=5)
    r = oracle.rng(2, 0)
    H, x, y, _ = oracle.generate_batch(r, 30, 20, 300, 7.0, 14.0)
    H32, y32, _ = scaled_inputs(H, y, x)
    H64, y64 = H32.astype(np.float64), y32.astype(np.float64)
    a = ref.batch_gradient(m, H64, y64, x, kind=2, lam1=1e-4)
    b = oracle.batch_gradient_f32(m, H64, y64, x, kind=2, lam1=1e-4)
    assert b["status"] == 0
    assert np.abs(a["grads"] - b["grads"]).max() <= 1e-5 * np.abs(a["grads"]).max()
    assert abs(a["data_loss"] - b["data_loss"]) <= 1e-6 * a["data_loss"]
    assert b["symbol_errors"] == a["symbol_errors"] and b["flagged"] == a["flagged"]
