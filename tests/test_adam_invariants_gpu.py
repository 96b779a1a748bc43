"""The reference's own Adam / update invariants (proj/tests/test_adam.cpp) on the
device Adam (`detnet_adam_step`, the seam's `adam_step`) and on the
device-resident training step (`detnet_train_grad` + `detnet_train_apply`):

* zero gradient leaves parameters unchanged            (test_adam.cpp:27-41)
* the first step moves by ~lr against the gradient sign (test_adam.cpp:43-54)
* t never drops below its clamp 1e-3                     (test_adam.cpp:56-66)
* frozen layers are bit-frozen under updates             (test_adam.cpp:68-85)
* masked weights never move, even with stale moments     (test_adam.cpp:87-111)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
K, N = 4, 8
Z, V = 8 * K, 2 * K


@pytest.fixture(scope="module")
def ctx():
    from paper_2003_09446_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _params(L, seed=5):
    from paper_2003_09446_b200.workload import xavier_params
    return xavier_params(K, L, seed=seed)


def _t_index():
    from paper_2003_09446_b200 import record_size
    return record_size(K, Z, V) - 1  # the record ends with t (grad_check.hpp:16-44 order)


def _step(ctx, L, frozen, p, masks, g, m1, m2, step, **kw):
    return ctx.adam_step(K, Z, V, L, frozen, p, masks, g, m1, m2, step, **kw)


def test_zero_gradient_leaves_parameters_unchanged(ctx):
    L = 3
    p0 = _params(L)
    p, m1, m2 = p0.copy(), np.zeros_like(p0), np.zeros_like(p0)
    g = np.zeros_like(p0)
    s = 0
    for _ in range(3):
        s = _step(ctx, L, 0, p, np.ones_like(p0), g, m1, m2, s, lr0=1e-2)
    assert s == 3
    assert np.array_equal(p, p0)
    assert not m1.any() and not m2.any()


def test_first_step_moves_by_lr_against_gradient_sign(ctx):
    L = 2
    p0 = _params(L)
    rs = np.random.default_rng(3)
    g = rs.standard_normal(p0.shape)
    g[np.abs(g) < 1e-3] = 1e-3
    p, m1, m2 = p0.copy(), np.zeros_like(p0), np.zeros_like(p0)
    lr = 1e-3
    _step(ctx, L, 0, p, np.ones_like(p0), g, m1, m2, 0, lr0=lr)
    d = p - p0
    ti = _t_index()
    body = np.ones(p0.shape, bool)
    body[:, ti] = False  # t is clamped separately
    # bias-corrected first step: m_hat / (sqrt(v_hat) + eps) = sign(g) up to eps
    assert np.allclose(d[body], -lr * np.sign(g[body]), rtol=1e-4, atol=0.0)


def test_t_never_drops_below_its_clamp(ctx):
    L = 1
    p = _params(L)
    ti = _t_index()
    p[0, ti] = 0.0011
    g = np.zeros_like(p)
    g[0, ti] = 1e6  # push t hard toward zero
    m1, m2 = np.zeros_like(p), np.zeros_like(p)
    s = 0
    for _ in range(5):
        s = _step(ctx, L, 0, p, np.ones_like(p), g, m1, m2, s, lr0=0.1)
    assert p[0, ti] >= 1e-3


def test_frozen_layers_are_bit_frozen_and_masked_weights_never_move(ctx):
    L, frozen = 4, 2
    p0 = _params(L)
    rs = np.random.default_rng(7)
    masks = (rs.random(p0.shape) > 0.4).astype(np.float64)
    masks[:, _t_index()] = 1.0
    p0 = p0 * masks
    g = rs.standard_normal(p0.shape)
    # stale moments everywhere, masked and frozen entries included (test_adam.cpp:87-111)
    m1 = rs.standard_normal(p0.shape) * 0.1
    m2 = rs.random(p0.shape) * 0.1
    m1_0, m2_0 = m1.copy(), m2.copy()
    p = p0.copy()
    s = 10
    for _ in range(4):
        s = _step(ctx, L, frozen, p, masks, g, m1, m2, s, lr0=1e-2)
    assert np.array_equal(p[:frozen], p0[:frozen])  # bit-frozen
    assert np.array_equal(m1[:frozen], m1_0[:frozen]) and np.array_equal(m2[:frozen], m2_0[:frozen])
    dead = masks[frozen:] == 0.0
    assert np.array_equal(p[frozen:][dead], p0[frozen:][dead])
    assert not p[frozen:][dead].any()
    live = ~dead
    assert (p[frozen:][live] != p0[frozen:][live]).mean() > 0.99


def test_device_training_steps_keep_frozen_and_masked_entries(ctx, oracle):
    """The same two invariants through detnet_train_grad + detnet_train_apply
    (device-resident parameters, masks and moments)."""
    import torch
    L, frozen, n = 4, 2, 600
    p0 = _params(L, seed=11)
    rs = np.random.default_rng(9)
    masks = (rs.random(p0.shape) > 0.3).astype(np.float64)
    masks[:, _t_index()] = 1.0
    r = oracle.rng(3, 0)
    Hd, xd, yd, _ = oracle.generate_batch(r, N, K, n, 7.0, 14.0)
    H = torch.tensor((Hd / np.sqrt(N)).astype(np.float32), device="cuda")
    y = torch.tensor((yd / np.sqrt(N)).astype(np.float32), device="cuda")
    x = torch.tensor(xd.astype(np.int8), device="cuda")
    model = ctx.model(K, N, Z, V, p0, masks=masks, frozen_prefix=frozen)
    raw = model.new_raw()
    for _ in range(3):
        model.train_grad(n, H, y, x, raw, trainable_only=True)
        model.train_apply(raw, n, kind=2, lam1=1e-3, lam2=1e-4, lr0=1e-2)
    p = model.get_params()
    assert np.array_equal(p[:frozen], p0[:frozen])
    dead = masks[frozen:] == 0.0
    assert np.array_equal(p[frozen:][dead], p0[frozen:][dead])
    assert (p[frozen:][~dead] != p0[frozen:][~dead]).mean() > 0.9
    assert (p[:, _t_index()] >= 1e-3).all()
    model.close()
