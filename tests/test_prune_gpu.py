"""the pruning planner on device-resident weights
(detnet_model_prune) against the reference's prune (compression.cpp:43-94):
masks bit-identical, cost_report identical, and the pruned model -- repacked
into the compacted tcgen05 / SIMT layouts -- evaluating like the oracle."""
import numpy as np
import pytest

from oracle.oracle import Model as OModel

pytestmark = pytest.mark.gpu
K, N, Z, V = 20, 30, 160, 40


@pytest.fixture(scope="module")
def ctx():
    import paper_2003_09446_b200 as eng
    return eng.Context(0)


def _trained_like(L, seed):
    """Xavier weights with a spread of column norms (a few columns/units
    scaled down), so every pruning rule has work to do."""
    from paper_2003_09446_b200.workload import xavier_params, record_layout
    p = xavier_params(K, L, seed=seed)
    sl, P = record_layout(K, Z, V)
    rs = np.random.default_rng(seed)
    for l in range(L):
        W1 = p[l, sl["W1"]].reshape(Z, 3 * K + V)
        W1 *= rs.uniform(0.05, 1.0, size=(1, 3 * K + V))
        W2 = p[l, sl["W2"]].reshape(K, Z)
        W3 = p[l, sl["W3"]].reshape(V, Z)
        sc = np.where(rs.random(Z) < 0.6, 0.02, 1.0)
        W2 *= sc
        W3 *= sc
        p[l, sl["W1"]] = W1.ravel(); p[l, sl["W2"]] = W2.ravel(); p[l, sl["W3"]] = W3.ravel()
        p[l, sl["b1"]] = rs.normal(0, 0.01, Z)
        p[l, sl["b2"]] = rs.normal(0, 0.01, K)
    return p


@pytest.mark.parametrize("kind,eta,eta1,eta2", [(0, 0.3, 0.0, 0.0), (1, 0.0, 0.2, 0.0),
                                                (2, 0.0, 0.2, 0.25), (1, 0.0, 0.0, 0.0)])
def test_prune_masks_bit_identical(ctx, ref, kind, eta, eta1, eta2):
    L = 6
    p = _trained_like(L, 7)
    m = ctx.model(K, N, Z, V, p)
    m.prune(kind, eta, eta1, eta2)
    got = m.get_masks()
    want = ref.prune(OModel(K, N, Z, V, L, p), kind, eta, eta1, eta2)
    assert np.array_equal(got, want)
    rep, per = m.cost_report()
    rref, pref = ref.cost_report(OModel(K, N, Z, V, L, p, masks=want))
    assert rep == rref
    assert np.array_equal(per, pref)
    assert m.flops_per_detection() == rref["flops"]


def test_pruned_model_evaluates_like_oracle(ctx, oracle, ref):
    """Group pruning of the designated units compacts the tcgen05 images to
    the live units; the evaluation must match the oracle on the pruned masks."""
    L = 8
    p = _trained_like(L, 9)
    m = ctx.model(K, N, Z, V, p)
    m.prune(2, 0.0, 0.25, 0.1)
    masks = m.get_masks()
    r = oracle.rng(5, 0)
    H, x, y, _ = oracle.generate_batch(r, N, K, 1024, 7.0, 14.0)
    H32 = (H / np.sqrt(N)).astype(np.float32)
    y32 = (y / np.sqrt(N)).astype(np.float32)
    ev, xh = m.batch_evaluate(H32, y32, x.astype(np.int8), want_xhat=True)
    want = oracle.evaluate(OModel(K, N, Z, V, L, p, masks=masks), H32.astype(np.float64),
                           y32.astype(np.float64), x, want_xhat=True)
    err = np.abs(xh - want["xhat"])
    assert np.mean(err < 1e-4 + 1e-4 * np.abs(want["xhat"])) > 0.999, err.max()
    assert abs(ev.data_loss - want["loss"].mean()) <= 1e-4 * abs(want["loss"].mean())


def test_prune_keeps_training_state(ctx, oracle):
    """Pruning between training steps keeps Adam moments and step count; the
    pruned entries stay frozen at their values (masked Adam skip)."""
    L = 4
    p = _trained_like(L, 3)
    m = ctx.model(K, N, Z, V, p)
    r = oracle.rng(6, 0)
    H, x, y, _ = oracle.generate_batch(r, N, K, 512, 7.0, 14.0)
    H32 = (H / np.sqrt(N)).astype(np.float32); y32 = (y / np.sqrt(N)).astype(np.float32)
    import torch
    raw = m.new_raw()
    Hd, yd, xd = (torch.from_numpy(a).cuda() for a in (H32, y32, x.astype(np.int8)))
    m.train_grad(512, Hd, yd, xd, raw)
    m.train_apply(raw, 512, lr0=1e-3)
    m.prune(1, eta1=0.2)
    before = m.get_params()
    mk = m.get_masks()
    m.train_grad(512, Hd, yd, xd, raw)
    m.train_apply(raw, 512, lr0=1e-3)
    after = m.get_params()
    frozen = mk == 0
    assert np.array_equal(after[frozen], before[frozen])
    assert not np.array_equal(after[~frozen], before[~frozen])


def test_prune_rejects_bad_thresholds(ctx):
    import paper_2003_09446_b200 as eng
    m = ctx.model(K, N, Z, V, _trained_like(2, 1))
    with pytest.raises(eng.ConfigError):
        m.prune(0, eta=1.0)
