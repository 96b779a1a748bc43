"""K1 parity (linalg.cpp:20-79, loss.cpp:14-19) through the preprocessing hook
detnet_preprocess_device: G = H^T H and q = H^T y against the oracle's FP64
values of the same FP32 inputs (FP32 accumulation: 1e-6 of max|G|), and the
loss denominator ||x - x_tilde||^2 of the fast FP32 Cholesky path within 1e-4
relative of the reference LU (measured: median 6e-7, max 4e-5 over 2^16
samples at 0-30 dB, tools/denom_check.py); the exact mode is the reference's
FP64 LU itself. Covers multi-tile persistent CTAs (run-to-run determinism),
high-SNR samples that take the exact fallback, and the noise-free guard."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
K, N = 20, 30


@pytest.fixture(scope="module")
def model():
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    ctx = Context(0)
    return ctx, ctx.model(K, N, 8 * K, 2 * K, xavier_params(K, 2, seed=9))


def _run(model, H, y, x):
    n = H.shape[0]
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (H, y, x)]
    g = torch.empty((n, K * (K + 1) // 2), dtype=torch.float32, device="cuda")
    q = torch.empty((n, K), dtype=torch.float32, device="cuda")
    d = torch.empty((n,), dtype=torch.float64, device="cuda")
    f = torch.empty((n,), dtype=torch.uint8, device="cuda")
    model.preprocess_device(n, *dev, g, q, d, f)
    return g.cpu().numpy(), q.cpu().numpy(), d.cpu().numpy(), f.cpu().numpy()


def _inputs(oracle, n, lo, hi, seed=2):
    H, x, y, _ = oracle.generate_batch(oracle.rng(seed, 0), N, K, n, lo, hi)
    return ((H / np.sqrt(N)).astype(np.float32), (y / np.sqrt(N)).astype(np.float32),
            x.astype(np.int8))


def _oracle_pre(oracle, H, y, x):
    iu = np.triu_indices(K)
    G, q, dn = [], [], []
    for i in range(H.shape[0]):
        st, qi, Gi, xt = oracle.preprocess(H[i].astype(np.float64), y[i].astype(np.float64))
        assert st == 0
        G.append(Gi[iu]); q.append(qi)
        s = 0.0
        for v in x[i].astype(np.float64) - xt:  # loss.cpp:14-19 order
            s += v * v
        dn.append(max(s, 1e-12))
    return np.array(G), np.array(q), np.array(dn)


@pytest.mark.parametrize("exact", [False, True])
def test_preprocess_matches_oracle(model, oracle, exact):
    ctx, m = model
    H, y, x = _inputs(oracle, 1000, 0.0, 14.0)
    ctx.set_exact_preprocess(exact)
    try:
        g, q, d, f = _run(m, H, y, x)
    finally:
        ctx.set_exact_preprocess(False)
    Gr, qr, dr = _oracle_pre(oracle, H, y, x)
    assert np.abs(g - Gr).max() <= 1e-6 * np.abs(Gr).max()
    assert np.abs(q - qr).max() <= 1e-6 * np.abs(qr).max()
    rel = np.abs(d - dr) / dr
    assert rel.max() <= (1e-12 if exact else 1e-4), rel.max()
    assert not f.any()


def test_preprocess_multi_tile_deterministic(model, oracle):
    """2^16 samples = 1024 K1 tiles on <= 296 persistent CTAs: the outputs are
    run-to-run identical and agree with the exact mode (pair-local hand-offs)."""
    import paper_2003_09446_b200 as eng
    ctx, m = model
    n = 1 << 16
    H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
    y = torch.empty((n, N), dtype=torch.float32, device="cuda")
    x = torch.empty((n, K), dtype=torch.int8, device="cuda")
    base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131 + 5))
    ctx.generate(base, 0, n, N, K, 0.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
    outs = []
    for exact in (False, False, True):
        ctx.set_exact_preprocess(exact)
        g = torch.empty((n, 210), dtype=torch.float32, device="cuda")
        d = torch.empty((n,), dtype=torch.float64, device="cuda")
        m.preprocess_device(n, H, y, x, g, None, d)
        outs.append((g.cpu().numpy(), d.cpu().numpy()))
    ctx.set_exact_preprocess(False)
    (g1, d1), (g2, d2), (ge, de) = outs
    assert np.array_equal(g1, g2) and np.array_equal(d1, d2)
    assert (np.abs(g1 - ge).max(1) <= 1e-6 * np.abs(ge).max(1)).all()
    assert (np.abs(d1 - de) / de).max() <= 1e-4


def test_high_snr_and_noise_free_take_exact_path(model, oracle):
    """Above ~30 dB the FP32 residual H x - y loses accuracy: those samples
    (and the noise-free one, whose guard fires) get the reference LU values."""
    ctx, m = model
    H, y, x = _inputs(oracle, 256, 60.0, 80.0, seed=5)
    H0, _, x0 = _inputs(oracle, 1, 7.0, 7.0, seed=6)
    y0 = np.einsum("nij,nj->ni", H0.astype(np.float64), x0.astype(np.float64)).astype(np.float32)
    H, y, x = np.concatenate([H, H0]), np.concatenate([y, y0]), np.concatenate([x, x0])
    g, q, d, f = _run(m, H, y, x)
    Gr, qr, dr = _oracle_pre(oracle, H, y, x)
    np.testing.assert_array_equal(d, dr)
    np.testing.assert_array_equal(f, (dr <= 1e-12).astype(np.uint8))
