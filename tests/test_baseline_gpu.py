"""ZF / ML / oracle detector baselines on the device
(detnet_batch_baseline_errors) against the reference library's own
batch_baseline_errors (kernels.cpp:202-223) on the reference's FP64 samples:
error counts must be identical (decisions are computed in the reference's
operation order, so even near-zero ZF components and ML ties agree)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2003_09446_b200 as eng
    return eng.Context(0)


def _batch(oracle, seed, N, K, n, lo, hi):
    r = oracle.rng(seed, 0)
    H, x, y, _ = oracle.generate_batch(r, N, K, n, lo, hi)
    return H, y, x


@pytest.mark.parametrize("K,N,n,lo,hi", [(2, 4, 3000, 0.0, 12.0), (4, 8, 3000, 0.0, 15.0),
                                         (8, 12, 2000, 4.0, 12.0), (20, 30, 4096, 7.0, 14.0),
                                         (3, 3, 2000, -5.0, 5.0),
                                         # wider than the register kernels: shared-memory ZF
                                         (21, 30, 1500, 7.0, 14.0), (32, 32, 600, 0.0, 20.0),
                                         (40, 64, 400, 5.0, 15.0), (70, 72, 64, 10.0, 20.0)])
def test_zf_errors_match_reference(ctx, oracle, ref, K, N, n, lo, hi):
    H, y, x = _batch(oracle, 11 + K, N, K, n, lo, hi)
    st, e_ref, s_ref = ref.baseline_errors(0, H, y, x)
    assert st == 0, st
    e, s = ctx.baseline_errors(0, H, y, x)
    assert (e, s) == (e_ref, s_ref)


@pytest.mark.parametrize("K,N,n", [(2, 4, 3000), (4, 6, 2000), (8, 10, 1000), (12, 16, 64)])
def test_ml_errors_match_reference(ctx, oracle, ref, K, N, n):
    H, y, x = _batch(oracle, 31 + K, N, K, n, 0.0, 10.0)
    st, e_ref, s_ref = ref.baseline_errors(1, H, y, x)
    assert st == 0, st
    e, s = ctx.baseline_errors(1, H, y, x)
    assert (e, s) == (e_ref, s_ref)


def test_ml_ties_first_strict_minimum(ctx, ref):
    """Duplicated columns make candidates tie exactly: the first strict
    minimum in ascending candidate order must win, as in channel.cpp:49-62."""
    rs = np.random.default_rng(5)
    K, N, n = 4, 6, 500
    H = rs.standard_normal((n, N, K))
    H[:, :, 1] = H[:, :, 0]  # s0 and s1 are interchangeable -> exact metric ties
    x = np.where(rs.random((n, K)) < 0.5, -1.0, 1.0)
    y = np.einsum("nij,nj->ni", H, x) + 0.3 * rs.standard_normal((n, N))
    st, e_ref, s_ref = ref.baseline_errors(1, H, y, x)
    assert st == 0
    assert ctx.baseline_errors(1, H, y, x) == (e_ref, s_ref)


def test_baseline_edges(ctx, ref):
    import paper_2003_09446_b200 as eng
    H = np.zeros((4, 6, 3)); y = np.zeros((4, 6)); x = np.ones((4, 3))
    # oracle kind: zero errors, symbols counted
    assert ctx.baseline_errors(2, H, y, x) == (0, 12)
    # singular normal equations -> SingularMatrixError like linalg.cpp:59-60
    assert ref.baseline_errors(0, H, y, x)[0] == 2
    with pytest.raises(eng.SingularMatrixError):
        ctx.baseline_errors(0, H, y, x)
    # ML beyond K = 16 fails in the reference (CapacityError from ml_decode,
    # rethrown as runtime_error by the OpenMP error slot of kernels.cpp:207-222)
    H = np.random.default_rng(1).standard_normal((1, 20, 17))
    assert ref.baseline_errors(1, H, np.zeros((1, 20)), np.ones((1, 17)))[0] != 0
    with pytest.raises(eng.UnsupportedError):
        ctx.baseline_errors(1, H, np.zeros((1, 20)), np.ones((1, 17)))
    # singular wide system on the shared-memory ZF path
    Hs = np.random.default_rng(2).standard_normal((3, 30, 24))
    Hs[1, :, 5] = Hs[1, :, 7]
    ys = np.random.default_rng(3).standard_normal((3, 30)); xs = np.ones((3, 24))
    assert ref.baseline_errors(0, Hs, ys, xs)[0] == 2
    with pytest.raises(eng.SingularMatrixError):
        ctx.baseline_errors(0, Hs, ys, xs)
    # empty batch
    assert ctx.baseline_errors(0, np.zeros((0, 6, 3)), np.zeros((0, 6)), np.zeros((0, 3))) == (0, 0)
