"""One seam call over a device group (detnet_ctx_create_group):
the batch is sharded at 8,192-sample chunk boundaries and every reduction is
folded in the canonical chunk order, so BatchEval, soft outputs and
gradients are bit-identical for any group size -- the reference's
thread-count invariance (kernels.cpp:93-103, 160-200; README.md:83-91;
tests/test_kernels.cpp:53-91). One GPU here: the group repeats device 0
(G "virtual shards", each a context of its own on its own host thread)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
K, N = 20, 30


def _inputs(oracle, n, seed=4):
    r = oracle.rng(seed, 0)
    H, x, y, _ = oracle.generate_batch(r, N, K, n, 7.0, 14.0)
    return ((H / np.sqrt(N)).astype(np.float32), (y / np.sqrt(N)).astype(np.float32),
            x.astype(np.int8))


@pytest.mark.parametrize("path", [0, 1])
def test_group_evaluate_bit_identical(oracle, path):
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    n, L = 41_000, 6  # 6 chunks, the last one ragged
    params = xavier_params(K, L, seed=9)
    H, y, x = _inputs(oracle, n)
    base_ev, base_xh = Context(0, path=path).model(K, N, 160, 40, params).batch_evaluate(
        H, y, x, want_xhat=True)
    for G in (1, 2, 3, 8):
        c = Context(devices=[0] * G, path=path)
        assert c.group_size == G
        ev, xh = c.model(K, N, 160, 40, params).batch_evaluate(H, y, x, want_xhat=True)
        assert (ev.data_loss, ev.loss_sum, ev.symbol_errors, ev.flagged) == \
            (base_ev.data_loss, base_ev.loss_sum, base_ev.symbol_errors, base_ev.flagged), G
        assert np.array_equal(xh, base_xh), G


@pytest.mark.parametrize("kind,lam1", [(0, 0.0), (2, 1e-4)])
def test_group_gradient_bit_identical(oracle, kind, lam1):
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    n, L = 40_000, 4
    params = xavier_params(K, L, seed=9)
    H, y, x = _inputs(oracle, n, seed=6)
    ev0, g0 = Context(0).model(K, N, 160, 40, params).batch_gradient(H, y, x, kind, 0.0, lam1)
    for G in (1, 2, 3, 8):
        c = Context(devices=[0] * G)
        ev, g = c.model(K, N, 160, 40, params).batch_gradient(H, y, x, kind, 0.0, lam1)
        assert np.array_equal(g, g0), (G, np.abs(g - g0).max())
        assert (ev.data_loss, ev.symbol_errors, ev.flagged) == (ev0.data_loss, ev0.symbol_errors,
                                                                ev0.flagged), G


def test_group_replicas_follow_device_training(oracle):
    """After device-side training steps on the first member, the next group
    evaluation refreshes the replicas (same result as a single device)."""
    import torch
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    L, n = 3, 20_000
    params = xavier_params(K, L, seed=2)
    H, y, x = _inputs(oracle, n, seed=8)
    outs = []
    for c in (Context(0), Context(devices=[0, 0, 0])):
        m = c.model(K, N, 160, 40, params)
        raw = m.new_raw()
        Hd, yd, xd = (torch.from_numpy(a).cuda() for a in (H[:4096], y[:4096], x[:4096]))
        for _ in range(3):
            m.train_grad(4096, Hd, yd, xd, raw)
            m.train_apply(raw, 4096, kind=2, lam1=1e-4, lr0=1e-3)
        outs.append(m.batch_evaluate(H, y, x))
    assert (outs[0].data_loss, outs[0].symbol_errors) == (outs[1].data_loss, outs[1].symbol_errors)


def test_rank_chunk_sums_fold_to_single_device(oracle):
    """parallel.reduce_stats's input: the per-chunk loss sums of each rank's
    chunk-aligned shard, folded in global order, equal one device's loss sum
    over the whole batch bit for bit (any number of ranks)."""
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.parallel import CHUNK, fold_chunks
    from paper_2003_09446_b200.workload import xavier_params
    n, L = 5 * CHUNK + 77, 5
    params = xavier_params(K, L, seed=9)
    H, y, x = _inputs(oracle, n, seed=11)
    c = Context(0)
    m = c.model(K, N, 160, 40, params)
    ev = m.batch_evaluate(H, y, x)
    whole = c.chunk_sums()
    assert len(whole) == 6 and fold_chunks(None, whole) == ev.loss_sum
    for cuts in ([0, 2 * CHUNK, n], [0, CHUNK, 3 * CHUNK, 4 * CHUNK, n]):
        parts = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            m.batch_evaluate(H[a:b], y[a:b], x[a:b])
            parts.extend(c.chunk_sums())
        assert fold_chunks(None, parts) == ev.loss_sum, cuts
