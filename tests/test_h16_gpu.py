"""Split-FP16 tensor-core stack (stack_h16.cu): the FP16 range guard and the
3xTF32 recompute of flagged tiles.

A tile whose scaled activations reach the FP16 limit is recomputed by the
3xTF32 kernel on the same inputs, so a recomputed tile must be bit-identical
to the 3xTF32 path (ctx path 2). DETNET_H16_LIMIT lowers the limit to force
the recompute of every tile."""
import numpy as np
import pytest

from oracle.oracle import Model as OModel

pytestmark = pytest.mark.gpu

K, N = 20, 30


@pytest.fixture(scope="module")
def ctx():
    from paper_2003_09446_b200 import Context
    return Context(0)


def _inputs(oracle, n, seed=2):
    r = oracle.rng(seed, 0)
    H, x, y, _ = oracle.generate_batch(r, N, K, n, 7.0, 14.0)
    return ((H / np.sqrt(N)).astype(np.float32), (y / np.sqrt(N)).astype(np.float32),
            x.astype(np.int8))


def _eval(ctx, m, path, H, y, x):
    ctx.set_path(path)
    try:
        return m.batch_evaluate(H, y, x, want_xhat=True)
    finally:
        ctx.set_path(0)


def test_default_path_is_split_fp16(ctx):
    from paper_2003_09446_b200.workload import xavier_params
    m = ctx.model(K, N, 160, 40, xavier_params(K, 4, seed=9))
    assert m.path_name == "tcgen05-split-fp16"
    ctx.set_path(2)
    assert m.path_name == "tcgen05-3xtf32"
    ctx.set_path(0)


def test_forced_recompute_is_bitwise_3xtf32(ctx, oracle, monkeypatch):
    from paper_2003_09446_b200.workload import xavier_params
    m = ctx.model(K, N, 160, 40, xavier_params(K, 12, seed=9))
    H, y, x = _inputs(oracle, 1000)
    ev2, xh2 = _eval(ctx, m, 2, H, y, x)
    evh, xhh = _eval(ctx, m, 0, H, y, x)
    assert not np.array_equal(xhh, xh2)  # the two kernels round differently
    monkeypatch.setenv("DETNET_H16_LIMIT", "0")  # every tile out of "range"
    evr, xhr = _eval(ctx, m, 0, H, y, x)
    assert np.array_equal(xhr, xh2)
    assert evr.data_loss == ev2.data_loss and evr.symbol_errors == ev2.symbol_errors
    assert evr.flagged == ev2.flagged


def test_forced_recompute_restarts_from_input_state(ctx, oracle, monkeypatch):
    from paper_2003_09446_b200.workload import xavier_params
    m = ctx.model(K, N, 160, 40, xavier_params(K, 12, seed=9))
    H, y, _ = _inputs(oracle, 300)
    rs = np.random.default_rng(4)
    xs = rs.uniform(-1, 1, (300, K)).astype(np.float32)
    vs = rs.normal(0, 1, (300, 40)).astype(np.float32)
    ctx.set_path(2)
    x2, v2, h2 = m.forward_range(H, y, 3, 9, xs, vs)
    ctx.set_path(0)
    monkeypatch.setenv("DETNET_H16_LIMIT", "0")
    xr, vr, hr = m.forward_range(H, y, 3, 9, xs, vs)
    assert np.array_equal(xr, x2) and np.array_equal(vr, v2) and np.array_equal(hr, h2)


def test_out_of_range_tile_is_recomputed(ctx, oracle):
    """Tile 1 gets received signals 1e5 times larger: its scaled q leaves the
    FP16 range, so that tile (only) must come from the 3xTF32 kernel, while
    the other tiles stay on split FP16 and within tolerance of the oracle."""
    from paper_2003_09446_b200.workload import xavier_params
    params = xavier_params(K, 10, seed=9)
    m = ctx.model(K, N, 160, 40, params)
    H, y, x = _inputs(oracle, 512)
    y[128:256] *= 1e5
    ev2, xh2 = _eval(ctx, m, 2, H, y, x)
    evh, xhh = _eval(ctx, m, 0, H, y, x)
    assert np.array_equal(xhh[128:256], xh2[128:256])
    assert not np.array_equal(xhh[:128], xh2[:128])
    ref = oracle.evaluate(OModel(K, N, 160, 40, 10, params), H.astype(np.float64),
                          y.astype(np.float64), x.astype(np.float64), want_xhat=True)
    ok = np.abs(xhh - ref["xhat"]) <= 1e-5 + 1e-4 * np.abs(ref["xhat"])
    assert np.mean(ok) > 0.99
    assert abs(evh.data_loss - ref["loss"].mean()) <= 1e-4 * abs(ref["loss"].mean())


def test_weights_outside_fp16_range_use_3xtf32(ctx, oracle):
    from paper_2003_09446_b200.workload import xavier_params
    params = xavier_params(K, 3, seed=9)
    params[1, 5] = 1e4  # x 16 (image scale) > FP16 max
    m = ctx.model(K, N, 160, 40, params)
    assert m.path_name == "tcgen05-3xtf32"


def test_hidden_unit_overflow_is_recomputed(ctx, oracle):
    """A hidden activation beyond the FP16 range (scaled z > 65504, i.e.
    z > 2047) flags its tile. Bias b1 = 3000 in layer 1 does that for every
    tile, so the whole batch must equal the 3xTF32 path bit for bit."""
    from paper_2003_09446_b200.workload import xavier_params
    params = xavier_params(K, 4, seed=9)
    IN = 3 * K + 40
    params[1, 160 * IN:160 * IN + 160] = 3000.0  # b1 of layer 1: x16 fits FP16, z = 32 u1 does not
    m = ctx.model(K, N, 160, 40, params)
    assert m.path_name == "tcgen05-split-fp16"
    H, y, x = _inputs(oracle, 400)
    ev2, xh2 = _eval(ctx, m, 2, H, y, x)
    evh, xhh = _eval(ctx, m, 0, H, y, x)
    assert np.array_equal(xhh, xh2)
    assert evh.data_loss == ev2.data_loss and evh.symbol_errors == ev2.symbol_errors


@pytest.mark.parametrize("path", [1, 2, 4])
def test_device_packing_matches_host_packing(oracle, path, monkeypatch):
    """Dense models are packed on the device at upload (SIMT records and both
    tensor-core image sets from the FP64 records); the host packers build the
    same layouts: evaluations agree bit for bit on every kernel path."""
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    params = xavier_params(K, 7, seed=12)
    H, y, x = _inputs(oracle, 3000)
    c = Context(0, path=path)
    dev = c.model(K, N, 160, 40, params)
    monkeypatch.setenv("DETNET_HOST_PACK", "1")
    host = c.model(K, N, 160, 40, params)
    monkeypatch.delenv("DETNET_HOST_PACK")
    ea, xa = dev.batch_evaluate(H, y, x, want_xhat=True)
    eb, xb = host.batch_evaluate(H, y, x, want_xhat=True)
    assert np.array_equal(xa, xb)
    assert (ea.loss_sum, ea.symbol_errors) == (eb.loss_sum, eb.symbol_errors)
