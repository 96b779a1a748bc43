"""BASELINE.json's configurations at their full sizes, checked through
properties that do not need the (slow) oracle over the whole batch:

* config 2 (L=40, 2^20 detections of one SNR point, device-resident):
  run-to-run determinism; additivity over sub-batches cut at the canonical
  8,192-sample chunk boundaries (integer outputs exact, the FP64 loss sum to
  1e-12); invariance under a permutation of those chunks; the first 2,048
  indices tie the result to the reference library (harness.cpp:133-138).
* config 1 (L=90, n=4,096, every x_l returned): the returned soft outputs
  reproduce the call's own BatchEval -- the error count from sign(x_L)
  (kernels.cpp:63-65, sign(0) = +1) exactly and loss_plain (loss.cpp:9-31)
  recomputed in numpy FP64 from x_l and the zero-forcing estimate to 1e-5.
* configs 3/4 (group / sparse-group masks, L=40, 2^20 detections): the masked
  model and its explicitly zeroed twin are bit-identical (acceptance C3,
  tests/test_compression.cpp:165-203), and both masks' evaluations are
  additive like config 2's.
* config 5 (L=40, batch 5,000): the batch gradient is the sample-weighted
  mean of the gradients of its two halves (linearity of backward_data,
  backward.cpp:105-165) and the FP64 mode reproduces it to 1e-9.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
K, N, Z, V = 20, 30, 160, 40
CHUNK = 8192


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _device_point(torch, ctx, n, snr, point=5, seed=1):
    import paper_2003_09446_b200 as eng
    H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
    y = torch.empty((n, N), dtype=torch.float32, device="cuda")
    x = torch.empty((n, K), dtype=torch.int8, device="cuda")
    base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(seed, 0), 0x45564131 + point))
    ctx.generate(base, 0, n, N, K, snr, snr, 1.0 / np.sqrt(N), H, y, x)
    torch.cuda.synchronize()
    return H, y, x


def _tuple(ev):
    return (ev.symbol_errors, ev.flagged, ev.symbols, ev.loss_sum)


def _additive(model, n, H, y, x, cuts):
    whole = model.batch_evaluate_device(n, H, y, x)
    parts = [model.batch_evaluate_device(b - a, H[a:b], y[a:b], x[a:b])
             for a, b in zip(cuts[:-1], cuts[1:])]
    assert sum(p.symbol_errors for p in parts) == whole.symbol_errors
    assert sum(p.flagged for p in parts) == whole.flagged
    assert sum(p.symbols for p in parts) == whole.symbols == n * K
    s = sum(p.loss_sum for p in parts)
    assert abs(s - whole.loss_sum) <= 1e-12 * abs(whole.loss_sum)
    assert abs(whole.data_loss - whole.loss_sum / n) <= 1e-15 * abs(whole.data_loss)
    return whole


def test_config2_full_point_properties(torch_cuda, ref):
    torch = torch_cuda
    from oracle.oracle import Model as OModel
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    n, L = 1 << 20, 40
    params = xavier_params(K, L, seed=9)
    ctx = Context(0)
    model = ctx.model(K, N, Z, V, params)
    assert model.path_name == "tcgen05-split-fp16"
    H, y, x = _device_point(torch, ctx, n, 10.0)
    # ragged cuts at chunk boundaries (1, 37, 64 and 26 chunks)
    cuts = [0, CHUNK, 38 * CHUNK, 102 * CHUNK, n]
    whole = _additive(model, n, H, y, x, cuts)
    again = model.batch_evaluate_device(n, H, y, x)
    assert _tuple(again) == _tuple(whole)  # bit-identical rerun
    assert 0.0 < whole.ber() < 1.0 and np.isfinite(whole.data_loss)
    # the same chunks in another order: the integers cannot change, the FP64
    # loss only by the order of the chunk fold
    perm = torch.randperm(n // CHUNK, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    idx = (perm[:, None] * CHUNK + torch.arange(CHUNK, device="cuda")[None, :]).reshape(-1)
    Hp, yp, xp = H[idx].contiguous(), y[idx].contiguous(), x[idx].contiguous()
    shuf = model.batch_evaluate_device(n, Hp, yp, xp)
    assert (shuf.symbol_errors, shuf.flagged) == (whole.symbol_errors, whole.flagged)
    assert abs(shuf.loss_sum - whole.loss_sum) <= 1e-12 * abs(whole.loss_sum)
    del Hp, yp, xp
    # tie to the reference on the first 2,048 indices of the stream
    m = 2048
    head = model.batch_evaluate_device(m, H[:m], y[:m], x[:m])
    r = ref.batch_evaluate(OModel(K, N, Z, V, L, params), H[:m].cpu().numpy().astype(np.float64),
                           y[:m].cpu().numpy().astype(np.float64), x[:m].cpu().numpy().astype(np.float64))
    assert head.flagged == r["flagged"]
    # untrained 40-layer stacks amplify last-bit differences into rare sign flips of
    # soft outputs near 0: allow 2 of 40,960 decisions
    assert abs(head.symbol_errors - r["symbol_errors"]) <= 2
    assert abs(head.data_loss - r["data_loss"]) <= 1e-4 * abs(r["data_loss"])
    ctx.close()


def test_config1_soft_outputs_reproduce_batch_eval(torch_cuda, oracle):
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    n, L = 4096, 90
    params = xavier_params(K, L, seed=9)
    r = oracle.rng(1, 0)
    Hd, xd, yd, _ = oracle.generate_batch(r, N, K, n, 7.0, 14.0)
    H = (Hd / np.sqrt(N)).astype(np.float32)
    y = (yd / np.sqrt(N)).astype(np.float32)
    x = xd.astype(np.int8)
    ctx = Context(0)
    ev, xh = ctx.model(K, N, Z, V, params).batch_evaluate(H, y, x, want_xhat=True)
    assert xh.shape == (n, L, K) and np.isfinite(xh).all()
    assert np.abs(xh).max() <= 1.0  # psi_t saturates at +-1 (model.cpp:32-51)
    dec = np.where(xh[:, L - 1, :] >= 0.0, 1, -1)
    assert int((dec != x).sum()) == ev.symbol_errors
    assert ev.symbols == n * K
    # loss_plain in FP64 from the returned x_l and the zero-forcing estimate
    H64, y64, x64 = H.astype(np.float64), y.astype(np.float64), x.astype(np.float64)
    G = np.einsum("sij,sik->sjk", H64, H64)
    q = np.einsum("sij,si->sj", H64, y64)
    xt = np.linalg.solve(G, q[:, :, None])[:, :, 0]
    denom = ((x64 - xt) ** 2).sum(axis=1)
    assert int((denom < 1e-12).sum()) == ev.flagged
    denom = np.maximum(denom, 1e-12)
    err = ((x64[:, None, :] - xh.astype(np.float64)) ** 2).sum(axis=2)  # [n][L]
    w = np.log(np.arange(1, L + 1, dtype=np.float64))
    loss = (err * w[None, :]).sum(axis=1) / denom
    assert abs(loss.mean() - ev.data_loss) <= 1e-5 * abs(ev.data_loss)
    ctx.close()


@pytest.mark.parametrize("cfg,path", [(3, 0), (4, 0), (4, 3)])  # path 3: the sparse JIT kernel
def test_masked_configs_full_size_masked_equals_zeroed(torch_cuda, cfg, path):
    torch = torch_cuda
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200 import workload as wl
    n, L = 1 << 20, 40
    params = wl.xavier_params(K, L, seed=9)
    masks = wl.group_masks(K, L, seed=31)
    if cfg == 4:
        params, masks = wl.sparse_group_model(params, masks, K)
    ctx = Context(0, path=path)
    H, y, x = _device_point(torch, ctx, n, 8.0, point=4)
    masked = ctx.model(K, N, Z, V, params, masks=masks)
    zeroed = ctx.model(K, N, Z, V, params * masks)
    a = _additive(masked, n, H, y, x, [0, 5 * CHUNK, 77 * CHUNK, n])
    b = zeroed.batch_evaluate_device(n, H, y, x)
    assert _tuple(a) == _tuple(b)
    assert masked.path_name == zeroed.path_name
    if path == 3:
        assert masked.path_name == "sparse-jit-fp32"
    ctx.close()


def test_config5_gradient_is_linear_in_the_batch(torch_cuda, oracle):
    from paper_2003_09446_b200 import Context
    from paper_2003_09446_b200.workload import xavier_params
    n, L = 5000, 40
    params = xavier_params(K, L, seed=9)
    r = oracle.rng(1, 2)
    Hd, xd, yd, _ = oracle.generate_batch(r, N, K, n, 7.0, 14.0)
    H = (Hd / np.sqrt(N)).astype(np.float32)
    y = (yd / np.sqrt(N)).astype(np.float32)
    x = xd.astype(np.int8)
    h = 2048  # a boundary of the 1,024-sample gradient splits
    for fp64, tol in ((False, 2e-5), (True, 1e-9)):
        ctx = Context(0)
        ctx.set_train_precision(fp64)
        model = ctx.model(K, N, Z, V, params)
        ev, g = model.batch_gradient(H, y, x, kind=0)
        ev1, g1 = model.batch_gradient(H[:h], y[:h], x[:h], kind=0)
        ev2, g2 = model.batch_gradient(H[h:], y[h:], x[h:], kind=0)
        mix = (h * g1 + (n - h) * g2) / n
        scale = np.abs(g).max()
        assert scale > 0 and np.isfinite(g).all()
        assert np.abs(g - mix).max() <= tol * scale, (fp64, np.abs(g - mix).max() / scale)
        assert ev.symbol_errors == ev1.symbol_errors + ev2.symbol_errors
        assert abs(ev.data_loss - (h * ev1.data_loss + (n - h) * ev2.data_loss) / n) \
            <= 1e-6 * abs(ev.data_loss)
        ctx.close()
