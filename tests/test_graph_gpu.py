"""Repeated detnet_batch_evaluate_device calls are replayed as one captured
CUDA graph (K1 + fallback + stack + reduce + result copy): the replays give
bit-identical results to the eager first call, count the same kernels, see new
input contents, and are invalidated by a model update and by context settings."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
K, N = 20, 30


def _ev(e):
    return (e.loss_sum, e.symbol_errors, e.symbols, e.flagged)


def test_graph_replay_matches_eager(oracle):
    import paper_2003_09446_b200 as eng
    from paper_2003_09446_b200.workload import xavier_params
    ctx = eng.Context(0)
    n, L = 3000, 6
    m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
    H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
    y = torch.empty((n, N), dtype=torch.float32, device="cuda")
    x = torch.empty((n, K), dtype=torch.int8, device="cuda")
    xh = torch.zeros((n, L, K), dtype=torch.float32, device="cuda")
    base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131))
    ctx.generate(base, 0, n, N, K, 7.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
    runs, xhs, launches = [], [], []
    for _ in range(4):  # eager, capture + replay, replay, replay
        l0 = ctx.launch_count
        runs.append(_ev(m.batch_evaluate_device(n, H, y, x, xhat_ptr=xh)))
        launches.append(ctx.launch_count - l0)
        xhs.append(xh.clone())
    assert all(r == runs[0] for r in runs), runs
    assert all(torch.equal(a, xhs[0]) for a in xhs)
    assert len(set(launches)) == 1 and launches[0] > 0, launches
    # new contents in the same buffers: the replay reads them
    ctx.generate(base, n, n, N, K, 7.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
    fresh = _ev(m.batch_evaluate_device(n, H, y, x, xhat_ptr=xh))
    assert fresh != runs[0]
    ctx.set_exact_preprocess(True)  # a settings change re-keys (eager run) ...
    m.batch_evaluate_device(n, H, y, x, xhat_ptr=xh)
    ctx.set_exact_preprocess(False)  # ... and back
    assert [_ev(m.batch_evaluate_device(n, H, y, x, xhat_ptr=xh)) for _ in range(3)] == [fresh] * 3
    # a model update invalidates the captured graph
    p2 = xavier_params(K, L, seed=10)
    m.update(p2)
    upd = [_ev(m.batch_evaluate_device(n, H, y, x, xhat_ptr=xh)) for _ in range(3)]
    ref = ctx.model(K, N, 160, 40, p2)
    assert all(u == upd[0] for u in upd)
    assert upd[0] == _ev(ref.batch_evaluate_device(n, H, y, x, xhat_ptr=xh))
    assert upd[0] != fresh


def test_graph_replay_sparse_jit_model(oracle):
    """The same replay for a sparse-group model on the NVRTC-compiled kernel
    (a library kernel launched through cudaLaunchKernel inside the capture),
    and a model update to other sparse weights regenerates it."""
    import paper_2003_09446_b200 as eng
    from paper_2003_09446_b200.workload import group_masks, sparse_group_model, xavier_params
    ctx = eng.Context(0, path=3)
    n, L = 3000, 5
    ps, ms = sparse_group_model(xavier_params(K, L, seed=9), group_masks(K, L, seed=31), K)
    m = ctx.model(K, N, 160, 40, ps, masks=ms)
    assert m.path_name == "sparse-jit-fp32"
    H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
    y = torch.empty((n, N), dtype=torch.float32, device="cuda")
    x = torch.empty((n, K), dtype=torch.int8, device="cuda")
    xh = torch.zeros((n, L, K), dtype=torch.float32, device="cuda")
    base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131))
    ctx.generate(base, 0, n, N, K, 7.0, 14.0, 1.0 / np.sqrt(N), H, y, x)
    runs, xhs = [], []
    for _ in range(4):
        runs.append(_ev(m.batch_evaluate_device(n, H, y, x, xhat_ptr=xh)))
        xhs.append(xh.clone())
    assert all(r == runs[0] for r in runs), runs
    assert all(torch.equal(a, xhs[0]) for a in xhs)
    p2, m2 = sparse_group_model(xavier_params(K, L, seed=10), group_masks(K, L, seed=32), K)
    m.update(p2, masks=m2)
    assert m.path_name == "sparse-jit-fp32"
    upd = [_ev(m.batch_evaluate_device(n, H, y, x, xhat_ptr=xh)) for _ in range(3)]
    ref = ctx.model(K, N, 160, 40, p2, masks=m2)
    assert all(u == upd[0] for u in upd)
    assert upd[0] == _ev(ref.batch_evaluate_device(n, H, y, x, xhat_ptr=xh))
    assert upd[0] != runs[0]
