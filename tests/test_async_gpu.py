"""detnet_batch_evaluate_device_async / detnet_eval_wait: evaluations enqueued
without host round trips give exactly the synchronous results, in any wait
order; contract errors for too many in flight and unknown tickets; empty
batches; SingularMatrixError surfaces at wait time."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
K, N = 20, 30


def _ev(e):
    return (e.loss_sum, e.symbol_errors, e.symbols, e.flagged)


@pytest.fixture(scope="module")
def setup():
    import paper_2003_09446_b200 as eng
    from paper_2003_09446_b200.workload import xavier_params
    ctx = eng.Context(0)
    m = ctx.model(K, N, 160, 40, xavier_params(K, 5, seed=9))
    batches = []
    for p in range(6):
        n = 700 + 333 * p
        H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
        y = torch.empty((n, N), dtype=torch.float32, device="cuda")
        x = torch.empty((n, K), dtype=torch.int8, device="cuda")
        base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131 + p))
        ctx.generate(base, 0, n, N, K, 2.0 * p, 2.0 * p, 1.0 / np.sqrt(N), H, y, x)
        batches.append((n, H, y, x))
    return ctx, m, batches


def test_async_matches_sync(setup):
    ctx, m, batches = setup
    sync = [_ev(m.batch_evaluate_device(n, H, y, x)) for n, H, y, x in batches]
    tickets = [m.batch_evaluate_device_async(n, H, y, x) for n, H, y, x in batches * 3]
    order = list(range(len(tickets)))[::-1]  # wait newest first
    got = {i: _ev(ctx.eval_wait(tickets[i])) for i in order}
    for i in range(len(tickets)):
        assert got[i] == sync[i % len(batches)]


def test_async_contract(setup):
    from paper_2003_09446_b200.detnet import ContractError
    ctx, m, batches = setup
    n, H, y, x = batches[0]
    ts = [m.batch_evaluate_device_async(n, H, y, x) for _ in range(64)]
    with pytest.raises(ContractError):
        m.batch_evaluate_device_async(n, H, y, x)
    first = _ev(ctx.eval_wait(ts[0]))
    with pytest.raises(ContractError):
        ctx.eval_wait(ts[0])  # already consumed
    for t in ts[1:]:
        assert _ev(ctx.eval_wait(t)) == first
    t = m.batch_evaluate_device_async(0, H, y, x)
    e = ctx.eval_wait(t)
    assert e.symbols == 0 and e.loss_sum == 0.0 and e.symbol_errors == 0


def test_async_singular(setup, oracle):
    from paper_2003_09446_b200.detnet import SingularMatrixError
    ctx, m, _ = setup
    H = np.zeros((8, N, K), dtype=np.float32)
    H[:, :K, :] = np.eye(K, dtype=np.float32)
    H[3] = 0.0  # singular channel
    y = np.ones((8, N), dtype=np.float32)
    x = np.ones((8, K), dtype=np.int8)
    dev = [torch.from_numpy(a).cuda() for a in (H, y, x)]
    t = m.batch_evaluate_device_async(8, *dev)
    with pytest.raises(SingularMatrixError):
        ctx.eval_wait(t)


def test_update_waits_for_inflight(setup):
    """A model update while evaluations are in flight waits for them: the
    in-flight ones see the old weights, later ones the new."""
    import paper_2003_09446_b200 as eng
    from paper_2003_09446_b200.workload import xavier_params
    ctx, _, batches = setup
    pa, pb = xavier_params(K, 5, seed=21), xavier_params(K, 5, seed=22)
    m = ctx.model(K, N, 160, 40, pa)
    ref_a, ref_b = ctx.model(K, N, 160, 40, pa), ctx.model(K, N, 160, 40, pb)
    n, H, y, x = batches[-1]
    want_a = _ev(ref_a.batch_evaluate_device(n, H, y, x))
    want_b = _ev(ref_b.batch_evaluate_device(n, H, y, x))
    t1 = [m.batch_evaluate_device_async(n, H, y, x) for _ in range(4)]
    m.update(pb)
    t2 = m.batch_evaluate_device_async(n, H, y, x)
    assert all(_ev(ctx.eval_wait(t)) == want_a for t in t1)
    assert _ev(ctx.eval_wait(t2)) == want_b


def test_training_steps_without_waits(setup):
    """train_grad(want_eval=False) + train_apply, stream-ordered with no host
    waits, leave the same parameters as the waiting sequence."""
    from paper_2003_09446_b200.workload import xavier_params
    ctx, _, batches = setup
    out = []
    for want in (True, False):
        m = ctx.model(K, N, 160, 40, xavier_params(K, 5, seed=23))
        raw = m.new_raw()
        for n, H, y, x in batches[:4]:
            m.train_grad(n, H, y, x, raw, want_eval=want)
            m.train_apply(raw, n, kind=2, lam1=1e-4, lr0=1e-3)
        out.append(m.get_params())
    assert np.array_equal(out[0], out[1])


def test_pinned_host_buffers_from_the_c_abi():
    """detnet_host_alloc / detnet_host_free: page-locked sample buffers give the
    same BatchEval as pageable ones (the seam stages its FP32 batches there)."""
    import ctypes as C
    import numpy as np
    from paper_2003_09446_b200 import Context, detnet as d
    from paper_2003_09446_b200.workload import xavier_params
    K, N, L, n = 20, 30, 4, 3000
    rs = np.random.default_rng(5)
    H = (rs.standard_normal((n, N, K)) / np.sqrt(N)).astype(np.float32)
    x = np.where(rs.random((n, K)) < 0.5, -1, 1).astype(np.int8)
    y = (np.einsum("sij,sj->si", H, x.astype(np.float32)) +
         0.2 * rs.standard_normal((n, N)).astype(np.float32)).astype(np.float32)
    lib = d._lib
    lib.detnet_host_alloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t]
    lib.detnet_host_free.argtypes = [C.c_void_p]
    ptrs = []
    for a in (H, y, x):
        p = C.c_void_p()
        assert lib.detnet_host_alloc(C.byref(p), a.nbytes) == 0 and p.value
        C.memmove(p.value, a.ctypes.data, a.nbytes)
        ptrs.append(p)
    z = C.c_void_p(1)
    assert lib.detnet_host_alloc(C.byref(z), 0) == 0 and not z.value
    ctx = Context(0)
    m = ctx.model(K, N, 8 * K, 2 * K, xavier_params(K, L, seed=9))
    want = m.batch_evaluate(H, y, x)
    ev = d._Eval()
    d._check(lib.detnet_batch_evaluate(m._h, n, ptrs[0].value, ptrs[1].value, ptrs[2].value, 0, None,
                                       C.byref(ev)))
    assert (ev.data_loss, ev.symbol_errors, ev.flagged) == (want.data_loss, want.symbol_errors,
                                                            want.flagged)
    for p in ptrs:
        assert lib.detnet_host_free(p) == 0
    assert lib.detnet_host_free(None) == 0
    ctx.close()
