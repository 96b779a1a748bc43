"""GPU parity of the model-specialised sparse kernel (sparse_jit.cu): the
surviving weights of a sparse model compiled into FFMA immediates.

The generator has branches the BASELINE config-4 model never takes (its
biases are zero): nonzero b1/b2/b3 (added last as FADD immediates), hidden
units with no surviving W1 entry (the constant relu(b1) folded into the
output biases, or dead when b1 <= 0), output rows with no surviving entry
(the bias alone), per-layer t != 0.5 (psi_t scale folded into W2/b2), and
n_tx other than 20 (the Gram 2x2 blocks pad an odd K). Each is checked end to
end against the oracle's masked_affine (model.cpp:58-80) with the tolerances
of tests/test_parity_gpu.py.
"""
import numpy as np
import pytest

from test_parity_gpu import _e2e_ok, _inputs, _omodel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2003_09446_b200 import Context
    c = Context(0)
    c.set_path(3)
    return c


def _sparse_model(K, L, seed, keep=0.08, bias=True, const_units=True):
    """Random sparse masks over every weight, nonzero biases, per-layer t."""
    from paper_2003_09446_b200.workload import record_layout, xavier_params
    Z, V = 8 * K, 2 * K
    IN = 3 * K + V
    sl, P = record_layout(K, Z, V)
    rs = np.random.default_rng(seed)
    params = xavier_params(K, L, seed=seed)
    masks = np.zeros_like(params)
    for l in range(L):
        for name in ("W1", "W2", "W3"):
            masks[l, sl[name]] = (rs.random(sl[name].stop - sl[name].start) < keep)
        masks[l, sl["b1"]] = masks[l, sl["b2"]] = masks[l, sl["b3"]] = masks[l, sl["t"]] = 1.0
        if bias:
            params[l, sl["b1"]] = rs.normal(0.0, 0.1, Z)
            params[l, sl["b2"]] = rs.normal(0.0, 0.05, K)
            params[l, sl["b3"]] = rs.normal(0.0, 0.05, V)
        params[l, sl["t"]] = rs.uniform(0.3, 0.9)
        if const_units:
            # two hidden units without W1 entries: one with b1 > 0 (a constant
            # z folded into the outputs), one with b1 < 0 (dead)
            W1 = masks[l, sl["W1"]].reshape(Z, IN)
            W1[:2, :] = 0.0
            masks[l, sl["W1"]] = W1.ravel()
            b1 = params[l, sl["b1"]]
            b1[0], b1[1] = 0.3, -0.3
            params[l, sl["b1"]] = b1
            W3 = masks[l, sl["W3"]].reshape(V, Z)
            W3[:, :2] = 1.0  # the constant unit reaches every v row
            masks[l, sl["W3"]] = W3.ravel()
    return params.astype(np.float32).astype(np.float64), masks


@pytest.mark.parametrize("K", [3, 4, 8, 20])
def test_sparse_jit_matches_oracle(ctx, oracle, K):
    L = 6
    # K = 20 at 4 %: ~1,000 surviving products per layer, under the JIT limit
    params, masks = _sparse_model(K, L, seed=11 + K, keep=0.04 if K == 20 else 0.08)
    H, y, x = _inputs(oracle, 700, K=K, N=2 * K, seed=3)
    m = ctx.model(K, 2 * K, 8 * K, 2 * K, params, masks=masks)
    assert m.path_name == "sparse-jit-fp32"
    ev, xh = m.batch_evaluate(H, y, x, want_xhat=True)
    ref = oracle.evaluate(_omodel(params, K=K, N=2 * K, masks=masks), H.astype(np.float64),
                          y.astype(np.float64), x.astype(np.float64), want_xhat=True)
    ok, stats = _e2e_ok(xh, ref["xhat"])
    assert ok, stats
    assert ev.symbol_errors == int(ref["errors"].sum())
    assert abs(ev.data_loss - ref["loss"].mean()) <= 1e-4 * abs(ref["loss"].mean())


def test_sparse_jit_ragged_batch_and_trainable_loss(ctx, oracle):
    """A batch that is not a whole number of tiles (the last tile's dead
    samples contribute nothing) and the trainable-only loss weights."""
    K, L = 20, 5
    params, masks = _sparse_model(K, L, seed=5, keep=0.04)
    H, y, x = _inputs(oracle, 333, K=K, N=2 * K, seed=9)
    m = ctx.model(K, 2 * K, 8 * K, 2 * K, params, masks=masks, frozen_prefix=2)
    assert m.path_name == "sparse-jit-fp32"
    ev = m.batch_evaluate(H, y, x, trainable_only=True)
    ref = oracle.batch_evaluate(_omodel(params, K=K, N=2 * K, masks=masks, frozen=2),
                                H.astype(np.float64), y.astype(np.float64),
                                x.astype(np.float64), trainable_only=True)
    assert ev.symbol_errors == ref["symbol_errors"]
    assert abs(ev.data_loss - ref["data_loss"]) <= 1e-4 * abs(ref["data_loss"])


def test_sparse_jit_same_model_twice_bit_identical(ctx, oracle):
    """Two models with the same weights share one compiled kernel (the cubin
    cache keyed by the generated source) and give the same bits."""
    K, L = 8, 4
    params, masks = _sparse_model(K, L, seed=21)
    H, y, x = _inputs(oracle, 512, K=K, N=2 * K, seed=4)
    a = ctx.model(K, 2 * K, 8 * K, 2 * K, params, masks=masks)
    b = ctx.model(K, 2 * K, 8 * K, 2 * K, params.copy(), masks=masks.copy())
    ea, xa = a.batch_evaluate(H, y, x, want_xhat=True)
    eb, xb = b.batch_evaluate(H, y, x, want_xhat=True)
    assert ea.data_loss == eb.data_loss and ea.symbol_errors == eb.symbol_errors
    assert np.array_equal(xa, xb)


def test_dense_model_on_sparse_path_runs_simt(ctx, oracle):
    """The sparse path only takes models whose every layer is sparse enough
    (at most 1,500 surviving products); a dense model asked for path 3 runs
    the FP32 SIMT kernel."""
    from paper_2003_09446_b200.workload import xavier_params
    K = 20
    params = xavier_params(K, 3, seed=9)
    m = ctx.model(K, 30, 160, 40, params)
    assert m.path_name == "simt-fp32"


_CACHE_SNIPPET = """
import sys, json, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from test_sparse_jit_gpu import _sparse_model
from test_parity_gpu import _inputs
from oracle.oracle import Oracle
from paper_2003_09446_b200 import Context
c = Context(0); c.set_path(3)
p, m = _sparse_model(8, 5, seed=77)
H, y, x = _inputs(Oracle(), 256, K=8, N=16, seed=2)
ev = c.model(8, 16, 64, 16, p, masks=m).batch_evaluate(H, y, x)
print(json.dumps([ev.data_loss, ev.symbol_errors]))
"""


def test_sparse_jit_disk_cache(tmp_path):
    """A second process with the same model loads the cubin the first one
    wrote ($DETNET_JIT_CACHE) and computes the same bits."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _CACHE_SNIPPET.format(root=root, tests=os.path.join(root, "tests"))
    env = dict(os.environ, DETNET_JIT_CACHE=str(tmp_path / "jit"))
    outs = []
    for _ in range(2):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
        files = [f for f in os.listdir(tmp_path / "jit") if f.endswith(".cubin")]
        assert len(files) == 1, files
    assert outs[0] == outs[1]


@pytest.mark.parametrize("n,L", [(1, 1), (129, 1), (5, 3)])
def test_sparse_jit_small_edges(ctx, oracle, n, L):
    """A single sample, one partial tile, depth 1 (loss 0 at L = 1,
    acceptance.cpp:326-339) on the generated kernel."""
    K = 8
    params, masks = _sparse_model(K, L, seed=31 + n)
    H, y, x = _inputs(oracle, n, K=K, N=2 * K, seed=6)
    m = ctx.model(K, 2 * K, 8 * K, 2 * K, params, masks=masks)
    assert m.path_name == "sparse-jit-fp32"
    ev, xh = m.batch_evaluate(H, y, x, want_xhat=True)
    ref = oracle.evaluate(_omodel(params, K=K, N=2 * K, masks=masks), H.astype(np.float64),
                          y.astype(np.float64), x.astype(np.float64), want_xhat=True)
    assert ev.symbol_errors == int(ref["errors"].sum())
    assert np.allclose(xh, ref["xhat"].reshape(xh.shape), rtol=1e-4, atol=1e-5)
    if L == 1:
        assert ev.data_loss == 0.0
