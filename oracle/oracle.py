"""TEST INFRASTRUCTURE ONLY -- ctypes access to the parity checkers.

* ``Oracle``  : the plain-C restatement (oracle/detnet_oracle.c), built into
  oracle/build/libdetnet_oracle.so. Kind "port".
* ``RefLib``  : the UNMODIFIED reference library compiled from
  /root/reference/proj/src (oracle/Makefile -> oracle/_ref/libunfold_ref.so)
  behind a thin extern "C" shim. Kind "reference".

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module. The product (paper_2003_09446_b200) never does.

Flat layouts follow oracle/detnet_oracle.h: samples H [n][N][K], y [n][N],
x [n][K]; params/masks/grads as L "layer records" (W1 b1 W2 b2 W3 b3 t).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libdetnet_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libunfold_ref.so")

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_longlong)
_ip = C.POINTER(C.c_int)


def _ptr(a, t=_dp):
    if a is None:
        return None
    return a.ctypes.data_as(t)


class _Model(C.Structure):
    _fields_ = [("n_tx", C.c_int), ("n_rx", C.c_int), ("z_dim", C.c_int), ("v_dim", C.c_int),
                ("depth", C.c_int), ("frozen_prefix", C.c_int), ("params", _dp), ("masks", _dp)]


class _LossSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("lam", C.c_double), ("lam1", C.c_double), ("lam2", C.c_double)]


class _AdamCfg(C.Structure):
    _fields_ = [("lr0", C.c_double), ("decay_factor", C.c_double), ("decay_step", C.c_int),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


class _Rng(C.Structure):
    _fields_ = [("s", C.c_uint64)]


def record_size(K, Z, V):
    IN = 3 * K + V
    return Z * IN + Z + K * Z + K + V * Z + V + 1


def record_slices(K, Z, V):
    """Offsets of W1 b1 W2 b2 W3 b3 t inside one layer record."""
    IN = 3 * K + V
    out, off = {}, 0
    for name, size in (("W1", Z * IN), ("b1", Z), ("W2", K * Z), ("b2", K), ("W3", V * Z),
                       ("b3", V), ("t", 1)):
        out[name] = slice(off, off + size)
        off += size
    return out


@dataclass
class Model:
    """DetNet parameters in the flat layer-record layout (FP64 values)."""
    n_tx: int
    n_rx: int
    z_dim: int
    v_dim: int
    depth: int
    params: np.ndarray            # [depth, P] float64
    masks: np.ndarray | None = None
    frozen_prefix: int = 0

    @property
    def in_dim(self):
        return 3 * self.n_tx + self.v_dim

    def c(self):
        self._keep = (np.ascontiguousarray(self.params, np.float64),
                      None if self.masks is None else np.ascontiguousarray(self.masks, np.float64))
        return _Model(self.n_tx, self.n_rx, self.z_dim, self.v_dim, self.depth, self.frozen_prefix,
                      _ptr(self._keep[0]), _ptr(self._keep[1]))


def _spec(kind=0, lam=0.0, lam1=0.0, lam2=0.0):
    return _LossSpec(kind, lam, lam1, lam2)


class Oracle:
    """The plain-C restatement (port)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        L.or_mix64.restype = C.c_uint64
        L.or_mix64.argtypes = [C.c_uint64]
        L.or_rng_new.restype = _Rng
        L.or_rng_new.argtypes = [C.c_uint64, C.c_uint64]
        L.or_next_u64.restype = C.c_uint64
        L.or_next_u64.argtypes = [C.POINTER(_Rng)]
        L.or_next_uniform.restype = C.c_double
        L.or_next_uniform.argtypes = [C.POINTER(_Rng)]
        L.or_next_gaussian.restype = C.c_double
        L.or_next_gaussian.argtypes = [C.POINTER(_Rng)]
        L.or_stream.restype = _Rng
        L.or_stream.argtypes = [C.POINTER(_Rng), C.c_uint64]
        L.or_split.restype = _Rng
        L.or_split.argtypes = [C.POINTER(_Rng)]
        L.or_generate_batch.argtypes = [C.POINTER(_Rng), C.c_int, C.c_int, C.c_long, C.c_long,
                                        C.c_double, C.c_double, _dp, _dp, _dp, _dp]
        L.or_generate_range.argtypes = [C.POINTER(_Rng), C.c_int, C.c_int, C.c_long, C.c_long,
                                        C.c_double, C.c_double, _dp, _dp, _dp, _dp]
        L.or_preprocess.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.or_layer.argtypes = [C.POINTER(_Model), C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                               _dp, _dp, _dp]
        L.or_evaluate.argtypes = [C.POINTER(_Model), C.c_long, _dp, _dp, _dp, C.c_int, _dp, _lp,
                                  _ip, _dp, C.POINTER(C.c_long)]
        L.or_batch_evaluate.argtypes = [C.POINTER(_Model), C.c_long, _dp, _dp, _dp, C.c_int, _dp,
                                        _lp, _lp, _lp]
        L.or_evaluate_f32.argtypes = [C.POINTER(_Model), C.c_long, _dp, _dp, _dp, C.c_int, _dp,
                                      _lp, _dp]
        L.or_batch_gradient.argtypes = [C.POINTER(_Model), C.c_long, _dp, _dp, _dp,
                                        C.POINTER(_LossSpec), C.c_int, _dp, _dp, _lp, _lp, _lp]
        L.or_batch_gradient_f32.argtypes = L.or_batch_gradient.argtypes
        L.or_regularizer.restype = C.c_double
        L.or_regularizer.argtypes = [C.POINTER(_Model), C.POINTER(_LossSpec)]
        L.or_adam_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp,
                                   _dp, _dp, C.POINTER(C.c_int64), C.POINTER(_AdamCfg)]
        L.or_flops_per_detection.restype = C.c_longlong
        L.or_flops_per_detection.argtypes = [C.POINTER(_Model), C.c_int]

    # -- rng / inputs --------------------------------------------------
    def rng(self, seed, stream=0):
        return self.lib.or_rng_new(seed, stream)

    def draws(self, seed, stream, n, kind="u64"):
        r = self.rng(seed, stream)
        f = {"u64": self.lib.or_next_u64, "uniform": self.lib.or_next_uniform,
             "gaussian": self.lib.or_next_gaussian}[kind]
        return [f(C.byref(r)) for _ in range(n)]

    def generate_batch(self, rng, n_rx, n_tx, count, lo, hi, first=0):
        """generate_batch(rng, ...) -> (H, x, y, sigma2); advances rng by one draw."""
        H = np.empty((count, n_rx, n_tx)); x = np.empty((count, n_tx)); y = np.empty((count, n_rx))
        s2 = np.empty(count)
        self.lib.or_generate_batch(C.byref(rng), n_rx, n_tx, first, count, lo, hi, _ptr(H), _ptr(x),
                                   _ptr(y), _ptr(s2))
        return H, x, y, s2

    def generate_range(self, base, n_rx, n_tx, first, count, lo, hi):
        H = np.empty((count, n_rx, n_tx)); x = np.empty((count, n_tx)); y = np.empty((count, n_rx))
        s2 = np.empty(count)
        self.lib.or_generate_range(C.byref(base), n_rx, n_tx, first, count, lo, hi, _ptr(H), _ptr(x),
                                   _ptr(y), _ptr(s2))
        return H, x, y, s2

    # -- forward ------------------------------------------------------
    def preprocess(self, H, y):
        N, K = H.shape
        q = np.empty(K); G = np.empty((K, K)); xt = np.empty(K)
        st = self.lib.or_preprocess(N, K, _ptr(np.ascontiguousarray(H)), _ptr(np.ascontiguousarray(y)),
                                    _ptr(q), _ptr(G), _ptr(xt))
        return st, q, G, xt

    def layer(self, m: Model, l, q, G, xh, v):
        cm = m.c()
        K, Z, V = m.n_tx, m.z_dim, m.v_dim
        xo = np.empty(K); vo = np.empty(V); ino = np.empty(m.in_dim); u1 = np.empty(Z)
        zo = np.empty(Z); u2 = np.empty(K)
        args = [np.ascontiguousarray(a, np.float64) for a in (q, G, xh, v)]
        self.lib.or_layer(C.byref(cm), l, *[_ptr(a) for a in args], _ptr(xo), _ptr(vo), _ptr(ino),
                          _ptr(u1), _ptr(zo), _ptr(u2))
        return xo, vo, dict(in_=ino, u1=u1, z=zo, u2=u2)

    def evaluate(self, m: Model, H, y, x, first_term=1, want_xhat=False):
        n = H.shape[0]
        cm = m.c()
        loss = np.empty(n); err = np.empty(n, np.int64); flag = np.empty(n, np.int32)
        xh = np.empty((n, m.depth, m.n_tx)) if want_xhat else None
        bad = C.c_long(-1)
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        st = self.lib.or_evaluate(C.byref(cm), n, _ptr(H), _ptr(y), _ptr(x), first_term, _ptr(loss),
                                  _ptr(err, _lp), _ptr(flag, _ip), _ptr(xh), C.byref(bad))
        return dict(status=st, loss=loss, errors=err, flagged=flag, xhat=xh, bad=bad.value)

    def evaluate_f32(self, m: Model, H, y, x, first_term=1, want_xhat=True):
        n = H.shape[0]
        cm = m.c()
        loss = np.empty(n); err = np.empty(n, np.int64)
        xh = np.empty((n, m.depth, m.n_tx)) if want_xhat else None
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        st = self.lib.or_evaluate_f32(C.byref(cm), n, _ptr(H), _ptr(y), _ptr(x), first_term,
                                      _ptr(loss), _ptr(err, _lp), _ptr(xh))
        return dict(status=st, loss=loss, errors=err, xhat=xh)

    def batch_evaluate(self, m: Model, H, y, x, trainable_only=False):
        cm = m.c()
        dl = C.c_double(); e = C.c_longlong(); s = C.c_longlong(); f = C.c_longlong()
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        st = self.lib.or_batch_evaluate(C.byref(cm), H.shape[0], _ptr(H), _ptr(y), _ptr(x),
                                        int(trainable_only), C.byref(dl), C.byref(e), C.byref(s),
                                        C.byref(f))
        return dict(status=st, data_loss=dl.value, symbol_errors=e.value, symbols=s.value,
                    flagged=f.value)

    # -- training -----------------------------------------------------
    def batch_gradient(self, m: Model, H, y, x, kind=0, lam=0.0, lam1=0.0, lam2=0.0,
                       trainable_only=False):
        cm = m.c()
        sp = _spec(kind, lam, lam1, lam2)
        g = np.zeros_like(m.params)
        dl = C.c_double(); e = C.c_longlong(); s = C.c_longlong(); f = C.c_longlong()
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        st = self.lib.or_batch_gradient(C.byref(cm), H.shape[0], _ptr(H), _ptr(y), _ptr(x),
                                        C.byref(sp), int(trainable_only), _ptr(g), C.byref(dl),
                                        C.byref(e), C.byref(s), C.byref(f))
        return dict(status=st, grads=g, data_loss=dl.value, symbol_errors=e.value,
                    symbols=s.value, flagged=f.value)

    def batch_gradient_f32(self, m: Model, H, y, x, kind=0, lam=0.0, lam1=0.0, lam2=0.0,
                           trainable_only=False):
        """O32: the FP32 restatement of batch_gradient (FP32's own spread)."""
        cm = m.c()
        sp = _spec(kind, lam, lam1, lam2)
        g = np.zeros_like(m.params)
        dl = C.c_double(); e = C.c_longlong(); s = C.c_longlong(); f = C.c_longlong()
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        st = self.lib.or_batch_gradient_f32(C.byref(cm), H.shape[0], _ptr(H), _ptr(y), _ptr(x),
                                            C.byref(sp), int(trainable_only), _ptr(g), C.byref(dl),
                                            C.byref(e), C.byref(s), C.byref(f))
        return dict(status=st, grads=g, data_loss=dl.value, symbol_errors=e.value,
                    symbols=s.value, flagged=f.value)

    def regularizer(self, m: Model, kind=0, lam=0.0, lam1=0.0, lam2=0.0):
        cm = m.c()
        sp = _spec(kind, lam, lam1, lam2)
        return self.lib.or_regularizer(C.byref(cm), C.byref(sp))

    def adam_step(self, m: Model, grads, mom1, mom2, step, lr0=1e-4, decay=0.97, decay_step=1000,
                  b1=0.9, b2=0.999, eps=1e-8):
        """In-place on m.params, mom1, mom2; returns the new step."""
        cfg = _AdamCfg(lr0, decay, decay_step, b1, b2, eps)
        st = C.c_int64(step)
        masks = None if m.masks is None else np.ascontiguousarray(m.masks)
        self.lib.or_adam_step(m.n_tx, m.z_dim, m.v_dim, m.depth, m.frozen_prefix, _ptr(m.params),
                              _ptr(masks), _ptr(np.ascontiguousarray(grads)), _ptr(mom1),
                              _ptr(mom2), C.byref(st), C.byref(cfg))
        return st.value

    def flops_per_detection(self, m: Model, include_preprocess=True):
        cm = m.c()
        return self.lib.or_flops_per_detection(C.byref(cm), int(include_preprocess))


class RefLib:
    """The reference library itself (compiled, unmodified, namespace unfold_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_new.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_free.argtypes = [C.c_void_p]
        for name in ("ref_rng_stream",):
            getattr(L, name).restype = C.c_void_p
            getattr(L, name).argtypes = [C.c_void_p, C.c_uint64]
        L.ref_rng_split.restype = C.c_void_p
        L.ref_rng_split.argtypes = [C.c_void_p]
        for name, rt in (("ref_rng_next_u64", C.c_uint64), ("ref_rng_next_uniform", C.c_double),
                         ("ref_rng_next_gaussian", C.c_double), ("ref_rng_state", C.c_uint64),
                         ("ref_rng_next_bit", C.c_int)):
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [C.c_void_p]
        L.ref_generate_batch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.c_double, _dp, _dp, _dp, _dp, C.c_int]
        L.ref_batch_evaluate.argtypes = [C.POINTER(_Model), C.c_long, _dp, _dp, _dp, C.c_int,
                                         C.c_int, _dp, _lp]
        L.ref_forward.argtypes = [C.POINTER(_Model), _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_zf_decode.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_prune.argtypes = [C.POINTER(_Model), C.c_int, C.c_double, C.c_double, C.c_double, _dp]
        L.ref_cost_report.argtypes = [C.POINTER(_Model), _lp, _lp]
        L.ref_baseline_errors.argtypes = [C.c_int, C.c_long, C.c_int, C.c_int, _dp, _dp, _dp,
                                          C.c_int, _lp, _lp]
        L.ref_batch_gradient.argtypes = [C.POINTER(_Model), C.c_long, _dp, _dp, _dp,
                                         C.POINTER(_LossSpec), C.c_int, C.c_int, _dp, _dp, _lp]
        L.ref_regularizer.restype = C.c_double
        L.ref_regularizer.argtypes = [C.POINTER(_Model), C.POINTER(_LossSpec)]
        L.ref_flops_per_detection.restype = C.c_longlong
        L.ref_flops_per_detection.argtypes = [C.POINTER(_Model), C.c_int]
        L.ref_adam_step.argtypes = [C.POINTER(_Model), _dp, _dp, _dp, _dp, C.POINTER(C.c_int64),
                                    C.POINTER(_AdamCfg)]

    def worker_count(self):
        return self.lib.ref_worker_count()

    def _check(self, st):
        if st:
            raise RuntimeError(f"reference status {st}: {self.lib.ref_last_error().decode()}")

    def draws(self, seed, stream, n, kind="u64"):
        r = self.lib.ref_rng_new(seed, stream)
        f = {"u64": self.lib.ref_rng_next_u64, "uniform": self.lib.ref_rng_next_uniform,
             "gaussian": self.lib.ref_rng_next_gaussian}[kind]
        out = [f(r) for _ in range(n)]
        self.lib.ref_rng_free(r)
        return out

    def generate_batch(self, rng, n_rx, n_tx, count, lo, hi, parallel=True):
        H = np.empty((count, n_rx, n_tx)); x = np.empty((count, n_tx)); y = np.empty((count, n_rx))
        s2 = np.empty(count)
        self._check(self.lib.ref_generate_batch(rng, n_rx, n_tx, count, lo, hi, _ptr(H), _ptr(x),
                                                _ptr(y), _ptr(s2), int(parallel)))
        return H, x, y, s2

    def batch_evaluate(self, m: Model, H, y, x, trainable_only=False, parallel=True):
        cm = m.c()
        dl = C.c_double()
        o3 = np.zeros(3, np.int64)
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        st = self.lib.ref_batch_evaluate(C.byref(cm), H.shape[0], _ptr(H), _ptr(y), _ptr(x),
                                         int(trainable_only), int(parallel), C.byref(dl),
                                         _ptr(o3, _lp))
        return dict(status=st, data_loss=dl.value, symbol_errors=int(o3[0]), symbols=int(o3[1]),
                    flagged=int(o3[2]))

    def prune(self, m: Model, kind, eta=0.0, eta1=0.0, eta2=0.0):
        """prune (compression.cpp:87-94); returns the masks in record layout."""
        cm = m.c()
        out = np.zeros((m.depth, record_size(m.n_tx, m.z_dim, m.v_dim)))
        self._check(self.lib.ref_prune(C.byref(cm), kind, eta, eta1, eta2, _ptr(out)))
        return out

    def cost_report(self, m: Model):
        cm = m.c()
        o8 = np.zeros(8, np.int64)
        pl = np.zeros((m.depth, 3), np.int64)
        self._check(self.lib.ref_cost_report(C.byref(cm), _ptr(o8, _lp), _ptr(pl, _lp)))
        keys = ("layer_count", "params_total", "params_nonzero", "memory_dense_bytes",
                "memory_sparse_bytes", "flops", "flops_dense", "preprocess_flops")
        return dict(zip(keys, map(int, o8))), pl

    def baseline_errors(self, kind, H, y, x, parallel=True):
        """batch_baseline_errors (kernels.cpp:202-223): kind 0 zf, 1 ml, 2 oracle.
        Returns (status, errors, symbols)."""
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        e, s = C.c_longlong(), C.c_longlong()
        st = self.lib.ref_baseline_errors(kind, H.shape[0], H.shape[1], H.shape[2], _ptr(H), _ptr(y),
                                          _ptr(x), int(parallel), C.byref(e), C.byref(s))
        return st, e.value, s.value

    def forward(self, m: Model, H, y):
        cm = m.c()
        K, V, Z, L = m.n_tx, m.v_dim, m.z_dim, m.depth
        xh = np.empty((L + 1, K)); v = np.empty((L + 1, V)); ino = np.empty((L, m.in_dim))
        u1 = np.empty((L, Z)); z = np.empty((L, Z)); u2 = np.empty((L, K))
        self._check(self.lib.ref_forward(C.byref(cm), _ptr(np.ascontiguousarray(H, np.float64)),
                                         _ptr(np.ascontiguousarray(y, np.float64)), _ptr(xh),
                                         _ptr(v), _ptr(ino), _ptr(u1), _ptr(z), _ptr(u2)))
        return dict(x_hat=xh, v=v, in_=ino, u1=u1, z=z, u2=u2)

    def zf_decode(self, H, y):
        N, K = H.shape
        out = np.empty(K)
        self._check(self.lib.ref_zf_decode(N, K, _ptr(np.ascontiguousarray(H, np.float64)),
                                           _ptr(np.ascontiguousarray(y, np.float64)), _ptr(out)))
        return out

    def batch_gradient(self, m: Model, H, y, x, kind=0, lam=0.0, lam1=0.0, lam2=0.0,
                       trainable_only=False, parallel=True):
        cm = m.c()
        sp = _spec(kind, lam, lam1, lam2)
        g = np.zeros_like(m.params)
        dl = C.c_double()
        o3 = np.zeros(3, np.int64)
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        st = self.lib.ref_batch_gradient(C.byref(cm), H.shape[0], _ptr(H), _ptr(y), _ptr(x),
                                         C.byref(sp), int(trainable_only), int(parallel), _ptr(g),
                                         C.byref(dl), _ptr(o3, _lp))
        return dict(status=st, grads=g, data_loss=dl.value, symbol_errors=int(o3[0]),
                    symbols=int(o3[1]), flagged=int(o3[2]))

    def regularizer(self, m: Model, kind=0, lam=0.0, lam1=0.0, lam2=0.0):
        cm = m.c()
        sp = _spec(kind, lam, lam1, lam2)
        return self.lib.ref_regularizer(C.byref(cm), C.byref(sp))

    def flops_per_detection(self, m: Model, include_preprocess=True):
        cm = m.c()
        return self.lib.ref_flops_per_detection(C.byref(cm), int(include_preprocess))

    def adam_step(self, m: Model, grads, mom1, mom2, step, lr0=1e-4, decay=0.97, decay_step=1000,
                  b1=0.9, b2=0.999, eps=1e-8):
        cm = m.c()
        cfg = _AdamCfg(lr0, decay, decay_step, b1, b2, eps)
        st = C.c_int64(step)
        self._check(self.lib.ref_adam_step(C.byref(cm), _ptr(m.params),
                                           _ptr(np.ascontiguousarray(grads)), _ptr(mom1),
                                           _ptr(mom2), C.byref(st), C.byref(cfg)))
        return st.value


def available_ref():
    return os.path.exists(REF_SO)


# ---------------------------------------------------------------------------
# Workload builders shared by tests and the CPU-baseline legs.
# ---------------------------------------------------------------------------

def xavier_model(oracle: Oracle, n_tx=20, n_rx=30, depth=40, seed=9, z_dim=None, v_dim=None,
                 t0=0.5):
    """Xavier-uniform weights drawn with the reference Rng(seed), rounded to
    FP32 (stored as float64), zero biases, t = t0."""
    Z = z_dim or 8 * n_tx
    V = v_dim or 2 * n_tx
    K = n_tx
    IN = 3 * K + V
    P = record_size(K, Z, V)
    sl = record_slices(K, Z, V)
    r = oracle.rng(seed, 0)
    params = np.zeros((depth, P))
    for l in range(depth):
        for name, (rows, cols) in (("W1", (Z, IN)), ("W2", (K, Z)), ("W3", (V, Z))):
            a = (6.0 / (rows + cols)) ** 0.5
            vals = np.array([oracle.lib.or_next_uniform(C.byref(r)) for _ in range(rows * cols)])
            params[l, sl[name]] = (-a + (a - -a) * vals)
        params[l, sl["t"]] = t0
    params = params.astype(np.float32).astype(np.float64)
    return Model(K, n_rx, Z, V, depth, params)


def scaled_inputs(H, y, x):
    """Round the reference samples to FP32 after scaling H and y by 1/sqrt(N)
    (BASELINE.json's H ~ N(0, 1/N))."""
    N = H.shape[1]
    s = 1.0 / np.sqrt(N)
    H32 = (H * s).astype(np.float32)
    y32 = (y * s).astype(np.float32)
    x8 = x.astype(np.int8)
    return H32, y32, x8
