"""ctypes binding of the C-ABI (include/detnet_b200.h), mirroring the
reference's batch-kernel API (proj/include/unfold/kernels.hpp:29-65):

    ctx = Context(device=0)
    model = ctx.model(n_tx, n_rx, z_dim, v_dim, params, masks=None, frozen_prefix=0)
    ev = model.batch_evaluate(H, y, x)          # -> BatchEval
    model.batch_gradient(H, y, x, spec)          # -> (BatchEval, grads)

Errors map to the reference's exception taxonomy (errors.hpp:9-31). There is
no CPU fallback: constructing a Context without a B200 raises CudaError, and a
missing shared library raises ImportError at import time.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# DETNET_LIB: developer override (A/B runs of kernel variants built with
# `make OUT=... OBJDIR=... EXTRA=-D...`); the product loads the in-tree build.
LIB_PATH = os.environ.get("DETNET_LIB") or os.path.join(HERE, "lib", "libdetnet_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `make -C paper_2003_09446_b200/csrc` "
                      "(or __graft_entry__.build())")
_lib = C.CDLL(LIB_PATH)

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_bp = C.POINTER(C.c_int8)
_vp = C.c_void_p


# --- exception taxonomy (errors.hpp:9-31) -----------------------------------
class DetnetError(RuntimeError):
    pass


class ContractError(DetnetError, ValueError):
    pass


class SingularMatrixError(DetnetError):
    pass


class ConfigError(DetnetError):
    pass


class CudaError(DetnetError):
    pass


class UnsupportedError(DetnetError):
    pass


class DivergenceError(DetnetError):
    """Non-finite training objective (training.cpp:68-70)."""


_ERRS = {1: ContractError, 2: SingularMatrixError, 3: ConfigError, 4: CudaError, 5: CudaError,
         6: UnsupportedError, 7: DivergenceError}


def _check(rc):
    if rc:
        msg = _lib.detnet_last_error().decode()
        raise _ERRS.get(rc, DetnetError)(msg)


class _ModelDesc(C.Structure):
    _fields_ = [("n_tx", C.c_int), ("n_rx", C.c_int), ("z_dim", C.c_int), ("v_dim", C.c_int),
                ("depth", C.c_int), ("frozen_prefix", C.c_int), ("params", _dp), ("masks", _dp)]


class _Eval(C.Structure):
    _fields_ = [("data_loss", C.c_double), ("loss_sum", C.c_double),
                ("symbol_errors", C.c_longlong), ("symbols", C.c_longlong),
                ("flagged", C.c_longlong)]


class _Times(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_longlong * 8)]


class _LossSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("lam", C.c_double), ("lam1", C.c_double), ("lam2", C.c_double)]


class _AdamCfg(C.Structure):
    _fields_ = [("lr0", C.c_double), ("decay_factor", C.c_double), ("decay_step", C.c_int),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


class _IncCfg(C.Structure):
    _fields_ = [("start_layers", C.c_int), ("t_step", C.c_int), ("max_layers", C.c_int),
                ("halt_epsilon", C.c_double), ("target_ber", C.c_double),
                ("val_samples", C.c_int), ("val_snr_db", C.c_double),
                ("total_batches", C.c_int), ("batch_size", C.c_int),
                ("snr_lo_db", C.c_double), ("snr_hi_db", C.c_double), ("adam", _AdamCfg),
                ("spec", _LossSpec), ("weight_scale", C.c_double), ("t0", C.c_double),
                ("loss_layers_trainable_only", C.c_int), ("seed", C.c_uint64),
                ("sample_scale", C.c_double)]


class _StepRec(C.Structure):
    _fields_ = [("step", C.c_int), ("layer_count", C.c_int), ("train_loss", C.c_double),
                ("val_loss", C.c_double), ("val_ber", C.c_double), ("wall_ms", C.c_double)]


class _IncRes(C.Structure):
    _fields_ = [("halt_reason", C.c_int), ("depth", C.c_int), ("frozen_prefix", C.c_int),
                ("flagged_samples", C.c_longlong), ("optimizer_steps", C.c_longlong),
                ("seconds", C.c_double)]


_lib.detnet_last_error.restype = C.c_char_p
_lib.detnet_ctx_create.argtypes = [C.c_int, C.POINTER(_vp)]
_lib.detnet_ctx_create_group.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(_vp)]
_lib.detnet_ctx_group_size.argtypes = [_vp]
_lib.detnet_ctx_destroy.argtypes = [_vp]
_lib.detnet_ctx_set_path.argtypes = [_vp, C.c_int]
_lib.detnet_ctx_set_stream.argtypes = [_vp, _vp]
_lib.detnet_ctx_set_exact_preprocess.argtypes = [_vp, C.c_int]
_lib.detnet_ctx_stream.restype = _vp
_lib.detnet_ctx_stream.argtypes = [_vp]
_lib.detnet_ctx_set_profiling.argtypes = [_vp, C.c_int]
_lib.detnet_ctx_kernel_times.argtypes = [_vp, C.POINTER(_Times), C.c_int]
_lib.detnet_ctx_launch_count.restype = C.c_longlong
_lib.detnet_ctx_launch_count.argtypes = [_vp]
_lib.detnet_record_size.restype = C.c_long
_lib.detnet_record_size.argtypes = [C.c_int, C.c_int, C.c_int]
_lib.detnet_model_create.argtypes = [_vp, C.POINTER(_ModelDesc), C.POINTER(_vp)]
_lib.detnet_model_update.argtypes = [_vp, C.POINTER(_ModelDesc)]
_lib.detnet_model_destroy.argtypes = [_vp]
_lib.detnet_model_path.argtypes = [_vp]
_lib.detnet_model_flops_per_detection.restype = C.c_longlong
_lib.detnet_model_flops_per_detection.argtypes = [_vp, C.c_int]
_lib.detnet_batch_evaluate.argtypes = [_vp, C.c_long, _vp, _vp, _vp, C.c_int, _vp,
                                       C.POINTER(_Eval)]
_lib.detnet_batch_evaluate_device_async.argtypes = [_vp, C.c_long, _vp, _vp, _vp, C.c_int, _vp,
                                                   C.POINTER(C.c_longlong)]
_lib.detnet_eval_wait.argtypes = [_vp, C.c_longlong, _vp]
_lib.detnet_preprocess_device.argtypes = [_vp, C.c_long, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.detnet_batch_evaluate_device.argtypes = [_vp, C.c_long, _vp, _vp, _vp, C.c_int, _vp,
                                              C.POINTER(_Eval)]
_lib.detnet_forward_range.argtypes = [_vp, C.c_long, _vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp]
_lib.detnet_batch_gradient.argtypes = [_vp, C.c_long, _vp, _vp, _vp, C.POINTER(_LossSpec), C.c_int,
                                       _vp, C.POINTER(_Eval)]
_lib.detnet_adam_step.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp,
                                  _vp, _vp, C.POINTER(C.c_int64), C.POINTER(_AdamCfg)]
_lib.detnet_model_param_count.restype = C.c_long
_lib.detnet_model_param_count.argtypes = [_vp]
_lib.detnet_train_grad.argtypes = [_vp, C.c_long, _vp, _vp, _vp, C.c_int, _vp, C.POINTER(_Eval)]
_lib.detnet_train_grad_buckets.argtypes = [_vp, C.c_long, _vp, _vp, _vp, C.c_int, _vp,
                                           C.POINTER(C.c_void_p), C.POINTER(C.c_long), C.c_int]
_lib.detnet_stream_wait_event.argtypes = [_vp, _vp]
_lib.detnet_train_apply.argtypes = [_vp, _vp, C.c_long, C.POINTER(_LossSpec), C.POINTER(_AdamCfg)]
_lib.detnet_model_get_params.argtypes = [_vp, _vp]
_lib.detnet_train_incremental.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(_IncCfg), C.POINTER(_StepRec), C.c_int,
                                          C.POINTER(C.c_int), _vp, C.POINTER(_IncRes)]
_lib.detnet_ctx_chunk_sums.restype = C.c_long
_lib.detnet_ctx_chunk_sums.argtypes = [_vp, _vp, C.c_long]
_lib.detnet_train_raw_count.restype = C.c_long
_lib.detnet_train_raw_count.argtypes = [_vp]
_lib.detnet_train_status.argtypes = [_vp, _dp, _dp]
_lib.detnet_ctx_set_train_precision.argtypes = [_vp, C.c_int]
_lib.detnet_model_reset_adam.argtypes = [_vp]
class _CostReport(C.Structure):
    _fields_ = [("layer_count", C.c_int)] + [(f, C.c_longlong) for f in (
        "params_total", "params_nonzero", "memory_dense_bytes", "memory_sparse_bytes", "flops",
        "flops_dense", "preprocess_flops")]


class _LayerCost(C.Structure):
    _fields_ = [("params_total", C.c_longlong), ("params_nonzero", C.c_longlong),
                ("flops", C.c_longlong)]


_lib.detnet_ctx_set_train_forward.argtypes = [_vp, C.c_int]
_lib.detnet_model_prune.argtypes = [_vp, C.c_int, C.c_double, C.c_double, C.c_double]
_lib.detnet_model_get_masks.argtypes = [_vp, _vp]
_lib.detnet_model_cost_report.argtypes = [_vp, C.POINTER(_CostReport), C.POINTER(_LayerCost)]
_lib.detnet_batch_baseline_errors.argtypes = [_vp, C.c_int, C.c_long, C.c_int, C.c_int, _vp, _vp,
                                               _vp, C.POINTER(C.c_longlong),
                                               C.POINTER(C.c_longlong)]
_lib.detnet_generate_host.argtypes = [_vp, C.c_uint64, C.c_long, C.c_long, C.c_int, C.c_int,
                                      C.c_double, C.c_double, _vp, _vp, _vp, _vp]
_lib.detnet_rng_seed.restype = C.c_uint64
_lib.detnet_rng_seed.argtypes = [C.c_uint64, C.c_uint64]
_lib.detnet_rng_stream.restype = C.c_uint64
_lib.detnet_rng_stream.argtypes = [C.c_uint64, C.c_uint64]
_lib.detnet_rng_split.restype = C.c_uint64
_lib.detnet_rng_split.argtypes = [C.POINTER(C.c_uint64)]
_lib.detnet_generate_device.argtypes = [_vp, C.c_uint64, C.c_long, C.c_long, C.c_int, C.c_int,
                                        C.c_double, C.c_double, C.c_double, _vp, _vp, _vp, _vp]

EXPORTED = [n for n in dir(_lib) if n.startswith("detnet_")]


def lib_path():
    return LIB_PATH


@dataclass
class BatchEval:
    """unfold::BatchEval (kernels.hpp:16-25)."""
    data_loss: float
    symbol_errors: int
    symbols: int
    flagged: int
    loss_sum: float = 0.0

    def ber(self):
        return self.symbol_errors / self.symbols if self.symbols else 0.0


def _addr(a):
    """Data pointer of a numpy array, a torch tensor, or a raw int address."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


PATH_AUTO, PATH_SIMT, PATH_TC, PATH_SPARSE = 0, 1, 2, 3


class _Ordered:
    """Orders the context stream after torch's current stream on entry and
    torch's current stream after the context stream on exit, so device
    buffers the caller produced (or reuses) with torch ops never race the
    engine (the C-ABI only orders work on its own stream; a context created
    here launches on its own non-blocking stream). A no-op when torch is not
    in use or both are the same stream."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.pair = None

    def __enter__(self):
        import sys
        torch = sys.modules.get("torch")
        if torch is None or not torch.cuda.is_available() or not torch.cuda.is_initialized():
            return self
        dev = torch.device("cuda", self.ctx.device)
        cur = torch.cuda.current_stream(dev)
        own = self.ctx.stream
        if not own or cur.cuda_stream == own:
            return self
        ext = torch.cuda.ExternalStream(own, device=dev)
        ext.wait_stream(cur)
        self.pair = (ext, cur)
        return self

    def __exit__(self, *exc):
        if self.pair:
            self.pair[1].wait_stream(self.pair[0])
        return False


class Context:
    """One CUDA device (detnet_ctx). Single-owner, like unfold::Rng."""

    def __init__(self, device=0, path=PATH_AUTO, devices=None):
        """devices: a list of device ids -> a device group (detnet_ctx_create_group):
        host-buffer batch_evaluate / batch_gradient shard over all of them with
        results bit-identical to one device. A device may repeat."""
        h = _vp()
        if devices is not None:
            arr = (C.c_int * len(devices))(*devices)
            _check(_lib.detnet_ctx_create_group(arr, len(devices), C.byref(h)))
            device = devices[0]
        else:
            _check(_lib.detnet_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self.set_path(path)

    @property
    def group_size(self):
        return _lib.detnet_ctx_group_size(self._h)

    def close(self):
        if getattr(self, "_h", None):
            _lib.detnet_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_path(self, path):
        _check(_lib.detnet_ctx_set_path(self._h, path))

    def set_exact_preprocess(self, on=True):
        _check(_lib.detnet_ctx_set_exact_preprocess(self._h, int(on)))

    def set_train_forward(self, tensor_cores=True):
        """Training forward on tcgen05 (dense K=20 models) instead of FP32 SIMT."""
        _check(_lib.detnet_ctx_set_train_forward(self._h, int(tensor_cores)))

    def set_train_precision(self, fp64=True):
        """FP64 training in the reference's operation order (bit-identical
        batch_gradient / adam_step) instead of the FP32 default."""
        _check(_lib.detnet_ctx_set_train_precision(self._h, int(fp64)))

    def set_stream(self, stream_ptr):
        _check(_lib.detnet_ctx_set_stream(self._h, stream_ptr))

    @property
    def stream(self):
        return _lib.detnet_ctx_stream(self._h)

    def eval_wait(self, ticket):
        """BatchEval of an evaluation enqueued by Model.batch_evaluate_device_async."""
        ev = _Eval()
        _check(_lib.detnet_eval_wait(self._h, ticket, C.byref(ev)))
        return BatchEval(ev.data_loss, ev.symbol_errors, ev.symbols, ev.flagged, ev.loss_sum)

    def set_profiling(self, on=True):
        _check(_lib.detnet_ctx_set_profiling(self._h, int(on)))

    def kernel_times(self, reset=False):
        t = _Times()
        _check(_lib.detnet_ctx_kernel_times(self._h, C.byref(t), int(reset)))
        names = ["generate", "preprocess", "stack", "reduce", "backward", "adam", "other", "x"]
        return {n: (t.ms[i], t.launches[i]) for i, n in enumerate(names)}

    @property
    def launch_count(self):
        return _lib.detnet_ctx_launch_count(self._h)

    def train_incremental(self, n_tx, n_rx, start_layers, t_step, max_layers, total_batches,
                          batch_size, val_samples, seed, z_dim=None, v_dim=None, halt_epsilon=0.01,
                          target_ber=0.0, val_snr_db=12.0, snr_lo_db=0.0, snr_hi_db=15.0,
                          lr0=1e-4, decay_factor=0.97, decay_step=1000, beta1=0.9, beta2=0.999,
                          eps=1e-8, kind=0, lam=0.0, lam1=0.0, lam2=0.0, weight_scale=1.0, t0=0.5,
                          trainable_only=False, sample_scale=1.0):
        """train_incremental (training.cpp:22-141) on the device. Returns
        (records, result dict, final params [depth][record])."""
        Z = z_dim or 8 * n_tx
        V = v_dim or 2 * n_tx
        cfg = _IncCfg(start_layers, t_step, max_layers, halt_epsilon, target_ber, val_samples,
                      val_snr_db, total_batches, batch_size, snr_lo_db, snr_hi_db,
                      _AdamCfg(lr0, decay_factor, decay_step, beta1, beta2, eps),
                      _LossSpec(kind, lam, lam1, lam2), weight_scale, t0, int(trainable_only),
                      seed, sample_scale)
        nmax = max_layers - start_layers + 2
        recs = (_StepRec * nmax)()
        nrec = C.c_int()
        res = _IncRes()
        P = record_size(n_tx, Z, V)
        params = np.zeros((max_layers, P))
        _check(_lib.detnet_train_incremental(self._h, n_tx, n_rx, Z, V, C.byref(cfg), recs, nmax,
                                             C.byref(nrec), params.ctypes.data, C.byref(res)))
        records = [{"step": r.step, "layers": r.layer_count, "train_loss": r.train_loss,
                    "val_loss": r.val_loss, "val_ber": r.val_ber, "wall_ms": r.wall_ms}
                   for r in recs[:nrec.value]]
        result = {"halt": ["target_ber", "converged", "max_layers"][res.halt_reason],
                  "depth": res.depth, "frozen_prefix": res.frozen_prefix,
                  "flagged": res.flagged_samples, "optimizer_steps": res.optimizer_steps,
                  "seconds": res.seconds}
        return records, result, params[:res.depth]

    def chunk_sums(self):
        """Per-8,192-sample-chunk loss sums of the last reduction (float64)."""
        n = _lib.detnet_ctx_chunk_sums(self._h, None, 0)
        if n < 0:
            _check(-n)
        out = np.zeros(n)
        if n:
            _lib.detnet_ctx_chunk_sums(self._h, out.ctypes.data, n)
        return out

    def model(self, n_tx, n_rx, z_dim, v_dim, params, masks=None, frozen_prefix=0):
        return Model(self, n_tx, n_rx, z_dim, v_dim, params, masks, frozen_prefix)

    # -- on-device generator (generate_batch keying, kernels.cpp:116-136) --
    def generate(self, base_state, first, count, n_rx, n_tx, snr_lo, snr_hi, scale, H, y, x,
                 sigma2=None):
        with _Ordered(self):
            _check(_lib.detnet_generate_device(self._h, base_state, first, count, n_rx, n_tx,
                                               snr_lo, snr_hi, scale, _addr(H), _addr(y),
                                               _addr(x), _addr(sigma2)))

    def generate_host(self, base_state, first, count, n_rx, n_tx, snr_lo, snr_hi):
        """FP64 unscaled samples (what unfold::generate_batch returns)."""
        H = np.empty((count, n_rx, n_tx)); x = np.empty((count, n_tx)); y = np.empty((count, n_rx))
        s2 = np.empty(count)
        _check(_lib.detnet_generate_host(self._h, base_state, first, count, n_rx, n_tx, snr_lo,
                                         snr_hi, _addr(H), _addr(x), _addr(y), _addr(s2)))
        return H, x, y, s2

    def baseline_errors(self, kind, H, y, x):
        """Detector baselines (batch_baseline_errors, kernels.cpp:202-223) on the
        device: kind 0 = ZF, 1 = ML (K <= 16), 2 = oracle; FP64 host samples in
        the reference layout. Returns (errors, symbols)."""
        H, y, x = (np.ascontiguousarray(a, np.float64) for a in (H, y, x))
        e, s = C.c_longlong(), C.c_longlong()
        _check(_lib.detnet_batch_baseline_errors(self._h, int(kind), H.shape[0], H.shape[1],
                                                 H.shape[2], _addr(H), _addr(y), _addr(x),
                                                 C.byref(e), C.byref(s)))
        return e.value, s.value

    def adam_step(self, n_tx, z_dim, v_dim, depth, frozen_prefix, params, masks, grads, m1, m2,
                  step, lr0=1e-4, decay_factor=0.97, decay_step=1000, beta1=0.9, beta2=0.999,
                  eps=1e-8):
        cfg = _AdamCfg(lr0, decay_factor, decay_step, beta1, beta2, eps)
        st = C.c_int64(step)
        _check(_lib.detnet_adam_step(self._h, n_tx, z_dim, v_dim, depth, frozen_prefix,
                                     _addr(params), _addr(masks), _addr(grads), _addr(m1),
                                     _addr(m2), C.byref(st), C.byref(cfg)))
        return st.value


def stream_wait_event(stream, event):
    """Order `stream` (a cudaStream_t handle, e.g. torch's .cuda_stream) after
    `event` (a bucket event of Model.train_grad_buckets)."""
    _check(_lib.detnet_stream_wait_event(C.c_void_p(stream), C.c_void_p(event)))


def rng_seed(seed, stream_id=0):
    return _lib.detnet_rng_seed(seed, stream_id)


def rng_stream(state, stream_id):
    return _lib.detnet_rng_stream(state, stream_id)


def rng_split(state):
    """Rng::split(): returns (child_state, advanced_state)."""
    s = C.c_uint64(state)
    child = _lib.detnet_rng_split(C.byref(s))
    return child, s.value


def record_size(n_tx, z_dim, v_dim):
    return _lib.detnet_record_size(n_tx, z_dim, v_dim)


class Model:
    """Device-resident ModelParams (detnet_model)."""

    def __init__(self, ctx, n_tx, n_rx, z_dim, v_dim, params, masks=None, frozen_prefix=0):
        self.ctx = ctx
        self.n_tx, self.n_rx, self.z_dim, self.v_dim = n_tx, n_rx, z_dim, v_dim
        self.depth = int(np.asarray(params).shape[0])
        self.frozen_prefix = frozen_prefix
        h = _vp()
        d = self._desc(params, masks)
        _check(_lib.detnet_model_create(ctx._h, C.byref(d), C.byref(h)))
        self._h = h

    def _desc(self, params, masks):
        P = record_size(self.n_tx, self.z_dim, self.v_dim)
        p = np.ascontiguousarray(params, np.float64).reshape(-1, P)
        mk = None if masks is None else np.ascontiguousarray(masks, np.float64).reshape(-1, P)
        self._keep = (p, mk)
        self.depth = p.shape[0]
        return _ModelDesc(self.n_tx, self.n_rx, self.z_dim, self.v_dim, p.shape[0],
                          self.frozen_prefix, p.ctypes.data_as(_dp),
                          None if mk is None else mk.ctypes.data_as(_dp))

    def update(self, params, masks=None, frozen_prefix=None):
        if frozen_prefix is not None:
            self.frozen_prefix = frozen_prefix
        d = self._desc(params, masks)
        _check(_lib.detnet_model_update(self._h, C.byref(d)))

    def close(self):
        if getattr(self, "_h", None):
            _lib.detnet_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def path_name(self):
        return {1: "simt-fp32", 2: "tcgen05-3xtf32", 3: "sparse-csr-fp32",
                4: "tcgen05-split-fp16", 5: "sparse-jit-fp32"}[
            _lib.detnet_model_path(self._h)]

    def flops_per_detection(self, include_preprocess=True):
        return _lib.detnet_model_flops_per_detection(self._h, int(include_preprocess))

    @staticmethod
    def _samples(H, y, x):
        H = np.ascontiguousarray(H, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        x = np.ascontiguousarray(x, np.int8)
        return H, y, x

    def batch_evaluate(self, H, y, x, trainable_only=False, want_xhat=False):
        """batch_evaluate over host samples; returns BatchEval (and x_hat [n][L][K])."""
        H, y, x = self._samples(H, y, x)
        n = H.shape[0]
        xh = np.empty((n, self.depth, self.n_tx), np.float32) if want_xhat else None
        ev = _Eval()
        _check(_lib.detnet_batch_evaluate(self._h, n, _addr(H), _addr(y), _addr(x),
                                          int(trainable_only), _addr(xh), C.byref(ev)))
        out = BatchEval(ev.data_loss, ev.symbol_errors, ev.symbols, ev.flagged, ev.loss_sum)
        return (out, xh) if want_xhat else out

    def batch_evaluate_device(self, n, H_ptr, y_ptr, x_ptr, trainable_only=False, xhat_ptr=None):
        """Device-resident samples (torch tensors or raw device addresses)."""
        ev = _Eval()
        with _Ordered(self.ctx):
            _check(_lib.detnet_batch_evaluate_device(self._h, n, _addr(H_ptr), _addr(y_ptr),
                                                     _addr(x_ptr), int(trainable_only),
                                                     _addr(xhat_ptr), C.byref(ev)))
        return BatchEval(ev.data_loss, ev.symbol_errors, ev.symbols, ev.flagged, ev.loss_sum)

    def batch_evaluate_device_async(self, n, H_ptr, y_ptr, x_ptr, trainable_only=False,
                                    xhat_ptr=None):
        """Enqueue an evaluation of device-resident samples; returns a ticket
        for Context.eval_wait (up to 64 in flight)."""
        t = C.c_longlong()
        with _Ordered(self.ctx):
            _check(_lib.detnet_batch_evaluate_device_async(self._h, n, _addr(H_ptr), _addr(y_ptr),
                                                           _addr(x_ptr), int(trainable_only),
                                                           _addr(xhat_ptr), C.byref(t)))
        return t.value

    def preprocess_device(self, n, H_ptr, y_ptr, x_ptr, gram_ptr=None, q_ptr=None, denom_ptr=None,
                          flag_ptr=None):
        """K1 alone on device-resident samples: sample-major G upper triangle,
        q = H^T y, loss denominator and guard flag (any output may be None)."""
        with _Ordered(self.ctx):
            _check(_lib.detnet_preprocess_device(self._h, n, _addr(H_ptr), _addr(y_ptr),
                                                 _addr(x_ptr), _addr(gram_ptr), _addr(q_ptr),
                                                 _addr(denom_ptr), _addr(flag_ptr)))

    def forward_range(self, H, y, l_begin, l_end, x_state, v_state, want_xhat=True):
        """Layers [l_begin, l_end) from state (x_state [n][K], v_state [n][V])."""
        H, y, _ = self._samples(H, y, np.zeros((1,), np.int8))
        n = H.shape[0]
        xs = np.ascontiguousarray(x_state, np.float32).copy()
        vs = np.ascontiguousarray(v_state, np.float32).copy()
        xh = np.empty((n, l_end - l_begin, self.n_tx), np.float32) if want_xhat else None
        _check(_lib.detnet_forward_range(self._h, n, _addr(H), _addr(y), l_begin, l_end,
                                         _addr(xs), _addr(vs), _addr(xh)))
        return xs, vs, xh

    @property
    def param_count(self):
        return _lib.detnet_model_param_count(self._h)

    @property
    def raw_count(self):
        """Length of a detnet_train_grad raw buffer: the gradient sums plus
        this rank's data-loss sum (all-reduce the whole buffer)."""
        return _lib.detnet_train_raw_count(self._h)

    def new_raw(self):
        import torch
        return torch.zeros(self.raw_count, dtype=torch.float64,
                           device=torch.device("cuda", self.ctx.device))

    def train_status(self):
        """(objective, regularizer) of the last train_apply; raises
        DivergenceError if training halted on a non-finite objective."""
        o, r = C.c_double(), C.c_double()
        _check(_lib.detnet_train_status(self._h, C.byref(o), C.byref(r)))
        return o.value, r.value

    def train_grad(self, n, H_ptr, y_ptr, x_ptr, raw_ptr, trainable_only=False, want_eval=True):
        """Device-resident gradient sums (detnet_train_grad) into raw_ptr (FP64).
        want_eval=False: only enqueue (returns None, no host wait)."""
        ev = _Eval()
        with _Ordered(self.ctx):
            _check(_lib.detnet_train_grad(self._h, n, _addr(H_ptr), _addr(y_ptr), _addr(x_ptr),
                                          int(trainable_only), _addr(raw_ptr),
                                          C.byref(ev) if want_eval else None))
        if not want_eval:
            return None
        return BatchEval(ev.data_loss, ev.symbol_errors, ev.symbols, ev.flagged, ev.loss_sum)

    def train_grad_buckets(self, n, H_ptr, y_ptr, x_ptr, raw_ptr, trainable_only=False,
                           max_buckets=9):
        """detnet_train_grad_buckets: enqueue the gradient with the raw sums
        finalised bucket by bucket; returns [(event, lo, hi)] -- raw[lo:hi] is
        final once the event completes (wait with stream_wait_event)."""
        evs = (C.c_void_p * max_buckets)()
        rng = (C.c_long * (2 * max_buckets))()
        with _Ordered(self.ctx):
            nb = _lib.detnet_train_grad_buckets(self._h, n, _addr(H_ptr), _addr(y_ptr),
                                                _addr(x_ptr), int(trainable_only), _addr(raw_ptr),
                                                evs, rng, max_buckets)
        if nb < 0:
            _check(-nb)
        return [(evs[b], rng[2 * b], rng[2 * b + 1]) for b in range(nb)]

    def train_apply(self, raw_ptr, n_global, kind=0, lam=0.0, lam1=0.0, lam2=0.0, lr0=1e-4,
                    decay_factor=0.97, decay_step=1000, beta1=0.9, beta2=0.999, eps=1e-8):
        spec = _LossSpec(kind, lam, lam1, lam2)
        cfg = _AdamCfg(lr0, decay_factor, decay_step, beta1, beta2, eps)
        with _Ordered(self.ctx):
            _check(_lib.detnet_train_apply(self._h, _addr(raw_ptr), n_global, C.byref(spec),
                                           C.byref(cfg)))

    def get_params(self):
        out = np.empty((self.depth, record_size(self.n_tx, self.z_dim, self.v_dim)))
        _check(_lib.detnet_model_get_params(self._h, _addr(out)))
        return out

    def reset_adam(self):
        _check(_lib.detnet_model_reset_adam(self._h))

    # -- pruning planner (compression.cpp:43-94) and cost report (131-159) --
    def prune(self, kind, eta=0.0, eta1=0.0, eta2=0.0):
        """kind 0 element(eta), 1 group(eta1), 2 sparse_group(eta1, eta2), on the
        device master weights; the packed layouts are rebuilt."""
        _check(_lib.detnet_model_prune(self._h, int(kind), eta, eta1, eta2))

    def get_masks(self):
        out = np.empty((self.depth, record_size(self.n_tx, self.z_dim, self.v_dim)))
        _check(_lib.detnet_model_get_masks(self._h, _addr(out)))
        return out

    def cost_report(self):
        r = _CostReport()
        pl = (_LayerCost * self.depth)()
        _check(_lib.detnet_model_cost_report(self._h, C.byref(r), pl))
        rep = {f: getattr(r, f) for f, _ in _CostReport._fields_}
        per = np.array([[c.params_total, c.params_nonzero, c.flops] for c in pl], np.int64)
        return rep, per

    def batch_gradient(self, H, y, x, kind=0, lam=0.0, lam1=0.0, lam2=0.0, trainable_only=False):
        H, y, x = self._samples(H, y, x)
        n = H.shape[0]
        P = record_size(self.n_tx, self.z_dim, self.v_dim)
        grads = np.zeros((self.depth, P))
        ev = _Eval()
        spec = _LossSpec(kind, lam, lam1, lam2)
        _check(_lib.detnet_batch_gradient(self._h, n, _addr(H), _addr(y), _addr(x), C.byref(spec),
                                          int(trainable_only), _addr(grads), C.byref(ev)))
        return BatchEval(ev.data_loss, ev.symbol_errors, ev.symbols, ev.flagged, ev.loss_sum), grads
