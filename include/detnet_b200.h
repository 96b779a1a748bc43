/*
 * detnet_b200.h -- C-ABI of the B200-native DetNet layer-stack engine.
 *
 * The reference (`unfold`, /root/reference/proj) has no FFI: its batch-kernel
 * seam is the C++ API in include/unfold/kernels.hpp:29-65 plus adam_step
 * (adam.hpp:36-37), swapped at link time. This header is that seam as plain C
 * (pointers, sizes, status codes; no torch, no C++ types). The C++ adapter in
 * paper_2003_09446_b200/host/unfold_b200.cpp re-exposes it as the reference's
 * own `unfold::` functions (drop-in for src/kernels.cpp), and Python binds it
 * with ctypes (paper_2003_09446_b200/detnet.py).
 *
 * Conventions
 *  - Samples (ChannelSample, channel.hpp:11-16) are FP32 on this boundary:
 *      H [n][n_rx][n_tx] row-major, y [n][n_rx], x [n][n_tx] as int8 +-1.
 *  - Parameters (ModelParams/LayerParams, model.hpp:27-47) are FP64 "layer
 *    records", one per layer, in the tests/grad_check.hpp:16-44 order:
 *      record = W1[Z][IN] b1[Z] W2[K][Z] b2[K] W3[V][Z] b3[V] t,  IN = 3K+V.
 *    Masks use the same layout (t slot ignored); NULL means all ones. The
 *    effective weight is W (.) M (model.cpp:58-80).
 *  - Gradients and Adam moments (Gradients/AdamState, backward.hpp:11-28,
 *    adam.hpp:23-27) use the same record layout; frozen records are zero.
 *  - Every call returns a detnet_status; on error detnet_last_error() holds
 *    the message. The C++ adapter maps statuses back to the reference's
 *    exception types (errors.hpp:9-31).
 *  - A context is single-owner (not thread-safe), like unfold::Rng.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns DETNET_ERR_CUDA.
 */
#ifndef DETNET_B200_H
#define DETNET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DETNET_OK = 0,
    DETNET_ERR_CONTRACT = 1, /* ContractError: shapes, arguments (matrix.hpp:34-36) */
    DETNET_ERR_SINGULAR = 2, /* SingularMatrixError: ZF pivot test (linalg.cpp:59-60) */
    DETNET_ERR_CONFIG = 3,   /* ConfigError: count < 1, N < K (kernels.cpp:118-120) */
    DETNET_ERR_CUDA = 4,     /* CUDA runtime / launch failure, or no device */
    DETNET_ERR_NCCL = 5,     /* collective failure (multi-GPU) */
    DETNET_ERR_UNSUPPORTED = 6, /* dims outside the compiled kernel set */
    DETNET_ERR_DIVERGENCE = 7 /* DivergenceError: non-finite training objective (training.cpp:68-70) */
} detnet_status;

typedef struct detnet_ctx detnet_ctx;
typedef struct detnet_model detnet_model;

/* ---- context ---------------------------------------------------------- */
int detnet_ctx_create(int device, detnet_ctx **out);
void detnet_ctx_destroy(detnet_ctx *ctx);
/* A device group: one context per listed device (a device may repeat: that
 * runs several shards on one GPU). The host-buffer detnet_batch_evaluate and
 * detnet_batch_gradient (FP32 mode) of a group model shard the batch over all
 * members at 8,192-sample chunk boundaries, one host thread per member, and
 * fold the members' chunk sums in the canonical chunk order every kernel
 * uses, so BatchEval and gradients are bit-identical for any group size
 * (the reference's thread-count invariance, kernels.cpp:93-103, 160-200).
 * Settings apply to every member; models are replicated. Device-pointer entry
 * points (_device, _async, train_grad/apply, preprocess, forward_range) and
 * the FP64 training mode run on the first device; after device-side training
 * or pruning the replicas are refreshed before the next group call. */
int detnet_ctx_create_group(const int *devices, int count, detnet_ctx **out);
int detnet_ctx_group_size(const detnet_ctx *ctx);
const char *detnet_last_error(void);

/* Page-locked host memory for sample / output buffers. detnet_batch_evaluate,
 * detnet_batch_gradient and detnet_generate_host move pinned buffers at the full
 * PCIe rate, asynchronously and overlapped with compute; pageable buffers are
 * staged by the driver at a fraction of it. What the reference's callers do with
 * their std::vector<ChannelSample> batches (kernels.hpp:34-47) the seam does by
 * converting into buffers from here. bytes = 0 returns a null pointer. */
int detnet_host_alloc(void **ptr, size_t bytes);
int detnet_host_free(void *ptr);
/* Kernel-path selection: 0 auto (tcgen05 split-FP16 where compiled, with
 * 3xTF32 recompute of out-of-range tiles; else 3xTF32; else SIMT), 1 SIMT
 * FP32, 2 tcgen05 3xTF32 only, 3 sparse (the model-specialised kernel,
 * NVRTC-compiled once per weight version, for models with <= 1,500
 * surviving products per layer; else SIMT), 4 tcgen05 split-FP16. */
int detnet_ctx_set_path(detnet_ctx *ctx, int path);
/* Training forward (detnet_train_grad / detnet_batch_gradient) on tcgen05
 * (1, default: split FP16 for dense K=20 models) or FP32 CUDA cores (0). The
 * tensor-core forward is ~4x faster; its per-operation error (~2^-22) is a
 * few times FP32's, which over 100 chaotic training steps moves the loss by
 * as much as FP32 rounding itself does (training parity); the FP64
 * mode (detnet_ctx_set_train_precision) is the reference-exact path. The
 * reverse sweep and the weight-gradient contractions run on tcgen05 (3xTF32)
 * for the K=20/z=160/v=40 dims in either case. */
int detnet_ctx_set_train_forward(detnet_ctx *ctx, int tensor_cores);
/* Training arithmetic: 0 FP32 (default, the fast path), 1 FP64 in the
 * reference's operation order -- the forward trace, reverse sweep and the
 * min(16, n)-block gradient accumulation of kernels.cpp:160-200 with separate
 * IEEE multiplies/adds, so detnet_batch_gradient / detnet_train_grad +
 * detnet_train_apply are bit-identical to the reference's batch_gradient +
 * adam_step on FP32-representable samples (one rank). */
int detnet_ctx_set_train_precision(detnet_ctx *ctx, int fp64);

/* Preprocessing mode: 0 (default) FP32 Cholesky + FP64 refinement with the
 * reference LU as fallback for ill-conditioned samples (FP64-accurate loss
 * denominators); 1 the reference LU for every sample (bit-identical q, G,
 * x_tilde and denominators, slower). */
int detnet_ctx_set_exact_preprocess(detnet_ctx *ctx, int on);
/* CUDA stream (cudaStream_t) the context launches on; NULL = its own stream. */
int detnet_ctx_set_stream(detnet_ctx *ctx, void *stream);
void *detnet_ctx_stream(detnet_ctx *ctx);

/* Per-kernel device time, measured with CUDA events around every launch on
 * the launching stream when profiling is on (detnet_ctx_set_profiling). */
typedef struct {
    double ms[8];         /* by kernel class, see DETNET_K_* */
    long long launches[8];
} detnet_kernel_times;
enum { DETNET_K_GENERATE = 0, DETNET_K_PREPROCESS = 1, DETNET_K_STACK = 2, DETNET_K_REDUCE = 3,
       DETNET_K_BACKWARD = 4, DETNET_K_ADAM = 5, DETNET_K_OTHER = 6 };
int detnet_ctx_set_profiling(detnet_ctx *ctx, int on);
int detnet_ctx_kernel_times(detnet_ctx *ctx, detnet_kernel_times *out, int reset);
/* Total number of kernels this context launched (all classes). */
long long detnet_ctx_launch_count(detnet_ctx *ctx);
/* The canonical per-8,192-sample-chunk loss sums of the context's last
 * evaluation / gradient reduction (waits for the context stream): returns
 * the chunk count (copies min(cap, count) into out), or -status. Ranks that
 * own chunk-aligned shards fold the gathered sums in global chunk order to
 * get the single-device loss sum bit for bit (parallel.reduce_stats). */
long detnet_ctx_chunk_sums(detnet_ctx *ctx, double *out, long cap);

/* ---- parameters (ModelParams) ----------------------------------------- */
typedef struct {
    int n_tx, n_rx, z_dim, v_dim, depth, frozen_prefix;
    const double *params; /* depth * record, host memory */
    const double *masks;  /* depth * record or NULL (all ones) */
} detnet_model_desc;

long detnet_record_size(int n_tx, int z_dim, int v_dim);
/* Upload/pack parameters once per params version (SURVEY 8b "Ownership"). */
int detnet_model_create(detnet_ctx *ctx, const detnet_model_desc *desc, detnet_model **out);
int detnet_model_update(detnet_model *m, const detnet_model_desc *desc);
void detnet_model_destroy(detnet_model *m);
/* Kernel path the stack of this model runs on under the context's current
 * path setting: 1 SIMT FP32, 2 tcgen05 3xTF32, 3 sparse CSR, 4 tcgen05
 * split-FP16, 5 sparse model-specialised (NVRTC-compiled from the model's
 * surviving weights at its first evaluation). */
int detnet_model_path(const detnet_model *m);
/* Analytic census, flops_per_detection (compression.cpp:120-129). */
long long detnet_model_flops_per_detection(const detnet_model *m, int include_preprocess);

/* ---- batch evaluation (batch_evaluate, kernels.cpp:138-158) ------------ */
typedef struct {
    double data_loss;      /* mean per-sample depth-weighted loss (BatchEval) */
    double loss_sum;       /* sum over samples, fixed tile order */
    long long symbol_errors;
    long long symbols;
    long long flagged;     /* samples whose denominator guard fired */
} detnet_eval;

/* Host buffers. Copies host->device in chunks overlapped with compute.
 * loss_layers_trainable_only: LossLayers::trainable_only (loss.hpp:16-19).
 * xhat_out (optional, host): [n][depth][n_tx] soft outputs x_hat_1..x_hat_L
 * (ForwardTrace::x_hat[1..L], model.hpp:52-63). */
int detnet_batch_evaluate(detnet_model *m, long n, const float *H, const float *y,
                          const int8_t *x, int loss_layers_trainable_only, float *xhat_out,
                          detnet_eval *out);
/* Same with device-resident inputs/outputs (no host copies of the samples). */
int detnet_batch_evaluate_device(detnet_model *m, long n, const float *H_dev, const float *y_dev,
                                 const int8_t *x_dev, int loss_layers_trainable_only,
                                 float *xhat_dev, detnet_eval *out);

/* Asynchronous form of detnet_batch_evaluate_device: enqueues the whole
 * evaluation on the context stream and returns a ticket at once; the
 * BatchEval (and SingularMatrixError) comes from detnet_eval_wait. At most 64
 * evaluations may be in flight per context (CONTRACT error beyond). Lets a
 * caller keep the device busy across many batches with no host round trip
 * between them; results are identical to the synchronous call. */
int detnet_batch_evaluate_device_async(detnet_model *m, long n, const float *H_dev,
                                       const float *y_dev, const int8_t *x_dev,
                                       int loss_layers_trainable_only, float *xhat_dev,
                                       long long *ticket);
int detnet_eval_wait(detnet_ctx *ctx, long long ticket, detnet_eval *out);

/* The per-sample preprocessing alone (K1 + its exact-LU fallback; the part of
 * evaluate_one before the layer loop, kernels.cpp:55-58, linalg.cpp:20-79),
 * device buffers in and out, sample-major: gram_dev [n][K(K+1)/2] the upper
 * triangle of G = H^T H row by row (linalg.cpp:31-42), q_dev [n][K] = H^T y,
 * denom_dev [n] = max(||x - x_tilde||^2, 1e-12) (loss.cpp:14-19), flag_dev [n]
 * the guard flag. Any output pointer may be NULL. A parity hook for the
 * preprocessing; SingularMatrixError like batch_evaluate. */
int detnet_preprocess_device(detnet_model *m, long n, const float *H_dev, const float *y_dev,
                             const int8_t *x_dev, float *gram_dev, float *q_dev,
                             double *denom_dev, uint8_t *flag_dev);

/* Layers [l_begin, l_end) from a given state (host buffers): the teacher-
 * forced single-layer check of SURVEY 7.3/H1. x_state [n][K], v_state [n][V]
 * are read and overwritten with the state after layer l_end-1; xhat_out
 * (optional) [n][l_end-l_begin][K]. */
int detnet_forward_range(detnet_model *m, long n, const float *H, const float *y, int l_begin,
                         int l_end, float *x_state, float *v_state, float *xhat_out);

/* ---- training step (batch_gradient / adam_step) ------------------------ */
typedef struct {
    int kind;              /* 0 plain, 1 element_l1, 2 sparse_group (loss.hpp:7-14) */
    double lambda, lambda1, lambda2;
} detnet_loss_spec;

/* batch_gradient (kernels.cpp:160-200): mean data-term gradient plus the
 * regularizer gradient, host grads in record layout (frozen records 0). */
int detnet_batch_gradient(detnet_model *m, long n, const float *H, const float *y,
                          const int8_t *x, const detnet_loss_spec *spec,
                          int loss_layers_trainable_only, double *grads_out, detnet_eval *out);

typedef struct {
    double lr0, decay_factor;
    int decay_step;
    double beta1, beta2, eps;
} detnet_adam_config;

/* Device-resident training step, split so ranks can all-reduce (sum) the raw
 * gradient between the two calls (one data-parallel rank per GPU):
 *  detnet_train_grad: samples (device) -> raw_dev [param_count] FP64 sums of
 *    the per-sample data-term gradients (unscaled, unmasked, record layout)
 *    and this rank's BatchEval (loss sum, errors, flagged); out may be NULL:
 *    then the call only enqueues (no wait, no SingularMatrixError check);
 *  detnet_train_apply: raw (all-reduced) -> mean over n_global samples, masks,
 *    regularizer gradient, Adam update of the model's device master params
 *    (moments kept in the model; reset with detnet_model_reset_adam, as
 *    training.cpp:55 starts a fresh AdamState per incremental step). Stream-
 *    ordered on the context stream; it does not wait for the device. */
long detnet_model_param_count(const detnet_model *m);
/* raw_dev holds detnet_train_raw_count(m) = param_count + 1 doubles: the
 * gradient sums, then this rank's data-loss sum (sample order in FP64 mode);
 * ranks all-reduce (sum) the whole buffer. */
long detnet_train_raw_count(const detnet_model *m);
int detnet_train_grad(detnet_model *m, long n, const float *H_dev, const float *y_dev,
                      const int8_t *x_dev, int loss_layers_trainable_only, double *raw_dev,
                      detnet_eval *out);
/* detnet_train_grad, enqueue only, with the raw sums finalised in buckets as
 * the reverse sweep produces them (top layers first, one bucket per sweep
 * chunk, the loss-sum slot last): after the call, raw entries
 * [ranges[2b], ranges[2b+1]) are final once events[b] (a cudaEvent_t owned by
 * the context, valid until its next training call) has completed on the
 * device. A data-parallel caller all-reduces each bucket on a side stream
 * while the rest of the sweep runs, then orders the context
 * stream after it before detnet_train_apply. Frozen layers' slots are zero on
 * every rank and in no bucket. Returns the bucket count or -status. Bit for
 * bit the sums of detnet_train_grad. */
int detnet_train_grad_buckets(detnet_model *m, long n, const float *H, const float *y,
                              const int8_t *x, int trainable_only, double *raw_dev, void **events,
                              long *ranges, int max_buckets);
/* cudaStreamWaitEvent(stream, event) for callers without a CUDA runtime of
 * their own (the bucket events above). */
int detnet_stream_wait_event(void *stream, void *event);
/* Also forms objective = raw[param_count] / n_global + regularizer(params,
 * spec) before the update (training.cpp:65-70, loss.cpp:81-91, bit-identical
 * order); a non-finite objective halts training on the device (no update, the
 * reference throws before adam_step) and this and every later call returns
 * DETNET_ERR_DIVERGENCE once the host has seen it (detnet_train_status). */
int detnet_train_apply(detnet_model *m, const double *raw_dev, long n_global,
                       const detnet_loss_spec *spec, const detnet_adam_config *cfg);
/* Waits for the context stream; objective and regularizer value of the last
 * detnet_train_apply (either pointer may be NULL); DETNET_ERR_DIVERGENCE if
 * training halted on a non-finite objective. */
int detnet_train_status(detnet_model *m, double *objective, double *regularizer);
int detnet_model_get_params(detnet_model *m, double *params_out);
int detnet_model_reset_adam(detnet_model *m);

/* adam_step (adam.cpp:48-79) on host arrays: params (record layout, updated
 * in place), grads, first/second moments, *step advanced by one. */
int detnet_adam_step(detnet_ctx *ctx, int n_tx, int z_dim, int v_dim, int depth,
                     int frozen_prefix, double *params, const double *masks, const double *grads,
                     double *m1, double *m2, int64_t *step, const detnet_adam_config *cfg);

/* ---- incremental-depth training (train_incremental, training.cpp:22-141) --
 * The reference's whole schedule as one device-resident call: batches from the
 * on-device generator with the reference's keying (master Rng(seed): init
 * stream 1, train stream 2, validation stream 3), parameters / Adam moments /
 * objective in HBM, a fresh Adam state per incremental step, validation on the
 * device-resident evaluation set, the reference's halting tests, freeze + append
 * with init_layer draws (model.cpp:140-166). sample_scale multiplies H and y
 * (1.0 = the reference's N(0,1) channels, 1/sqrt(N) = BASELINE's N(0,1/N)). */
typedef struct {
    int start_layers, t_step, max_layers;          /* IncrementalConfig */
    double halt_epsilon, target_ber;
    int val_samples;
    double val_snr_db;
    int total_batches, batch_size;                 /* TrainConfig */
    double snr_lo_db, snr_hi_db;
    detnet_adam_config adam;
    detnet_loss_spec spec;
    double weight_scale, t0;                       /* InitOptions */
    int loss_layers_trainable_only;
    uint64_t seed;
    double sample_scale;
} detnet_incremental_config;
typedef struct {
    int step, layer_count;                         /* StepRecord */
    double train_loss, val_loss, val_ber, wall_ms;
} detnet_step_record;
typedef struct {
    int halt_reason;                               /* 0 target_ber, 1 converged, 2 max_layers */
    int depth, frozen_prefix;
    long long flagged_samples, optimizer_steps;
    double seconds;
} detnet_incremental_result;
/* records: up to max_records step records (*n_records = how many steps ran);
 * params_out (nullable): max_layers * record doubles, the final parameters. */
int detnet_train_incremental(detnet_ctx *ctx, int n_tx, int n_rx, int z_dim, int v_dim,
                             const detnet_incremental_config *cfg, detnet_step_record *records,
                             int max_records, int *n_records, double *params_out,
                             detnet_incremental_result *result);

/* ---- on-device channel generator (make_sample/generate_batch) --------- */
/* Rng(seed, stream_id) state (rng.cpp:18-19). */
uint64_t detnet_rng_seed(uint64_t seed, uint64_t stream_id);
/* Rng::stream(id) (rng.cpp:40-42); does not advance. */
uint64_t detnet_rng_stream(uint64_t state, uint64_t id);
/* Rng::split() (rng.cpp:44): returns the child state and advances *state. */
uint64_t detnet_rng_split(uint64_t *state);
/* Samples [first, first+count) of generate_batch whose split base state is
 * `base` (kernels.cpp:121-127): sample i uses base.stream(i) and the
 * make_sample draw order (channel.cpp:14-32). H and y are multiplied by
 * `scale` (1/sqrt(N) for H ~ N(0,1/N)) and rounded to FP32. Device buffers. */
int detnet_generate_device(detnet_ctx *ctx, uint64_t base, long first, long count, int n_rx,
                           int n_tx, double snr_lo_db, double snr_hi_db, double scale,
                           float *H_dev, float *y_dev, int8_t *x_dev, double *sigma2_dev);

/* Same generator with unscaled FP64 host outputs, exactly the fields of the
 * ChannelSamples unfold::generate_batch returns: H [count][n_rx][n_tx],
 * x [count][n_tx] (+-1.0), y [count][n_rx], sigma2 [count] (nullable). */
int detnet_generate_host(detnet_ctx *ctx, uint64_t base, long first, long count, int n_rx,
                         int n_tx, double snr_lo_db, double snr_hi_db, double *H, double *x,
                         double *y, double *sigma2);

/* Detector baselines on the device: replaces
 * batch_baseline_errors (kernels.hpp:48-49; kernels.cpp:105-112, 202-223).
 * kind 0 = ZF (sign of solve_normal_equations(gram(H), H^T y)),
 * 1 = ML (exhaustive, K <= 16; DETNET_ERR_UNSUPPORTED otherwise, the
 * reference's CapacityError), 2 = oracle (0 errors). Host FP64 samples in the
 * reference layout (H [n][N][K], y [n][N], x [n][K] as +-1.0); decisions are
 * bit-identical to the reference. A singular ZF system returns
 * DETNET_ERR_SINGULAR (SingularMatrixError, linalg.cpp:59-60). */
/* Pruning planner on the device-resident master weights:
 * replaces prune / prune_element / prune_group / prune_sparse_group
 * (compression.hpp; compression.cpp:43-94) with bit-identical masks.
 * kind 0 = element(eta), 1 = group(eta1), 2 = sparse_group(eta1, eta2);
 * thresholds in [0, 1) (else DETNET_ERR_CONFIG, PruneSpec::validate). The
 * packed layouts (dense / compacted tcgen05 / sparse) are rebuilt from the
 * result; Adam state is kept. */
int detnet_model_prune(detnet_model *model, int kind, double eta, double eta1, double eta2);
/* Current masks in the layer-record layout (ones where unmasked). */
int detnet_model_get_masks(detnet_model *model, double *masks_out);

/* cost_report (compression.hpp CostReport/LayerCost; compression.cpp:131-159). */
typedef struct {
    long long params_total, params_nonzero, flops;
} detnet_layer_cost;
typedef struct {
    int layer_count;
    long long params_total, params_nonzero, memory_dense_bytes, memory_sparse_bytes, flops,
        flops_dense, preprocess_flops;
} detnet_cost_report;
int detnet_model_cost_report(detnet_model *model, detnet_cost_report *report,
                             detnet_layer_cost *per_layer /* [depth] or NULL */);

int detnet_batch_baseline_errors(detnet_ctx *ctx, int kind, long n, int n_rx, int n_tx,
                                 const double *H, const double *y, const double *x,
                                 long long *errors, long long *symbols);

#ifdef __cplusplus
}
#endif
#endif
