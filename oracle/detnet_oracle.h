/*
 * detnet_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A from-scratch plain-C restatement of the reference's CPU algorithm for the
 * batched DetNet layer stack (arXiv 2003.09446, reference `unfold` library).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it. The product path (libdetnet_b200.so) never links or calls it.
 *
 * Parity status: pinned. tests/test_oracle.py checks every function below
 * bit-for-bit against the reference itself (oracle/_ref/libunfold_ref.so,
 * compiled from /root/reference/proj/src by oracle/Makefile) and against the
 * committed golden vectors in tests/golden/ that tools/make_golden.py
 * generated from that build.
 *
 * Layouts (shared with include/detnet_b200.h):
 *   samples : H [n][N][K] row-major, y [n][N], x [n][K] (+-1)
 *   params  : L consecutive "layer records" of P doubles each,
 *             record = W1[Z][IN] b1[Z] W2[K][Z] b2[K] W3[V][Z] b3[V] t
 *             (the tests/grad_check.hpp:16-44 flattening order);
 *   masks   : same record layout (t slot ignored), NULL = all ones;
 *   grads, Adam moments: same record layout as params.
 */
#ifndef DETNET_ORACLE_H
#define DETNET_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng: splitmix64 counter generator (rng.cpp:12-46) ---------------- */
typedef struct { uint64_t s; } or_rng;
uint64_t or_mix64(uint64_t z);
or_rng or_rng_new(uint64_t seed, uint64_t stream_id);
uint64_t or_next_u64(or_rng *r);
double or_next_uniform(or_rng *r);
double or_next_uniform_range(or_rng *r, double lo, double hi);
int or_next_bit(or_rng *r);
double or_next_gaussian(or_rng *r);
or_rng or_stream(const or_rng *r, uint64_t id);
or_rng or_split(or_rng *r);

/* ---- channel (channel.cpp:9-32, kernels.cpp:116-136) ------------------- */
double or_snr_to_sigma2(double snr_db, int n_tx);
void or_make_sample(or_rng *r, int n_rx, int n_tx, double lo_db, double hi_db,
                    double *H, double *x, double *y, double *sigma2);
/* generate_batch: advances *r by one draw (split), sample i uses stream(i).
 * first/count select a sub-range of sample indices (random access). */
void or_generate_batch(or_rng *r, int n_rx, int n_tx, long first, long count,
                       double lo_db, double hi_db, double *H, double *x, double *y,
                       double *sigma2);
/* Same, from an already-split base state (no advance). */
void or_generate_range(const or_rng *base, int n_rx, int n_tx, long first, long count,
                       double lo_db, double hi_db, double *H, double *x, double *y,
                       double *sigma2);

/* ---- model ------------------------------------------------------------ */
typedef struct {
    int n_tx, n_rx, z_dim, v_dim, depth, frozen_prefix;
    const double *params; /* depth * record */
    const double *masks;  /* NULL = all ones */
} or_model;

long or_record_size(int n_tx, int z_dim, int v_dim);

/* Preprocessing (linalg.cpp:20-79): q = H^T y, G = H^T H, x_tilde = G^-1 q.
 * Returns 0, or 2 if the ZF solve is singular. */
int or_preprocess(int n_rx, int n_tx, const double *H, const double *y, double *q,
                  double *G, double *x_tilde);

/* One layer of forward_pre (model.cpp:103-120) from state (xh, v). Outputs
 * x_hat_{l+1}, v_{l+1}; u1/z/u2/in optional (NULL). */
void or_layer(const or_model *m, int l, const double *q, const double *G, const double *xh,
              const double *v, double *xh_out, double *v_out, double *in_out,
              double *u1_out, double *z_out, double *u2_out);

/* Per-sample evaluate_one (kernels.cpp:55-67) over a batch. Per-sample outputs
 * are optional (NULL). xhat_out: [n][L][K] = x_hat_1..x_hat_L.
 * Returns 0 or 2 (singular ZF: first offending sample index in *bad). */
int or_evaluate(const or_model *m, long n, const double *H, const double *y, const double *x,
                int first_term, double *loss_out, long long *err_out, int *flag_out,
                double *xhat_out, long *bad);

/* batch_evaluate (kernels.cpp:138-158 / 240-246): fixed sample-order sums. */
int or_batch_evaluate(const or_model *m, long n, const double *H, const double *y,
                      const double *x, int loss_layers_trainable_only, double *data_loss,
                      long long *errors, long long *symbols, long long *flagged);

/* FP32 restatement of the forward (same loop order, float arithmetic after
 * q and G are formed in double and rounded once): the FP32 error floor. */
int or_evaluate_f32(const or_model *m, long n, const double *H, const double *y,
                    const double *x, int first_term, double *loss_out, long long *err_out,
                    double *xhat_out);

/* ---- training --------------------------------------------------------- */
enum { OR_LOSS_PLAIN = 0, OR_LOSS_L1 = 1, OR_LOSS_SGL = 2 };
typedef struct { int kind; double lambda, lambda1, lambda2; } or_loss_spec;

/* batch_gradient (kernels.cpp:160-200): 16 fixed blocks, merged in order,
 * scaled by 1/n, then backward_regularizer (backward.cpp:201-220).
 * grads: depth * record (frozen records left 0). */
int or_batch_gradient(const or_model *m, long n, const double *H, const double *y,
                      const double *x, const or_loss_spec *spec,
                      int loss_layers_trainable_only, double *grads, double *data_loss,
                      long long *errors, long long *symbols, long long *flagged);

/* FP32 restatement of batch_gradient (O32): per-sample forward and reverse
 * sweep in FP32 in the reference's order, FP32 per-block accumulation, FP64
 * preprocessing, merge, scaling and regularizer. Calibrates FP32's intrinsic
 * spread against the FP64 reference over a training run. OpenMP over the
 * fixed blocks (results independent of the thread count). */
int or_batch_gradient_f32(const or_model *m, long n, const double *H, const double *y,
                          const double *x, const or_loss_spec *spec,
                          int loss_layers_trainable_only, double *grads, double *data_loss,
                          long long *errors, long long *symbols, long long *flagged);

/* regularizer value (loss.cpp:81-91) */
double or_regularizer(const or_model *m, const or_loss_spec *spec);

typedef struct {
    double lr0, decay_factor;
    int decay_step;
    double beta1, beta2, eps;
} or_adam_config;

/* adam_step (adam.cpp:48-79): params (mutable, depth*record), m/v moments
 * (depth*record), *step advanced by one. */
void or_adam_step(int n_tx, int z_dim, int v_dim, int depth, int frozen_prefix,
                  double *params, const double *masks, const double *grads, double *m,
                  double *v, int64_t *step, const or_adam_config *cfg);

/* flops_per_detection census (compression.cpp:120-129) */
long long or_flops_per_detection(const or_model *m, int include_preprocess);

#ifdef __cplusplus
}
#endif
#endif
