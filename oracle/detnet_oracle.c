/*
 * detnet_oracle.c -- TEST INFRASTRUCTURE ONLY: CPU restatement of the
 * reference DetNet hot path, used as the parity checker. See detnet_oracle.h.
 *
 * Every function restates one reference function (file:line relative to
 * /root/reference/proj) in the same operation order, so that with
 * -ffp-contract=off it reproduces the reference's FP64 results bit for bit.
 */
#include "detnet_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */
/* rng.cpp:10-16 */
static const uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.cpp:18-19 */
or_rng or_rng_new(uint64_t seed, uint64_t stream_id) {
    or_rng r;
    r.s = or_mix64(or_mix64(seed ^ 0x853c49e6748fea9bULL) + stream_id);
    return r;
}

/* rng.cpp:21 */
uint64_t or_next_u64(or_rng *r) { r->s += kGamma; return or_mix64(r->s); }

/* rng.cpp:23-29 */
double or_next_uniform(or_rng *r) { return (double)(or_next_u64(r) >> 11) * 0x1.0p-53; }
double or_next_uniform_range(or_rng *r, double lo, double hi) {
    return lo + (hi - lo) * or_next_uniform(r);
}

/* rng.cpp:31 */
int or_next_bit(or_rng *r) { return (or_next_u64(r) >> 63) != 0; }

/* rng.cpp:33-38: Box-Muller, cosine branch, u1 in (0,1] */
double or_next_gaussian(or_rng *r) {
    double u1 = 1.0 - or_next_uniform(r);
    double u2 = or_next_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* rng.cpp:40-42 */
or_rng or_stream(const or_rng *r, uint64_t id) {
    or_rng o;
    o.s = or_mix64(r->s ^ or_mix64(id + 0xda3e39cb94b95bdbULL));
    return o;
}

/* rng.cpp:44 */
or_rng or_split(or_rng *r) {
    or_rng o;
    o.s = or_mix64(or_next_u64(r));
    return o;
}

/* -------------------------------------------------------------- channel */
/* channel.cpp:9-12 */
double or_snr_to_sigma2(double snr_db, int n_tx) { return n_tx * pow(10.0, -snr_db / 10.0); }

/* channel.cpp:14-32: draw order SNR (ranged only) -> H row-major -> x bits -> noise */
void or_make_sample(or_rng *r, int n_rx, int n_tx, double lo_db, double hi_db, double *H,
                    double *x, double *y, double *sigma2) {
    const double snr_db = (lo_db == hi_db) ? lo_db : or_next_uniform_range(r, lo_db, hi_db);
    const double s2 = or_snr_to_sigma2(snr_db, n_tx);
    for (int i = 0; i < n_rx * n_tx; ++i) H[i] = or_next_gaussian(r);
    for (int j = 0; j < n_tx; ++j) x[j] = or_next_bit(r) ? 1.0 : -1.0;
    /* y = matvec(H, x) (linalg.cpp:8-18) */
    for (int i = 0; i < n_rx; ++i) {
        double acc = 0.0;
        for (int j = 0; j < n_tx; ++j) acc += H[i * n_tx + j] * x[j];
        y[i] = acc;
    }
    const double sigma = sqrt(s2);
    for (int i = 0; i < n_rx; ++i) y[i] += sigma * or_next_gaussian(r);
    if (sigma2) *sigma2 = s2;
}

void or_generate_range(const or_rng *base, int n_rx, int n_tx, long first, long count,
                       double lo_db, double hi_db, double *H, double *x, double *y,
                       double *sigma2) {
    for (long i = 0; i < count; ++i) {
        or_rng s = or_stream(base, (uint64_t)(first + i));
        or_make_sample(&s, n_rx, n_tx, lo_db, hi_db, H + i * (long)n_rx * n_tx,
                       x + i * (long)n_tx, y + i * (long)n_rx, sigma2 ? sigma2 + i : NULL);
    }
}

/* kernels.cpp:116-136: base = rng.split(); sample i <- base.stream(i) */
void or_generate_batch(or_rng *r, int n_rx, int n_tx, long first, long count, double lo_db,
                       double hi_db, double *H, double *x, double *y, double *sigma2) {
    const or_rng base = or_split(r);
    or_generate_range(&base, n_rx, n_tx, first, count, lo_db, hi_db, H, x, y, sigma2);
}

/* ---------------------------------------------------------------- model */
typedef struct {
    long W1, b1, W2, b2, W3, b3, t, size;
} rec_off;

static rec_off offsets(int K, int Z, int V) {
    const int IN = 3 * K + V;
    rec_off o;
    o.W1 = 0;
    o.b1 = o.W1 + (long)Z * IN;
    o.W2 = o.b1 + Z;
    o.b2 = o.W2 + (long)K * Z;
    o.W3 = o.b2 + K;
    o.b3 = o.W3 + (long)V * Z;
    o.t = o.b3 + V;
    o.size = o.t + 1;
    return o;
}

long or_record_size(int n_tx, int z_dim, int v_dim) { return offsets(n_tx, z_dim, v_dim).size; }

/* linalg.cpp:20-29 (H^T y, i outer), 31-42 (gram, upper triangle mirrored),
 * 44-79 (partially pivoted elimination, tol 1e-12 * max|G|). */
int or_preprocess(int N, int K, const double *H, const double *y, double *q, double *G,
                  double *xt) {
    for (int j = 0; j < K; ++j) q[j] = 0.0;
    for (int i = 0; i < N; ++i) {
        const double vi = y[i];
        for (int j = 0; j < K; ++j) q[j] += H[i * K + j] * vi;
    }
    for (int a = 0; a < K; ++a)
        for (int b = a; b < K; ++b) {
            double acc = 0.0;
            for (int i = 0; i < N; ++i) acc += H[i * K + a] * H[i * K + b];
            G[a * K + b] = acc;
            G[b * K + a] = acc;
        }
    if (!xt) return 0;
    double gmax = 0.0;
    for (int i = 0; i < K * K; ++i) gmax = fmax(gmax, fabs(G[i]));
    const double tol = 1e-12 * gmax;
    double A[64 * 64];
    double *Ap = K <= 64 ? A : (double *)malloc(sizeof(double) * K * K);
    memcpy(Ap, G, sizeof(double) * K * K);
    for (int j = 0; j < K; ++j) xt[j] = q[j];
    int status = 0;
    for (int col = 0; col < K && !status; ++col) {
        int piv = col;
        for (int r = col + 1; r < K; ++r)
            if (fabs(Ap[r * K + col]) > fabs(Ap[piv * K + col])) piv = r;
        if (fabs(Ap[piv * K + col]) <= tol) { status = 2; break; }
        if (piv != col) {
            for (int j = 0; j < K; ++j) {
                double tmp = Ap[col * K + j];
                Ap[col * K + j] = Ap[piv * K + j];
                Ap[piv * K + j] = tmp;
            }
            double tmp = xt[col]; xt[col] = xt[piv]; xt[piv] = tmp;
        }
        const double d = Ap[col * K + col];
        for (int r = col + 1; r < K; ++r) {
            const double f = Ap[r * K + col] / d;
            if (f == 0.0) continue;
            for (int j = col; j < K; ++j) Ap[r * K + j] -= f * Ap[col * K + j];
            xt[r] -= f * xt[col];
        }
    }
    if (!status)
        for (int i = K - 1; i >= 0; --i) {
            double acc = xt[i];
            for (int j = i + 1; j < K; ++j) acc -= Ap[i * K + j] * xt[j];
            xt[i] = acc / Ap[i * K + i];
        }
    if (Ap != A) free(Ap);
    return status;
}

/* model.cpp:58-80 masked path (bit-identical to the all-ones path):
 * acc = b*mb, then j ascending acc += (w*m)*x */
static void masked_affine(const double *W, const double *M, const double *b, const double *mb,
                          int rows, int cols, const double *x, double *out) {
    for (int i = 0; i < rows; ++i) {
        const double *row = W + (long)i * cols;
        double acc;
        if (M) {
            const double *mrow = M + (long)i * cols;
            acc = b[i] * mb[i];
            for (int j = 0; j < cols; ++j) acc += row[j] * mrow[j] * x[j];
        } else {
            acc = b[i];
            for (int j = 0; j < cols; ++j) acc += row[j] * x[j];
        }
        out[i] = acc;
    }
}

/* model.cpp:32-41 */
static double soft_sign1(double u, double t) {
    if (u <= -t) return -1.0;
    if (u >= t) return 1.0;
    return u / t;
}

/* model.cpp:103-120, one iteration */
void or_layer(const or_model *m, int l, const double *q, const double *G, const double *xh,
              const double *v, double *xh_out, double *v_out, double *in_out, double *u1_out,
              double *z_out, double *u2_out) {
    const int K = m->n_tx, Z = m->z_dim, V = m->v_dim, IN = 3 * K + V;
    const rec_off o = offsets(K, Z, V);
    const double *p = m->params + l * o.size;
    const double *mk = m->masks ? m->masks + l * o.size : NULL;
    double in[1024], u1[4096], z[4096], u2[1024];
    for (int i = 0; i < K; ++i) in[i] = q[i];
    for (int i = 0; i < K; ++i) in[K + i] = xh[i];
    for (int i = 0; i < K; ++i) { /* gx = matvec(G, x_hat) (linalg.cpp:8-18) */
        double acc = 0.0;
        for (int j = 0; j < K; ++j) acc += G[i * K + j] * xh[j];
        in[2 * K + i] = acc;
    }
    for (int i = 0; i < V; ++i) in[3 * K + i] = v[i];
    masked_affine(p + o.W1, mk ? mk + o.W1 : NULL, p + o.b1, mk ? mk + o.b1 : NULL, Z, IN, in, u1);
    for (int i = 0; i < Z; ++i) z[i] = u1[i] > 0.0 ? u1[i] : 0.0;
    masked_affine(p + o.W2, mk ? mk + o.W2 : NULL, p + o.b2, mk ? mk + o.b2 : NULL, K, Z, z, u2);
    const double t = p[o.t];
    for (int i = 0; i < K; ++i) xh_out[i] = soft_sign1(u2[i], t);
    masked_affine(p + o.W3, mk ? mk + o.W3 : NULL, p + o.b3, mk ? mk + o.b3 : NULL, V, Z, z, v_out);
    if (in_out) memcpy(in_out, in, sizeof(double) * IN);
    if (u1_out) memcpy(u1_out, u1, sizeof(double) * Z);
    if (z_out) memcpy(z_out, z, sizeof(double) * Z);
    if (u2_out) memcpy(u2_out, u2, sizeof(double) * K);
}

/* loss.cpp:9-31 with kernels.cpp:63-65 error count; x_hat_k for k = 1..L */
static double loss_plain(int K, int L, const double *xhat /* [L][K] */, const double *x,
                         const double *xt, int first_term, int *flagged) {
    double denom = 0.0;
    for (int i = 0; i < K; ++i) {
        const double d = x[i] - xt[i];
        denom += d * d;
    }
    *flagged = denom < 1e-12;
    if (denom < 1e-12) denom = 1e-12;
    double loss = 0.0;
    for (int k = first_term > 1 ? first_term : 1; k <= L; ++k) {
        double err = 0.0;
        for (int i = 0; i < K; ++i) {
            const double d = x[i] - xhat[(k - 1) * K + i];
            err += d * d;
        }
        loss += log((double)k) * err / denom;
    }
    return loss;
}

int or_evaluate(const or_model *m, long n, const double *H, const double *y, const double *x,
                int first_term, double *loss_out, long long *err_out, int *flag_out,
                double *xhat_out, long *bad) {
    const int K = m->n_tx, N = m->n_rx, V = m->v_dim, L = m->depth;
    double *tr = (double *)malloc(sizeof(double) * (size_t)L * K);
    double q[256], G[256 * 256 / 16], xt[256], xh[256], v[1024], xn[256], vn[1024];
    int status = 0;
    for (long s = 0; s < n; ++s) {
        const double *Hs = H + s * (long)N * K, *ys = y + s * (long)N, *xs = x + s * (long)K;
        if (or_preprocess(N, K, Hs, ys, q, G, xt)) {
            status = 2;
            if (bad) *bad = s;
            break;
        }
        for (int i = 0; i < K; ++i) xh[i] = 0.0;
        for (int i = 0; i < V; ++i) v[i] = 0.0;
        for (int l = 0; l < L; ++l) {
            or_layer(m, l, q, G, xh, v, xn, vn, NULL, NULL, NULL, NULL);
            memcpy(xh, xn, sizeof(double) * K);
            memcpy(v, vn, sizeof(double) * V);
            memcpy(tr + (long)l * K, xh, sizeof(double) * K);
        }
        int flagged = 0;
        const double loss = loss_plain(K, L, tr, xs, xt, first_term, &flagged);
        long long errors = 0;
        for (int i = 0; i < K; ++i) errors += (xh[i] >= 0.0 ? 1.0 : -1.0) != xs[i];
        if (loss_out) loss_out[s] = loss;
        if (err_out) err_out[s] = errors;
        if (flag_out) flag_out[s] = flagged;
        if (xhat_out) memcpy(xhat_out + s * (long)L * K, tr, sizeof(double) * (size_t)L * K);
    }
    free(tr);
    return status;
}

/* kernels.cpp:69-71, 93-103 */
int or_batch_evaluate(const or_model *m, long n, const double *H, const double *y,
                      const double *x, int trainable_only, double *data_loss,
                      long long *errors, long long *symbols, long long *flagged) {
    const int first = trainable_only ? m->frozen_prefix + 1 : 1;
    double *loss = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
    long long *err = (long long *)malloc(sizeof(long long) * (n > 0 ? n : 1));
    int *flag = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    const int st = or_evaluate(m, n, H, y, x, first, loss, err, flag, NULL, NULL);
    double dl = 0.0;
    long long e = 0, f = 0;
    if (!st) {
        for (long s = 0; s < n; ++s) { dl += loss[s]; e += err[s]; f += flag[s]; }
        if (n > 0) dl /= (double)n;
    }
    *data_loss = dl;
    *errors = e;
    *symbols = (long long)n * m->n_tx;
    *flagged = f;
    free(loss); free(err); free(flag);
    return st;
}

/* FP32 restatement: q, G formed in double, rounded once; layers in float. */
int or_evaluate_f32(const or_model *m, long n, const double *H, const double *y,
                    const double *x, int first_term, double *loss_out, long long *err_out,
                    double *xhat_out) {
    const int K = m->n_tx, N = m->n_rx, Z = m->z_dim, V = m->v_dim, L = m->depth;
    const int IN = 3 * K + V;
    const rec_off o = offsets(K, Z, V);
    const long P = o.size;
    float *w = (float *)malloc(sizeof(float) * (size_t)L * P);
    for (long i = 0; i < (long)L * P; ++i)
        w[i] = (float)(m->params[i] * (m->masks ? m->masks[i] : 1.0));
    double *tr = (double *)malloc(sizeof(double) * (size_t)L * K);
    double q[256], G[4096], xt[256];
    float qf[256], Gf[4096], xh[256], v[1024], in[1024], z[4096], u2[256], vn[1024];
    int status = 0;
    for (long s = 0; s < n; ++s) {
        const double *Hs = H + s * (long)N * K, *ys = y + s * (long)N, *xs = x + s * (long)K;
        if (or_preprocess(N, K, Hs, ys, q, G, xt)) { status = 2; break; }
        for (int i = 0; i < K; ++i) qf[i] = (float)q[i];
        for (int i = 0; i < K * K; ++i) Gf[i] = (float)G[i];
        for (int i = 0; i < K; ++i) xh[i] = 0.f;
        for (int i = 0; i < V; ++i) v[i] = 0.f;
        for (int l = 0; l < L; ++l) {
            const float *p = w + l * P;
            for (int i = 0; i < K; ++i) in[i] = qf[i];
            for (int i = 0; i < K; ++i) in[K + i] = xh[i];
            for (int i = 0; i < K; ++i) {
                float acc = 0.f;
                for (int j = 0; j < K; ++j) acc += Gf[i * K + j] * xh[j];
                in[2 * K + i] = acc;
            }
            for (int i = 0; i < V; ++i) in[3 * K + i] = v[i];
            for (int i = 0; i < Z; ++i) {
                float acc = p[o.b1 + i];
                for (int j = 0; j < IN; ++j) acc += p[o.W1 + (long)i * IN + j] * in[j];
                z[i] = acc > 0.f ? acc : 0.f;
            }
            const float t = (float)m->params[l * P + o.t];
            for (int i = 0; i < K; ++i) {
                float acc = p[o.b2 + i];
                for (int j = 0; j < Z; ++j) acc += p[o.W2 + (long)i * Z + j] * z[j];
                u2[i] = acc;
            }
            for (int i = 0; i < V; ++i) {
                float acc = p[o.b3 + i];
                for (int j = 0; j < Z; ++j) acc += p[o.W3 + (long)i * Z + j] * z[j];
                vn[i] = acc;
            }
            for (int i = 0; i < K; ++i) xh[i] = u2[i] <= -t ? -1.f : (u2[i] >= t ? 1.f : u2[i] / t);
            memcpy(v, vn, sizeof(float) * V);
            for (int i = 0; i < K; ++i) tr[(long)l * K + i] = xh[i];
        }
        int flagged;
        const double loss = loss_plain(K, L, tr, xs, xt, first_term, &flagged);
        long long errors = 0;
        for (int i = 0; i < K; ++i) errors += (xh[i] >= 0.f ? 1.0 : -1.0) != xs[i];
        if (loss_out) loss_out[s] = loss;
        if (err_out) err_out[s] = errors;
        if (xhat_out) memcpy(xhat_out + s * (long)L * K, tr, sizeof(double) * (size_t)L * K);
    }
    free(w); free(tr);
    return status;
}

/* ------------------------------------------------------------- backward */
/* backward.cpp:21-29: grad += u_bar (x) in, gated by mask; zero rows skipped */
static void accumulate_outer(double *grad, int rows, int cols, const double *u_bar,
                             const double *in, const double *mask) {
    for (int i = 0; i < rows; ++i) {
        const double g = u_bar[i];
        if (g == 0.0) continue;
        double *grow = grad + (long)i * cols;
        const double *mrow = mask ? mask + (long)i * cols : NULL;
        for (int j = 0; j < cols; ++j) grow[j] += g * in[j] * (mrow ? mrow[j] : 1.0);
    }
}

/* backward.cpp:32-43: out = (W (.) M)^T u, zero entries of u skipped */
static void masked_transpose_apply(const double *W, const double *M, int rows, int cols,
                                   const double *u, double *out) {
    for (int j = 0; j < cols; ++j) out[j] = 0.0;
    for (int i = 0; i < rows; ++i) {
        const double ui = u[i];
        if (ui == 0.0) continue;
        const double *wrow = W + (long)i * cols;
        const double *mrow = M ? M + (long)i * cols : NULL;
        for (int j = 0; j < cols; ++j) out[j] += wrow[j] * (mrow ? mrow[j] : 1.0) * ui;
    }
}

/* model.cpp:45-51 */
static double soft_sign_du(double u, double t) { return (u >= -t && u < t) ? 1.0 / t : 0.0; }
static double soft_sign_dt(double u, double t) { return (u >= -t && u < t) ? -u / (t * t) : 0.0; }

/* backward.cpp:105-165 for one sample, accumulating into grads (record layout) */
static void backward_data(const or_model *m, const double *G, const double *x,
                          const double *xt, const double *xhat /* [L+1][K] */,
                          const double *in /* [L][IN] */, const double *u1 /* [L][Z] */,
                          const double *z /* [L][Z] */, const double *u2 /* [L][K] */,
                          double *grads) {
    const int K = m->n_tx, Z = m->z_dim, V = m->v_dim, IN = 3 * K + V, L = m->depth;
    const rec_off o = offsets(K, Z, V);
    double denom = 0.0;
    for (int i = 0; i < K; ++i) {
        const double d = x[i] - xt[i];
        denom += d * d;
    }
    if (denom < 1e-12) denom = 1e-12;
    double a_bar[256], v_bar[1024], u2_bar[256], z_bar[4096], z_bar3[4096], u1_bar[4096];
    double in_bar[1024], a_prev[256];
    for (int i = 0; i < K; ++i) a_bar[i] = 0.0;
    for (int i = 0; i < V; ++i) v_bar[i] = 0.0;
    for (int l = L - 1; l >= m->frozen_prefix; --l) {
        const double *p = m->params + l * o.size;
        const double *mk = m->masks ? m->masks + l * o.size : NULL;
        double *g = grads + l * o.size;
        const int k_idx = l + 1;
        const double t = p[o.t];
        const double w = 2.0 * log((double)k_idx) / denom;
        for (int i = 0; i < K; ++i) a_bar[i] += w * (xhat[k_idx * K + i] - x[i]);
        double t_bar = 0.0;
        for (int i = 0; i < K; ++i) {
            u2_bar[i] = a_bar[i] * soft_sign_du(u2[l * K + i], t);
            t_bar += a_bar[i] * soft_sign_dt(u2[l * K + i], t);
        }
        g[o.t] += t_bar;
        accumulate_outer(g + o.W2, K, Z, u2_bar, z + (long)l * Z, mk ? mk + o.W2 : NULL);
        for (int i = 0; i < K; ++i) g[o.b2 + i] += u2_bar[i] * (mk ? mk[o.b2 + i] : 1.0);
        masked_transpose_apply(p + o.W2, mk ? mk + o.W2 : NULL, K, Z, u2_bar, z_bar);
        masked_transpose_apply(p + o.W3, mk ? mk + o.W3 : NULL, V, Z, v_bar, z_bar3);
        for (int i = 0; i < Z; ++i) z_bar[i] += z_bar3[i];
        accumulate_outer(g + o.W3, V, Z, v_bar, z + (long)l * Z, mk ? mk + o.W3 : NULL);
        for (int i = 0; i < V; ++i) g[o.b3 + i] += v_bar[i] * (mk ? mk[o.b3 + i] : 1.0);
        for (int i = 0; i < Z; ++i) u1_bar[i] = u1[(long)l * Z + i] > 0.0 ? z_bar[i] : 0.0;
        accumulate_outer(g + o.W1, Z, IN, u1_bar, in + (long)l * IN, mk ? mk + o.W1 : NULL);
        for (int i = 0; i < Z; ++i) g[o.b1 + i] += u1_bar[i] * (mk ? mk[o.b1 + i] : 1.0);
        masked_transpose_apply(p + o.W1, mk ? mk + o.W1 : NULL, Z, IN, u1_bar, in_bar);
        for (int i = 0; i < K; ++i) { /* a_prev = matvec(G, gx_bar) */
            double acc = 0.0;
            for (int j = 0; j < K; ++j) acc += G[i * K + j] * in_bar[2 * K + j];
            a_prev[i] = acc;
        }
        for (int i = 0; i < K; ++i) a_prev[i] += in_bar[K + i];
        memcpy(a_bar, a_prev, sizeof(double) * K);
        for (int i = 0; i < V; ++i) v_bar[i] = in_bar[3 * K + i];
    }
}

static double sign0(double w) { return w > 0.0 ? 1.0 : (w < 0.0 ? -1.0 : 0.0); }

/* backward.cpp:169-173 */
static void add_l1_grad(double *grad, const double *W, const double *M, long n, double scale) {
    for (long i = 0; i < n; ++i) grad[i] += scale * sign0(W[i]) * (M ? M[i] : 1.0);
}

/* backward.cpp:175-199 */
static void add_group_grad(double *grad, const double *W, const double *M, int rows, int cols,
                           double *bgrad, const double *b, const double *mb, double scale) {
    for (int j = 0; j < cols; ++j) {
        double sq = 0.0;
        for (int i = 0; i < rows; ++i) {
            const double w = W[i * cols + j] * (M ? M[i * cols + j] : 1.0);
            sq += w * w;
        }
        if (sq == 0.0) continue;
        const double inv = scale / sqrt(sq);
        for (int i = 0; i < rows; ++i)
            grad[i * cols + j] += inv * W[i * cols + j] * (M ? M[i * cols + j] : 1.0);
    }
    double sq = 0.0;
    for (int i = 0; i < rows; ++i) {
        const double w = b[i] * (mb ? mb[i] : 1.0);
        sq += w * w;
    }
    if (sq > 0.0) {
        const double inv = scale / sqrt(sq);
        for (int i = 0; i < rows; ++i) bgrad[i] += inv * b[i] * (mb ? mb[i] : 1.0);
    }
}

/* backward.cpp:201-220 (scale = 1) */
static void backward_regularizer(const or_model *m, const or_loss_spec *spec, double *grads) {
    if (spec->kind == OR_LOSS_PLAIN) return;
    const int K = m->n_tx, Z = m->z_dim, V = m->v_dim, IN = 3 * K + V;
    const rec_off o = offsets(K, Z, V);
    for (int l = m->frozen_prefix; l < m->depth; ++l) {
        const double *p = m->params + l * o.size;
        const double *mk = m->masks ? m->masks + l * o.size : NULL;
        double *g = grads + l * o.size;
#define MK(off) (mk ? mk + (off) : NULL)
        if (spec->kind == OR_LOSS_L1) {
            add_l1_grad(g + o.W1, p + o.W1, MK(o.W1), (long)Z * IN, spec->lambda);
            add_l1_grad(g + o.W2, p + o.W2, MK(o.W2), (long)K * Z, spec->lambda);
            add_l1_grad(g + o.W3, p + o.W3, MK(o.W3), (long)V * Z, spec->lambda);
        } else {
            add_group_grad(g + o.W1, p + o.W1, MK(o.W1), Z, IN, g + o.b1, p + o.b1, MK(o.b1), spec->lambda1);
            add_group_grad(g + o.W2, p + o.W2, MK(o.W2), K, Z, g + o.b2, p + o.b2, MK(o.b2), spec->lambda1);
            add_group_grad(g + o.W3, p + o.W3, MK(o.W3), V, Z, g + o.b3, p + o.b3, MK(o.b3), spec->lambda1);
            add_l1_grad(g + o.W1, p + o.W1, MK(o.W1), (long)Z * IN, spec->lambda2);
            add_l1_grad(g + o.W2, p + o.W2, MK(o.W2), (long)K * Z, spec->lambda2);
            add_l1_grad(g + o.W3, p + o.W3, MK(o.W3), (long)V * Z, spec->lambda2);
        }
#undef MK
    }
}

/* loss.cpp:35-91 */
static double masked_l1(const double *W, const double *M, long n) {
    double acc = 0.0;
    for (long i = 0; i < n; ++i) acc += fabs(W[i]) * (M ? M[i] : 1.0);
    return acc;
}
static double group_norm_sum(const double *W, const double *M, int rows, int cols,
                             const double *b, const double *mb) {
    double acc = 0.0;
    for (int j = 0; j < cols; ++j) {
        double sq = 0.0;
        for (int i = 0; i < rows; ++i) {
            const double w = W[i * cols + j] * (M ? M[i * cols + j] : 1.0);
            sq += w * w;
        }
        acc += sqrt(sq);
    }
    double sq = 0.0;
    for (int i = 0; i < rows; ++i) {
        const double w = b[i] * (mb ? mb[i] : 1.0);
        sq += w * w;
    }
    return acc + sqrt(sq);
}

double or_regularizer(const or_model *m, const or_loss_spec *spec) {
    if (spec->kind == OR_LOSS_PLAIN) return 0.0;
    const int K = m->n_tx, Z = m->z_dim, V = m->v_dim, IN = 3 * K + V;
    const rec_off o = offsets(K, Z, V);
    double groups = 0.0, elems = 0.0;
    for (int l = 0; l < m->depth; ++l) {
        const double *p = m->params + l * o.size;
        const double *mk = m->masks ? m->masks + l * o.size : NULL;
#define MK(off) (mk ? mk + (off) : NULL)
        if (spec->kind == OR_LOSS_SGL)
            groups += group_norm_sum(p + o.W1, MK(o.W1), Z, IN, p + o.b1, MK(o.b1)) +
                      group_norm_sum(p + o.W2, MK(o.W2), K, Z, p + o.b2, MK(o.b2)) +
                      group_norm_sum(p + o.W3, MK(o.W3), V, Z, p + o.b3, MK(o.b3));
        elems += masked_l1(p + o.W1, MK(o.W1), (long)Z * IN) + masked_l1(p + o.W2, MK(o.W2), (long)K * Z) +
                 masked_l1(p + o.W3, MK(o.W3), (long)V * Z);
#undef MK
    }
    if (spec->kind == OR_LOSS_L1) return spec->lambda * elems;
    return spec->lambda1 * groups + spec->lambda2 * elems;
}

/* kernels.cpp:77-91, 160-200 (ref:: twin 248-272) */
int or_batch_gradient(const or_model *m, long n, const double *H, const double *y,
                      const double *x, const or_loss_spec *spec, int trainable_only,
                      double *grads, double *data_loss, long long *errors, long long *symbols,
                      long long *flagged) {
    const int K = m->n_tx, N = m->n_rx, Z = m->z_dim, V = m->v_dim, IN = 3 * K + V,
              L = m->depth;
    const rec_off o = offsets(K, Z, V);
    const long P = o.size;
    if (n < 1) return 1;
    const int first = trainable_only ? m->frozen_prefix + 1 : 1;
    memset(grads, 0, sizeof(double) * (size_t)L * P);
    const int blocks = n < 16 ? (int)n : 16;
    double *partial = (double *)malloc(sizeof(double) * (size_t)L * P);
    double *xhat = (double *)malloc(sizeof(double) * (size_t)(L + 1) * K);
    double *vv = (double *)malloc(sizeof(double) * (size_t)(L + 1) * V);
    double *in = (double *)malloc(sizeof(double) * (size_t)L * IN);
    double *u1 = (double *)malloc(sizeof(double) * (size_t)L * Z);
    double *z = (double *)malloc(sizeof(double) * (size_t)L * Z);
    double *u2 = (double *)malloc(sizeof(double) * (size_t)L * K);
    double *loss = (double *)malloc(sizeof(double) * n);
    long long *err = (long long *)malloc(sizeof(long long) * n);
    int *flag = (int *)malloc(sizeof(int) * n);
    double q[256], G[4096], xt[256];
    int status = 0;
    for (int b = 0; b < blocks && !status; ++b) {
        memset(partial, 0, sizeof(double) * (size_t)L * P);
        const long lo = (long)((long long)n * b / blocks);
        const long hi = (long)((long long)n * (b + 1) / blocks);
        for (long s = lo; s < hi; ++s) {
            const double *Hs = H + s * (long)N * K, *ys = y + s * (long)N, *xs = x + s * (long)K;
            if (or_preprocess(N, K, Hs, ys, q, G, xt)) { status = 2; break; }
            for (int i = 0; i < K; ++i) xhat[i] = 0.0;
            for (int i = 0; i < V; ++i) vv[i] = 0.0;
            for (int l = 0; l < L; ++l)
                or_layer(m, l, q, G, xhat + l * K, vv + l * V, xhat + (l + 1) * K,
                         vv + (l + 1) * V, in + (long)l * IN, u1 + (long)l * Z,
                         z + (long)l * Z, u2 + l * K);
            int fl = 0;
            loss[s] = loss_plain(K, L, xhat + K, xs, xt, first, &fl);
            flag[s] = fl;
            long long e = 0;
            for (int i = 0; i < K; ++i) e += (xhat[L * K + i] >= 0.0 ? 1.0 : -1.0) != xs[i];
            err[s] = e;
            backward_data(m, G, xs, xt, xhat, in, u1, z, u2, partial);
        }
        if (status) break;
        /* grads.add_scaled(partials[b], 1.0) (backward.cpp:47-61) */
        for (int l = m->frozen_prefix; l < L; ++l)
            for (long i = 0; i < P; ++i) grads[l * P + i] += 1.0 * partial[l * P + i];
    }
    if (!status) {
        const double sc = 1.0 / (double)n;
        for (int l = m->frozen_prefix; l < L; ++l)
            for (long i = 0; i < P; ++i) grads[l * P + i] *= sc;
        backward_regularizer(m, spec, grads);
        double dl = 0.0;
        long long e = 0, f = 0;
        for (long s = 0; s < n; ++s) { dl += loss[s]; e += err[s]; f += flag[s]; }
        *data_loss = dl / (double)n;
        *errors = e;
        *symbols = (long long)n * K;
        *flagged = f;
    }
    free(partial); free(xhat); free(vv); free(in); free(u1); free(z); free(u2);
    free(loss); free(err); free(flag);
    return status;
}

/* adam.cpp:23-79 */
static void update_span(double *w, const double *g, double *m, double *v, const double *mask,
                        long n, double lr, double b1, double b2, double eps, double bc1,
                        double bc2) {
    for (long i = 0; i < n; ++i) {
        if (mask && mask[i] == 0.0) continue;
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        const double mhat = m[i] / bc1;
        const double vhat = v[i] / bc2;
        w[i] -= lr * mhat / (sqrt(vhat) + eps);
    }
}

void or_adam_step(int K, int Z, int V, int depth, int frozen_prefix, double *params,
                  const double *masks, const double *grads, double *m, double *v,
                  int64_t *step, const or_adam_config *c) {
    const rec_off o = offsets(K, Z, V);
    const long P = o.size;
    const double lr = c->lr0 * pow(c->decay_factor, (double)(*step / c->decay_step));
    *step += 1;
    const double bc1 = 1.0 - pow(c->beta1, (double)*step);
    const double bc2 = 1.0 - pow(c->beta2, (double)*step);
    for (int l = frozen_prefix; l < depth; ++l) {
        double *p = params + l * P;
        const double *mk = masks ? masks + l * P : NULL;
        const double *g = grads + l * P;
        double *ml = m + l * P, *vl = v + l * P;
        /* W1, W2, W3, b1, b2, b3 each as its own masked span, then t unmasked */
        const long offs[6] = {o.W1, o.W2, o.W3, o.b1, o.b2, o.b3};
        const long lens[6] = {o.b1 - o.W1, o.b2 - o.W2, o.b3 - o.W3,
                              o.W2 - o.b1, o.W3 - o.b2, o.t - o.b3};
        for (int k = 0; k < 6; ++k)
            update_span(p + offs[k], g + offs[k], ml + offs[k], vl + offs[k],
                        mk ? mk + offs[k] : NULL, lens[k], lr, c->beta1, c->beta2, c->eps, bc1,
                        bc2);
        update_span(p + o.t, g + o.t, ml + o.t, vl + o.t, NULL, 1, lr, c->beta1, c->beta2,
                    c->eps, bc1, bc2);
        if (p[o.t] < 1e-3) p[o.t] = 1e-3;
    }
}

/* compression.cpp:120-129 */
long long or_flops_per_detection(const or_model *m, int include_preprocess) {
    const long long k = m->n_tx, n = m->n_rx;
    const int K = m->n_tx, Z = m->z_dim, V = m->v_dim, IN = 3 * K + V;
    const rec_off o = offsets(K, Z, V);
    long long flops = 0;
    for (int l = 0; l < m->depth; ++l) {
        long long nnz = 0;
        const double *mk = m->masks ? m->masks + l * o.size : NULL;
        const long spans[3][2] = {{o.W1, (long)Z * IN}, {o.W2, (long)K * Z}, {o.W3, (long)V * Z}};
        for (int s = 0; s < 3; ++s)
            for (long i = 0; i < spans[s][1]; ++i) nnz += mk ? (mk[spans[s][0] + i] != 0.0) : 1;
        flops += 2 * nnz + 2 * k * k;
    }
    if (include_preprocess) flops += 2 * n * k + 2 * n * k * k;
    return flops;
}

/* ---------------------------------------------------------------- O32 ---
 * FP32 restatement of batch_gradient (kernels.cpp:160-200) for calibrating
 * FP32's own spread against the FP64 reference over a training run
 * (SURVEY 7.1 step 0 / H7): the preprocessing (q, G, x_tilde, denominator)
 * stays FP64 and exact, as the GPU's training preprocessing does; every
 * per-sample forward (model.cpp:103-120) and reverse-sweep
 * (backward.cpp:105-165) operation is FP32 in the reference's order; each of
 * the min(16, n) blocks accumulates its samples' gradients in FP32 (the GPU
 * accumulates 256-sample splits in FP32); block merge, 1/n scaling and the
 * regularizer gradient are FP64 (backward_regularizer above). Blocks run in
 * parallel (OpenMP) with the same fixed merge order, so results do not depend
 * on the thread count. */
static void backward_data_f32(int K, int Z, int V, int L, int lf, const float *wm /* [L][P] W(.)M */,
                              const float *msk /* [L][P] masks or NULL */, const float *tp /* [L] t */,
                              const float *G, const float *x, double denom,
                              const float *xhat /* [L+1][K] */, const float *in, const float *z,
                              const float *u2, float *grads, const rec_off o) {
    const int IN = 3 * K + V;
    float a_bar[256], v_bar[1024], u2_bar[256], z_bar[4096], z_bar3[4096], u1_bar[4096];
    float in_bar[1024], a_prev[256];
    for (int i = 0; i < K; ++i) a_bar[i] = 0.f;
    for (int i = 0; i < V; ++i) v_bar[i] = 0.f;
    for (int l = L - 1; l >= lf; --l) {
        const float *p = wm + l * o.size;
        const float *mk = msk ? msk + l * o.size : NULL;
        float *g = grads + l * o.size;
        const float t = tp[l];
        const float w = (float)(2.0 * log((double)(l + 1)) / denom);
        for (int i = 0; i < K; ++i) a_bar[i] += w * (xhat[(l + 1) * K + i] - x[i]);
        float t_bar = 0.f;
        for (int i = 0; i < K; ++i) {
            const float u = u2[l * K + i];
            const int lin = u >= -t && u < t;
            u2_bar[i] = lin ? a_bar[i] * (1.f / t) : 0.f;
            t_bar += lin ? a_bar[i] * (-u / (t * t)) : 0.f;
        }
        g[o.t] += t_bar;
        for (int i = 0; i < K; ++i) {
            const float gg = u2_bar[i];
            if (gg == 0.f) continue;
            for (int j = 0; j < Z; ++j) g[o.W2 + i * Z + j] += gg * z[l * Z + j] * (mk ? mk[o.W2 + i * Z + j] : 1.f);
            g[o.b2 + i] += gg * (mk ? mk[o.b2 + i] : 1.f);
        }
        for (int j = 0; j < Z; ++j) { z_bar[j] = 0.f; z_bar3[j] = 0.f; }
        for (int i = 0; i < K; ++i) {
            if (u2_bar[i] == 0.f) continue;
            for (int j = 0; j < Z; ++j) z_bar[j] += p[o.W2 + i * Z + j] * u2_bar[i];
        }
        for (int i = 0; i < V; ++i) {
            if (v_bar[i] == 0.f) continue;
            for (int j = 0; j < Z; ++j) z_bar3[j] += p[o.W3 + i * Z + j] * v_bar[i];
        }
        for (int j = 0; j < Z; ++j) z_bar[j] += z_bar3[j];
        for (int i = 0; i < V; ++i) {
            const float gg = v_bar[i];
            if (gg == 0.f) continue;
            for (int j = 0; j < Z; ++j) g[o.W3 + i * Z + j] += gg * z[l * Z + j] * (mk ? mk[o.W3 + i * Z + j] : 1.f);
            g[o.b3 + i] += gg * (mk ? mk[o.b3 + i] : 1.f);
        }
        for (int i = 0; i < Z; ++i) u1_bar[i] = z[l * Z + i] > 0.f ? z_bar[i] : 0.f;
        for (int i = 0; i < Z; ++i) {
            const float gg = u1_bar[i];
            if (gg == 0.f) continue;
            for (int j = 0; j < IN; ++j) g[o.W1 + (long)i * IN + j] += gg * in[(long)l * IN + j] * (mk ? mk[o.W1 + (long)i * IN + j] : 1.f);
            g[o.b1 + i] += gg * (mk ? mk[o.b1 + i] : 1.f);
        }
        for (int j = 0; j < IN; ++j) in_bar[j] = 0.f;
        for (int i = 0; i < Z; ++i) {
            const float ui = u1_bar[i];
            if (ui == 0.f) continue;
            for (int j = 0; j < IN; ++j) in_bar[j] += p[o.W1 + (long)i * IN + j] * ui;
        }
        for (int i = 0; i < K; ++i) {
            float acc = 0.f;
            for (int j = 0; j < K; ++j) acc += G[i * K + j] * in_bar[2 * K + j];
            a_prev[i] = acc + in_bar[K + i];
        }
        memcpy(a_bar, a_prev, sizeof(float) * K);
        for (int i = 0; i < V; ++i) v_bar[i] = in_bar[3 * K + i];
    }
}

int or_batch_gradient_f32(const or_model *m, long n, const double *H, const double *y,
                          const double *x, const or_loss_spec *spec, int trainable_only,
                          double *grads, double *data_loss, long long *errors, long long *symbols,
                          long long *flagged) {
    const int K = m->n_tx, N = m->n_rx, Z = m->z_dim, V = m->v_dim, IN = 3 * K + V, L = m->depth;
    const rec_off o = offsets(K, Z, V);
    const long P = o.size;
    if (n < 1) return 1;
    const int first = trainable_only ? m->frozen_prefix + 1 : 1;
    const int lf = m->frozen_prefix;
    memset(grads, 0, sizeof(double) * (size_t)L * P);
    const int blocks = n < 16 ? (int)n : 16;
    float *wm = (float *)malloc(sizeof(float) * (size_t)L * P);
    float *msk = m->masks ? (float *)malloc(sizeof(float) * (size_t)L * P) : NULL;
    float *tp = (float *)malloc(sizeof(float) * L);
    for (long i = 0; i < (long)L * P; ++i) {
        wm[i] = (float)(m->params[i] * (m->masks ? m->masks[i] : 1.0));
        if (msk) msk[i] = (float)m->masks[i];
    }
    for (int l = 0; l < L; ++l) tp[l] = (float)m->params[l * P + o.t];
    float *part = (float *)calloc((size_t)blocks * L * P, sizeof(float));
    double *loss = (double *)malloc(sizeof(double) * n);
    long long *err = (long long *)malloc(sizeof(long long) * n);
    int *flag = (int *)malloc(sizeof(int) * n);
    int status = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < blocks; ++b) {
        float *xhat = (float *)malloc(sizeof(float) * (size_t)(L + 1) * K);
        float *in = (float *)malloc(sizeof(float) * (size_t)L * IN);
        float *z = (float *)malloc(sizeof(float) * (size_t)L * Z);
        float *u2 = (float *)malloc(sizeof(float) * (size_t)L * K);
        double q[256], G[4096], xt[256];
        float Gf[4096], qf[256], xf[256], v[1024], vn[1024];
        double *tr = (double *)malloc(sizeof(double) * (size_t)L * K);
        const long lo = (long)((long long)n * b / blocks);
        const long hi = (long)((long long)n * (b + 1) / blocks);
        for (long s = lo; s < hi; ++s) {
            const double *Hs = H + s * (long)N * K, *ys = y + s * (long)N, *xs = x + s * (long)K;
            if (or_preprocess(N, K, Hs, ys, q, G, xt)) {
#pragma omp atomic write
                status = 2;
                break;
            }
            for (int i = 0; i < K; ++i) { qf[i] = (float)q[i]; xf[i] = (float)xs[i]; }
            for (int i = 0; i < K * K; ++i) Gf[i] = (float)G[i];
            for (int i = 0; i < K; ++i) xhat[i] = 0.f;
            for (int i = 0; i < V; ++i) v[i] = 0.f;
            for (int l = 0; l < L; ++l) {
                const float *p = wm + l * P;
                float *inl = in + (long)l * IN;
                for (int i = 0; i < K; ++i) inl[i] = qf[i];
                for (int i = 0; i < K; ++i) inl[K + i] = xhat[l * K + i];
                for (int i = 0; i < K; ++i) {
                    float acc = 0.f;
                    for (int j = 0; j < K; ++j) acc += Gf[i * K + j] * xhat[l * K + j];
                    inl[2 * K + i] = acc;
                }
                for (int i = 0; i < V; ++i) inl[3 * K + i] = v[i];
                float *zl = z + (long)l * Z;
                for (int i = 0; i < Z; ++i) {
                    float acc = p[o.b1 + i];
                    for (int j = 0; j < IN; ++j) acc += p[o.W1 + (long)i * IN + j] * inl[j];
                    zl[i] = acc > 0.f ? acc : 0.f;
                }
                const float t = tp[l];
                for (int i = 0; i < K; ++i) {
                    float acc = p[o.b2 + i];
                    for (int j = 0; j < Z; ++j) acc += p[o.W2 + (long)i * Z + j] * zl[j];
                    u2[l * K + i] = acc;
                    xhat[(l + 1) * K + i] = acc <= -t ? -1.f : (acc >= t ? 1.f : acc / t);
                }
                for (int i = 0; i < V; ++i) {
                    float acc = p[o.b3 + i];
                    for (int j = 0; j < Z; ++j) acc += p[o.W3 + (long)i * Z + j] * zl[j];
                    vn[i] = acc;
                }
                memcpy(v, vn, sizeof(float) * V);
            }
            for (int i = 0; i < L * K; ++i) tr[i] = xhat[K + i];
            int fl = 0;
            loss[s] = loss_plain(K, L, tr, xs, xt, first, &fl);
            flag[s] = fl;
            long long e = 0;
            for (int i = 0; i < K; ++i) e += (xhat[L * K + i] >= 0.f ? 1.0 : -1.0) != xs[i];
            err[s] = e;
            double denom = 0.0;
            for (int i = 0; i < K; ++i) { const double d = xs[i] - xt[i]; denom += d * d; }
            if (denom < 1e-12) denom = 1e-12;
            backward_data_f32(K, Z, V, L, lf, wm, msk, tp, Gf, xf, denom, xhat, in, z, u2,
                              part + (size_t)b * L * P, o);
        }
        free(xhat); free(in); free(z); free(u2); free(tr);
    }
    if (!status) {
        for (int b = 0; b < blocks; ++b)
            for (int l = lf; l < L; ++l)
                for (long i = 0; i < P; ++i) grads[l * P + i] += (double)part[((size_t)b * L + l) * P + i];
        const double sc = 1.0 / (double)n;
        for (int l = lf; l < L; ++l)
            for (long i = 0; i < P; ++i) grads[l * P + i] *= sc;
        backward_regularizer(m, spec, grads);
        double dl = 0.0;
        long long e = 0, f = 0;
        for (long s = 0; s < n; ++s) { dl += loss[s]; e += err[s]; f += flag[s]; }
        *data_loss = dl / (double)n;
        *errors = e;
        *symbols = (long long)n * K;
        *flagged = f;
    }
    free(wm); free(msk); free(tp); free(part); free(loss); free(err); free(flag);
    return status;
}
