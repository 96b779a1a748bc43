// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, compiled by
// oracle/Makefile from /root/reference/proj/src with -Dunfold=unfold_ref into
// oracle/_ref/libunfold_ref.so. Python tests (ctypes) and bench.py's
// reference arm call the reference's own batch-kernel API through these.
// Flat layouts match oracle/detnet_oracle.h ("layer records").
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "unfold/compression.hpp"
#include "unfold/kernels.hpp"

using namespace unfold;

extern "C" {

struct ref_model {
    int n_tx, n_rx, z_dim, v_dim, depth, frozen_prefix;
    const double *params;
    const double *masks;
};

struct ref_loss_spec {
    int kind;
    double lambda, lambda1, lambda2;
};

struct ref_adam_config {
    double lr0, decay_factor;
    int decay_step;
    double beta1, beta2, eps;
};
}

namespace {

std::string g_msg;

long record_size(int K, int Z, int V) {
    const long IN = 3L * K + V;
    return Z * IN + Z + (long)K * Z + K + (long)V * Z + V + 1;
}

ModelParams to_params(const ref_model &m) {
    ModelParams p;
    p.n_tx = m.n_tx;
    p.n_rx = m.n_rx;
    p.dims = param_dims(m.n_tx, m.z_dim, m.v_dim);
    p.frozen_prefix = m.frozen_prefix;
    const int K = m.n_tx, Z = m.z_dim, V = m.v_dim, IN = p.dims.in_dim;
    const long P = record_size(K, Z, V);
    for (int l = 0; l < m.depth; ++l) {
        const double *r = m.params + l * P;
        const double *mk = m.masks ? m.masks + l * P : nullptr;
        LayerParams lp;
        auto take_m = [&](Matrix &dst, int rows, int cols, const double *src) {
            dst = Matrix(rows, cols);
            std::memcpy(dst.data.data(), src, sizeof(double) * rows * cols);
        };
        auto take_v = [&](Vec &dst, int n, const double *src) { dst.assign(src, src + n); };
        long off = 0;
        take_m(lp.W1, Z, IN, r + off);
        if (mk) take_m(lp.M1, Z, IN, mk + off); else { lp.M1 = Matrix(Z, IN); std::fill(lp.M1.data.begin(), lp.M1.data.end(), 1.0); }
        off += (long)Z * IN;
        take_v(lp.b1, Z, r + off);
        if (mk) take_v(lp.mb1, Z, mk + off); else lp.mb1.assign(Z, 1.0);
        off += Z;
        take_m(lp.W2, K, Z, r + off);
        if (mk) take_m(lp.M2, K, Z, mk + off); else { lp.M2 = Matrix(K, Z); std::fill(lp.M2.data.begin(), lp.M2.data.end(), 1.0); }
        off += (long)K * Z;
        take_v(lp.b2, K, r + off);
        if (mk) take_v(lp.mb2, K, mk + off); else lp.mb2.assign(K, 1.0);
        off += K;
        take_m(lp.W3, V, Z, r + off);
        if (mk) take_m(lp.M3, V, Z, mk + off); else { lp.M3 = Matrix(V, Z); std::fill(lp.M3.data.begin(), lp.M3.data.end(), 1.0); }
        off += (long)V * Z;
        take_v(lp.b3, V, r + off);
        if (mk) take_v(lp.mb3, V, mk + off); else lp.mb3.assign(V, 1.0);
        off += V;
        lp.t = r[off];
        lp.refresh_mask_flag();
        p.layers.push_back(std::move(lp));
    }
    return p;
}

void from_params(const ModelParams &p, double *out) {
    const long P = record_size(p.n_tx, p.dims.z_dim, p.dims.v_dim);
    for (int l = 0; l < p.depth(); ++l) {
        double *r = out + l * P;
        const LayerParams &lp = p.layers[l];
        long off = 0;
        auto put = [&](const std::vector<double> &v) {
            std::memcpy(r + off, v.data(), sizeof(double) * v.size());
            off += (long)v.size();
        };
        put(lp.W1.data); put(lp.b1); put(lp.W2.data); put(lp.b2); put(lp.W3.data); put(lp.b3);
        r[off] = lp.t;
    }
}

void from_grads(const Gradients &g, int K, int Z, int V, double *out) {
    const long P = record_size(K, Z, V);
    for (size_t l = 0; l < g.layers.size(); ++l) {
        double *r = out + l * P;
        const LayerGrads &gl = g.layers[l];
        if (gl.empty()) { std::memset(r, 0, sizeof(double) * P); continue; }
        long off = 0;
        auto put = [&](const std::vector<double> &v) {
            std::memcpy(r + off, v.data(), sizeof(double) * v.size());
            off += (long)v.size();
        };
        put(gl.W1.data); put(gl.b1); put(gl.W2.data); put(gl.b2); put(gl.W3.data); put(gl.b3);
        r[off] = gl.t;
    }
}

void to_grads(const double *in, int K, int Z, int V, Gradients &g) {
    const long P = record_size(K, Z, V);
    for (size_t l = 0; l < g.layers.size(); ++l) {
        const double *r = in + l * P;
        LayerGrads &gl = g.layers[l];
        if (gl.empty()) continue;
        long off = 0;
        auto get = [&](std::vector<double> &v) {
            std::memcpy(v.data(), r + off, sizeof(double) * v.size());
            off += (long)v.size();
        };
        get(gl.W1.data); get(gl.b1); get(gl.W2.data); get(gl.b2); get(gl.W3.data); get(gl.b3);
        gl.t = r[off];
    }
}

std::vector<ChannelSample> to_samples(int N, int K, long n, const double *H, const double *y,
                                      const double *x) {
    std::vector<ChannelSample> b(n);
    for (long s = 0; s < n; ++s) {
        b[s].H = Matrix(N, K);
        std::memcpy(b[s].H.data.data(), H + s * (long)N * K, sizeof(double) * N * K);
        b[s].y.assign(y + s * (long)N, y + (s + 1) * (long)N);
        b[s].x.assign(x + s * (long)K, x + (s + 1) * (long)K);
        b[s].sigma2 = 0.0;
    }
    return b;
}

LossSpec to_spec(const ref_loss_spec *s) {
    LossSpec spec;
    if (!s) return spec;
    spec.kind = s->kind == 0 ? LossKind::plain : (s->kind == 1 ? LossKind::element_l1 : LossKind::sparse_group);
    spec.lambda = s->lambda;
    spec.lambda1 = s->lambda1;
    spec.lambda2 = s->lambda2;
    return spec;
}

template <class F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const ContractError &e) { g_msg = e.what(); return 1; }
    catch (const SingularMatrixError &e) { g_msg = e.what(); return 2; }
    catch (const ConfigError &e) { g_msg = e.what(); return 3; }
    catch (const CapacityError &e) { g_msg = e.what(); return 6; }
    catch (const std::exception &e) { g_msg = e.what(); return 9; }
}

} // namespace

extern "C" {

const char *ref_last_error() { return g_msg.c_str(); }
int ref_worker_count() { return worker_count(); }

void *ref_rng_new(uint64_t seed, uint64_t stream_id) { return new Rng(seed, stream_id); }
void ref_rng_free(void *r) { delete static_cast<Rng *>(r); }
void *ref_rng_stream(void *r, uint64_t id) { return new Rng(static_cast<Rng *>(r)->stream(id)); }
void *ref_rng_split(void *r) { return new Rng(static_cast<Rng *>(r)->split()); }
uint64_t ref_rng_state(void *r) { return static_cast<Rng *>(r)->state(); }
uint64_t ref_rng_next_u64(void *r) { return static_cast<Rng *>(r)->next_u64(); }
double ref_rng_next_uniform(void *r) { return static_cast<Rng *>(r)->next_uniform(); }
double ref_rng_next_gaussian(void *r) { return static_cast<Rng *>(r)->next_gaussian(); }
int ref_rng_next_bit(void *r) { return static_cast<Rng *>(r)->next_bit(); }

// generate_batch (kernels.cpp:116-136) or its ref:: twin (225-236).
int ref_generate_batch(void *rng, int n_rx, int n_tx, int count, double lo, double hi,
                       double *H, double *x, double *y, double *sigma2, int parallel) {
    return guarded([&] {
        Rng &r = *static_cast<Rng *>(rng);
        const SnrRange snr{lo, hi};
        std::vector<ChannelSample> b = parallel ? generate_batch(r, n_rx, n_tx, count, snr)
                                                : ref::generate_batch(r, n_rx, n_tx, count, snr);
        for (int s = 0; s < count; ++s) {
            std::memcpy(H + (long)s * n_rx * n_tx, b[s].H.data.data(), sizeof(double) * n_rx * n_tx);
            std::memcpy(x + (long)s * n_tx, b[s].x.data(), sizeof(double) * n_tx);
            std::memcpy(y + (long)s * n_rx, b[s].y.data(), sizeof(double) * n_rx);
            if (sigma2) sigma2[s] = b[s].sigma2;
        }
    });
}

// batch_evaluate (kernels.cpp:138-158) / ref::batch_evaluate (240-246).
// out4 = {data_loss, symbol_errors, symbols, flagged}
int ref_batch_evaluate(const ref_model *m, long n, const double *H, const double *y,
                       const double *x, int trainable_only, int parallel, double *data_loss,
                       long long *out3) {
    return guarded([&] {
        const ModelParams p = to_params(*m);
        const auto batch = to_samples(m->n_rx, m->n_tx, n, H, y, x);
        const LossLayers ll = trainable_only ? LossLayers::trainable_only : LossLayers::all;
        const BatchEval ev = parallel ? batch_evaluate(p, batch, ll) : ref::batch_evaluate(p, batch, ll);
        *data_loss = ev.data_loss;
        out3[0] = ev.symbol_errors;
        out3[1] = ev.symbols;
        out3[2] = ev.flagged;
    });
}

// forward (model.cpp:124-128) on one sample: x_hat [L+1][K], v [L+1][V],
// optional in [L][IN], u1/z [L][Z], u2 [L][K].
int ref_forward(const ref_model *m, const double *H, const double *y, double *xhat, double *v,
                double *in, double *u1, double *z, double *u2) {
    return guarded([&] {
        const ModelParams p = to_params(*m);
        Matrix Hm(m->n_rx, m->n_tx);
        std::memcpy(Hm.data.data(), H, sizeof(double) * m->n_rx * m->n_tx);
        const Vec yv(y, y + m->n_rx);
        const ForwardTrace tr = forward(p, Hm, yv);
        const int K = m->n_tx, V = m->v_dim, Z = m->z_dim, IN = p.dims.in_dim;
        for (int l = 0; l <= m->depth; ++l) {
            std::memcpy(xhat + (long)l * K, tr.x_hat[l].data(), sizeof(double) * K);
            if (v) std::memcpy(v + (long)l * V, tr.v[l].data(), sizeof(double) * V);
        }
        for (int l = 0; l < m->depth; ++l) {
            if (in) std::memcpy(in + (long)l * IN, tr.in[l].data(), sizeof(double) * IN);
            if (u1) std::memcpy(u1 + (long)l * Z, tr.u1[l].data(), sizeof(double) * Z);
            if (z) std::memcpy(z + (long)l * Z, tr.z[l].data(), sizeof(double) * Z);
            if (u2) std::memcpy(u2 + (long)l * K, tr.u2[l].data(), sizeof(double) * K);
        }
    });
}

// zf_decode (channel.cpp:34-36)
int ref_zf_decode(int n_rx, int n_tx, const double *H, const double *y, double *out) {
    return guarded([&] {
        Matrix Hm(n_rx, n_tx);
        std::memcpy(Hm.data.data(), H, sizeof(double) * n_rx * n_tx);
        const Vec r = zf_decode(Hm, Vec(y, y + n_rx));
        std::memcpy(out, r.data(), sizeof(double) * n_tx);
    });
}

// batch_baseline_errors (kernels.cpp:202-223) / ref:: twin; kind 0 zf, 1 ml, 2 oracle
int ref_baseline_errors(int kind, long n, int n_rx, int n_tx, const double *H, const double *y,
                        const double *x, int parallel, long long *errors, long long *symbols) {
    return guarded([&] {
        const auto batch = to_samples(n_rx, n_tx, n, H, y, x);
        const BaselineKind k = kind == 0 ? BaselineKind::zf : (kind == 1 ? BaselineKind::ml : BaselineKind::oracle);
        const auto r = parallel ? batch_baseline_errors(batch, k) : ref::batch_baseline_errors(batch, k);
        *errors = r.first;
        *symbols = r.second;
    });
}

// prune (compression.cpp:87-94): masks out in the record layout (t slot 1)
int ref_prune(const ref_model *m, int kind, double eta, double eta1, double eta2, double *masks_out) {
    return guarded([&] {
        ModelParams p = to_params(*m);
        PruneSpec spec;
        spec.kind = kind == 0 ? PruneKind::element : (kind == 1 ? PruneKind::group : PruneKind::sparse_group);
        spec.eta = eta;
        spec.eta1 = eta1;
        spec.eta2 = eta2;
        prune(p, spec);
        const long P = record_size(m->n_tx, m->z_dim, m->v_dim);
        for (int l = 0; l < p.depth(); ++l) {
            double *r = masks_out + l * P;
            const LayerParams &lp = p.layers[l];
            long off = 0;
            auto put = [&](const std::vector<double> &v) {
                std::memcpy(r + off, v.data(), sizeof(double) * v.size());
                off += (long)v.size();
            };
            put(lp.M1.data); put(lp.mb1); put(lp.M2.data); put(lp.mb2); put(lp.M3.data); put(lp.mb3);
            r[off] = 1.0;
        }
    });
}

// cost_report (compression.cpp:131-159): out8 = {layer_count, params_total,
// params_nonzero, memory_dense, memory_sparse, flops, flops_dense, preprocess};
// per_layer [L][3] = {params_total, params_nonzero, flops}
int ref_cost_report(const ref_model *m, long long *out8, long long *per_layer) {
    return guarded([&] {
        const CostReport r = cost_report(to_params(*m));
        const long long v[8] = {r.layer_count, r.params_total, r.params_nonzero, r.memory_dense_bytes,
                                r.memory_sparse_bytes, r.flops, r.flops_dense, r.preprocess_flops};
        std::memcpy(out8, v, sizeof v);
        for (size_t l = 0; l < r.per_layer.size(); ++l) {
            per_layer[3 * l] = r.per_layer[l].params_total;
            per_layer[3 * l + 1] = r.per_layer[l].params_nonzero;
            per_layer[3 * l + 2] = r.per_layer[l].flops;
        }
    });
}

// batch_gradient (kernels.cpp:160-200) / ref:: twin (248-272). grads out in
// layer-record layout (frozen records zero).
int ref_batch_gradient(const ref_model *m, long n, const double *H, const double *y,
                       const double *x, const ref_loss_spec *spec, int trainable_only,
                       int parallel, double *grads, double *data_loss, long long *out3) {
    return guarded([&] {
        const ModelParams p = to_params(*m);
        const auto batch = to_samples(m->n_rx, m->n_tx, n, H, y, x);
        const LossLayers ll = trainable_only ? LossLayers::trainable_only : LossLayers::all;
        Gradients g = make_gradients(p);
        const LossSpec sp = to_spec(spec);
        const BatchEval ev = parallel ? batch_gradient(p, batch, sp, g, ll)
                                      : ref::batch_gradient(p, batch, sp, g, ll);
        from_grads(g, m->n_tx, m->z_dim, m->v_dim, grads);
        *data_loss = ev.data_loss;
        out3[0] = ev.symbol_errors;
        out3[1] = ev.symbols;
        out3[2] = ev.flagged;
    });
}

double ref_regularizer(const ref_model *m, const ref_loss_spec *spec) {
    return regularizer(to_params(*m), to_spec(spec));
}

long long ref_flops_per_detection(const ref_model *m, int include_preprocess) {
    return flops_per_detection(to_params(*m), include_preprocess != 0);
}

// adam_step (adam.cpp:48-79): params_io updated in place; m/v moments in
// record layout; *step is AdamState::step.
int ref_adam_step(const ref_model *m, double *params_io, const double *grads, double *mom1,
                  double *mom2, int64_t *step, const ref_adam_config *c) {
    return guarded([&] {
        ref_model mm = *m;
        mm.params = params_io;
        ModelParams p = to_params(mm);
        Gradients g = make_gradients(p);
        to_grads(grads, m->n_tx, m->z_dim, m->v_dim, g);
        AdamState st = make_adam_state(p);
        to_grads(mom1, m->n_tx, m->z_dim, m->v_dim, st.m);
        to_grads(mom2, m->n_tx, m->z_dim, m->v_dim, st.v);
        st.step = *step;
        TrainConfig cfg;
        cfg.lr0 = c->lr0;
        cfg.decay_factor = c->decay_factor;
        cfg.decay_step = c->decay_step;
        cfg.adam_beta1 = c->beta1;
        cfg.adam_beta2 = c->beta2;
        cfg.adam_eps = c->eps;
        adam_step(p, g, st, cfg);
        from_params(p, params_io);
        from_grads(st.m, m->n_tx, m->z_dim, m->v_dim, mom1);
        from_grads(st.v, m->n_tx, m->z_dim, m->v_dim, mom2);
        *step = st.step;
    });
}

} // extern "C"
