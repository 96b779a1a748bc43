// unfold_b200_adam.cpp -- drop-in replacement for proj/src/adam.cpp
// (proj/include/unfold/adam.hpp:7-37): the Adam update runs on the device
// through detnet_adam_step (include/detnet_b200.h); the schedule and state
// helpers keep the reference semantics:
//   lr = lr0 * decay^floor(step / decay_step) with the pre-increment step,
//   bias-corrected moments, masked entries (and their moments) untouched,
//   t unmasked and clamped to >= 1e-3, frozen layers skipped.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "detnet_b200.h"
#include "unfold/adam.hpp"

namespace unfold {

void TrainConfig::validate() const {
    const bool ok = lr0 > 0 && decay_factor > 0 && decay_step > 0 && batch_size > 0 &&
                    total_batches > 0 && adam_beta1 > 0 && adam_beta1 < 1 && adam_beta2 > 0 &&
                    adam_beta2 < 1 && adam_eps > 0;
    if (!ok)
        throw ConfigError("TrainConfig: all optimizer settings must be positive (betas in (0,1))");
    if (snr_hi_db < snr_lo_db) throw ConfigError("TrainConfig: snr range must satisfy lo <= hi");
}

AdamState make_adam_state(const ModelParams &params) {
    AdamState s;
    s.m = make_gradients(params);
    s.v = make_gradients(params);
    return s;
}

double learning_rate(const TrainConfig &config, int64_t step) {
    const int64_t stairs = step / config.decay_step;
    return config.lr0 * std::pow(config.decay_factor, static_cast<double>(stairs));
}

namespace {

detnet_ctx *adam_ctx() {
    static detnet_ctx *ctx = [] {
        detnet_ctx *c = nullptr;
        const int rc = detnet_ctx_create(0, &c);
        if (rc) throw std::runtime_error(std::string("detnet_b200: ") + detnet_last_error());
        return c;
    }();
    return ctx;
}

// layer-record packing of one Gradients-shaped object (frozen slots -> zeros)
void pack_grads(const Gradients &g, long P, std::vector<double> &out) {
    out.assign(static_cast<size_t>(P) * g.layers.size(), 0.0);
    for (size_t l = 0; l < g.layers.size(); ++l) {
        const LayerGrads &gl = g.layers[l];
        if (gl.empty()) continue;
        double *r = out.data() + l * P;
        long off = 0;
        for (const std::vector<double> *v :
             {&gl.W1.data, &gl.b1, &gl.W2.data, &gl.b2, &gl.W3.data, &gl.b3}) {
            std::memcpy(r + off, v->data(), sizeof(double) * v->size());
            off += static_cast<long>(v->size());
        }
        r[off] = gl.t;
    }
}

void unpack_grads(const std::vector<double> &in, long P, Gradients &g) {
    for (size_t l = 0; l < g.layers.size(); ++l) {
        LayerGrads &gl = g.layers[l];
        if (gl.empty()) continue;
        const double *r = in.data() + l * P;
        long off = 0;
        for (std::vector<double> *v : {&gl.W1.data, &gl.b1, &gl.W2.data, &gl.b2, &gl.W3.data, &gl.b3}) {
            std::memcpy(v->data(), r + off, sizeof(double) * v->size());
            off += static_cast<long>(v->size());
        }
        gl.t = r[off];
    }
}

} // namespace

void adam_step(ModelParams &params, const Gradients &grads, AdamState &state,
               const TrainConfig &config) {
    const long P = detnet_record_size(params.n_tx, params.dims.z_dim, params.dims.v_dim);
    const int L = params.depth();
    for (int l = params.frozen_prefix; l < L; ++l)
        require(!grads.layers[l].empty() && !state.m.layers[l].empty(),
                "adam_step: gradient/state shape mismatch");
    std::vector<double> p(static_cast<size_t>(P) * L), mk(static_cast<size_t>(P) * L, 1.0), g, m1, m2;
    for (int l = 0; l < L; ++l) {
        const LayerParams &lp = params.layers[l];
        double *r = p.data() + static_cast<size_t>(l) * P;
        double *mr = mk.data() + static_cast<size_t>(l) * P;
        long off = 0;
        const std::vector<double> *vs[6] = {&lp.W1.data, &lp.b1, &lp.W2.data, &lp.b2, &lp.W3.data, &lp.b3};
        const std::vector<double> *ms[6] = {&lp.M1.data, &lp.mb1, &lp.M2.data, &lp.mb2, &lp.M3.data, &lp.mb3};
        for (int k = 0; k < 6; ++k) {
            std::memcpy(r + off, vs[k]->data(), sizeof(double) * vs[k]->size());
            std::memcpy(mr + off, ms[k]->data(), sizeof(double) * ms[k]->size());
            off += static_cast<long>(vs[k]->size());
        }
        r[off] = lp.t;
    }
    pack_grads(grads, P, g);
    pack_grads(state.m, P, m1);
    pack_grads(state.v, P, m2);
    detnet_adam_config cfg{config.lr0, config.decay_factor, config.decay_step, config.adam_beta1,
                           config.adam_beta2, config.adam_eps};
    int64_t step = state.step;
    const int rc = detnet_adam_step(adam_ctx(), params.n_tx, params.dims.z_dim, params.dims.v_dim, L,
                                    params.frozen_prefix, p.data(), mk.data(), g.data(), m1.data(),
                                    m2.data(), &step, &cfg);
    if (rc == DETNET_ERR_CONTRACT) throw ContractError(detnet_last_error());
    if (rc) throw std::runtime_error(std::string("detnet_b200: ") + detnet_last_error());
    state.step = step;
    unpack_grads(m1, P, state.m);
    unpack_grads(m2, P, state.v);
    for (int l = params.frozen_prefix; l < L; ++l) {
        LayerParams &lp = params.layers[l];
        const double *r = p.data() + static_cast<size_t>(l) * P;
        long off = 0;
        for (std::vector<double> *v : {&lp.W1.data, &lp.b1, &lp.W2.data, &lp.b2, &lp.W3.data, &lp.b3}) {
            std::memcpy(v->data(), r + off, sizeof(double) * v->size());
            off += static_cast<long>(v->size());
        }
        lp.t = r[off];
    }
    params.train_steps += 1;
}

} // namespace unfold
