// incremental.cu -- the incremental-depth trainer (train_incremental,
// training.cpp:22-141) as one device-resident engine call.
//
// The reference's controller keeps ModelParams on the host: through the
// drop-in seam every optimizer step moves FP64 parameters, gradients and Adam
// moments across PCIe. Here the whole schedule runs on the engine: batches
// come from the on-device generator with the reference's keying (master
// Rng(seed): init stream 1, train stream 2, validation stream 3; one
// generate_batch split per batch, kernels.cpp:116-136), the parameters, Adam
// moments and objective stay in HBM (detnet_train_grad / detnet_train_apply,
// objective = data loss + regularizer with the divergence halt), validation
// is detnet_batch_evaluate_device on the device-resident evaluation set, and
// only the step records and, when the depth grows, the appended layers
// (init_layer draws, model.cpp:140-159, made on the host with the reference's
// own Rng arithmetic) cross the bus. The control flow -- a fresh AdamState per
// incremental step (training.cpp:55), the log of the step's mean objective,
// the halting tests in the reference's order (target BER, relative
// improvement below halt_epsilon, max_layers) and freeze + append
// (training.cpp:134-136) -- is the reference's.
#include <chrono>
#include <cmath>
#include <vector>

#include "engine.hpp"

namespace detnet {
namespace {

// Rng (rng.cpp:12-46) on the host, for the init draws
struct HostRng {
    uint64_t s;
    uint64_t next_u64() { return mix64(s += kGamma); }
    double next_uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_gaussian() {
        const double u1 = 1.0 - next_uniform();
        const double u2 = next_uniform();
        // 3.141592653589793 is the double std::numbers::pi denotes (rng.cpp:37)
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
    }
};

// init_layer (model.cpp:140-166) into one layer record: W1, W2, W3 as
// weight_scale / sqrt(fan_in) x N(0,1) in that draw order, zero biases, t0
void init_layer(HostRng &r, int K, int Z, int V, double scale, double t0, double *rec) {
    const int IN = 3 * K + V;
    const long P = record_size(K, Z, V);
    for (long e = 0; e < P; ++e) rec[e] = 0.0;
    auto draw = [&](long off, int rows, int cols) {
        const double std = scale / std::sqrt(static_cast<double>(cols));
        for (long i = 0; i < static_cast<long>(rows) * cols; ++i) rec[off + i] = std * r.next_gaussian();
    };
    const long oW1 = 0, oW2 = static_cast<long>(Z) * IN + Z, oW3 = oW2 + static_cast<long>(K) * Z + K;
    draw(oW1, Z, IN);
    draw(oW2, K, Z);
    draw(oW3, V, Z);
    rec[P - 1] = t0;
}

} // namespace
} // namespace detnet

using namespace detnet;

extern "C" int detnet_train_incremental(detnet_ctx *c, int K, int N, int Z, int V,
                                        const detnet_incremental_config *cfg,
                                        detnet_step_record *records, int max_records,
                                        int *n_records, double *params_out,
                                        detnet_incremental_result *res) {
    if (!c || !cfg || !res || !n_records) return fail(DETNET_ERR_CONTRACT, "null argument");
    *n_records = 0;
    *res = detnet_incremental_result{};
    // IncrementalConfig::validate / TrainConfig::validate (training.cpp:8-14, adam.cpp:7-14)
    if (cfg->start_layers < 1 || cfg->t_step < 1 || cfg->max_layers < cfg->start_layers)
        return fail(DETNET_ERR_CONFIG, "IncrementalConfig: need start_layers >= 1, t_step >= 1, "
                                       "max_layers >= start_layers");
    if (cfg->halt_epsilon < 0.0) return fail(DETNET_ERR_CONFIG, "IncrementalConfig: halt_epsilon must be >= 0");
    if (cfg->val_samples < 1) return fail(DETNET_ERR_CONFIG, "IncrementalConfig: val_samples must be >= 1");
    const detnet_adam_config &ad = cfg->adam;
    if (ad.lr0 <= 0 || ad.decay_factor <= 0 || ad.decay_step <= 0 || cfg->batch_size <= 0 ||
        cfg->total_batches <= 0 || ad.beta1 <= 0 || ad.beta1 >= 1 || ad.beta2 <= 0 ||
        ad.beta2 >= 1 || ad.eps <= 0)
        return fail(DETNET_ERR_CONFIG, "TrainConfig: all optimizer settings must be positive (betas in (0,1))");
    if (cfg->snr_hi_db < cfg->snr_lo_db)
        return fail(DETNET_ERR_CONFIG, "TrainConfig: snr range must satisfy lo <= hi");
    if (!(cfg->weight_scale > 0.0) || cfg->t0 < 1e-3)
        return fail(DETNET_ERR_CONTRACT, "init_params: invalid init options");
    if (N < K || K < 1) return fail(DETNET_ERR_CONFIG, "need N >= K >= 1");
    CK(cudaSetDevice(c->device));
    using clock = std::chrono::steady_clock;
    const auto t_start = clock::now();

    // master Rng(seed) and its streams (training.cpp:37-40)
    const uint64_t master = detnet_rng_seed(cfg->seed, 0);
    HostRng init_rng{detnet_rng_stream(master, 1)};
    uint64_t train_rng = detnet_rng_stream(master, 2);
    uint64_t val_rng = detnet_rng_stream(master, 3);
    const long P = record_size(K, Z, V);
    const double scale = cfg->sample_scale > 0.0 ? cfg->sample_scale : 1.0;

    // evaluation set: generate_batch(val_rng, ..., fixed(val_snr)) on the device
    const long nv = cfg->val_samples, nb = cfg->batch_size;
    DBuf vH, vy, vx, bH, by, bx, raw;
    if (vH.ensure(sizeof(float) * nv * N * K) || vy.ensure(sizeof(float) * nv * N) ||
        vx.ensure(static_cast<size_t>(nv) * K) || bH.ensure(sizeof(float) * nb * N * K) ||
        by.ensure(sizeof(float) * nb * N) || bx.ensure(static_cast<size_t>(nb) * K))
        return fail(DETNET_ERR_CUDA, "incremental: sample buffers");
    auto release = [&]() {
        for (DBuf *b : {&vH, &vy, &vx, &bH, &by, &bx, &raw}) b->release();
    };
    {
        const uint64_t base = detnet_rng_split(&val_rng);
        if (int rc = detnet_generate_device(c, base, 0, nv, N, K, cfg->val_snr_db, cfg->val_snr_db,
                                            scale, vH.as<float>(), vy.as<float>(), vx.as<int8_t>(),
                                            nullptr)) {
            release();
            return rc;
        }
    }
    // init_params(init_rng, K, N, start_layers, dims, init)
    std::vector<double> params(static_cast<size_t>(P) * cfg->start_layers);
    for (int l = 0; l < cfg->start_layers; ++l)
        init_layer(init_rng, K, Z, V, cfg->weight_scale, cfg->t0, params.data() + l * P);
    int depth = cfg->start_layers, frozen = 0;
    detnet_model *m = nullptr;
    detnet_model_desc d{K, N, Z, V, depth, frozen, params.data(), nullptr};
    if (int rc = detnet_model_create(c, &d, &m)) {
        release();
        return rc;
    }
    int rc = 0;
    double prev_val = 0.0;
    long long global_step = 0, flagged = 0;
    for (int step_idx = 0;; ++step_idx) {
        const auto step_t0 = clock::now();
        if ((rc = detnet_model_reset_adam(m))) break; // a fresh AdamState (training.cpp:55)
        if (raw.ensure(sizeof(double) * detnet_train_raw_count(m))) {
            rc = fail(DETNET_ERR_CUDA, "incremental: gradient buffer");
            break;
        }
        double step_obj = 0.0;
        for (int b = 0; b < cfg->total_batches && !rc; ++b) {
            const uint64_t base = detnet_rng_split(&train_rng);
            if ((rc = detnet_generate_device(c, base, 0, nb, N, K, cfg->snr_lo_db, cfg->snr_hi_db,
                                             scale, bH.as<float>(), by.as<float>(), bx.as<int8_t>(),
                                             nullptr)))
                break;
            detnet_eval ev{};
            if ((rc = detnet_train_grad(m, nb, bH.as<float>(), by.as<float>(), bx.as<int8_t>(),
                                        cfg->loss_layers_trainable_only, raw.as<double>(), &ev)))
                break;
            flagged += ev.flagged;
            if ((rc = detnet_train_apply(m, raw.as<double>(), nb, &cfg->spec, &cfg->adam))) break;
            double obj = 0.0;
            if ((rc = detnet_train_status(m, &obj, nullptr))) break; // DivergenceError
            ++global_step;
            step_obj += obj;
        }
        if (rc) break;
        // validation on the evaluation set (training.cpp:89-91)
        detnet_eval ve{};
        if ((rc = detnet_batch_evaluate_device(m, nv, vH.as<float>(), vy.as<float>(), vx.as<int8_t>(),
                                               cfg->loss_layers_trainable_only, nullptr, &ve)))
            break;
        const double val_loss = ve.data_loss;
        const double val_ber = ve.symbols ? static_cast<double>(ve.symbol_errors) / ve.symbols : 0.0;
        if (*n_records < max_records && records) {
            detnet_step_record &r = records[*n_records];
            r.step = step_idx;
            r.layer_count = depth;
            r.train_loss = step_obj / cfg->total_batches;
            r.val_loss = val_loss;
            r.val_ber = val_ber;
            r.wall_ms = std::chrono::duration<double, std::milli>(clock::now() - step_t0).count();
        }
        ++*n_records;
        // halting (training.cpp:117-131)
        if (cfg->target_ber > 0.0 && val_ber <= cfg->target_ber) { res->halt_reason = 0; break; }
        if (step_idx > 0 && cfg->halt_epsilon > 0.0) {
            const double improvement = prev_val > 0.0 ? (prev_val - val_loss) / prev_val : 0.0;
            if (improvement < cfg->halt_epsilon) { res->halt_reason = 1; break; }
        }
        prev_val = val_loss;
        if (depth >= cfg->max_layers) { res->halt_reason = 2; break; }
        // freeze the trained prefix and append fresh layers (training.cpp:134-136)
        const int add = std::min(cfg->t_step, cfg->max_layers - depth);
        params.resize(static_cast<size_t>(P) * (depth + add));
        if ((rc = detnet_model_get_params(m, params.data()))) break;
        for (int l = depth; l < depth + add; ++l)
            init_layer(init_rng, K, Z, V, cfg->weight_scale, cfg->t0, params.data() + l * P);
        frozen = depth;
        depth += add;
        d = detnet_model_desc{K, N, Z, V, depth, frozen, params.data(), nullptr};
        if ((rc = detnet_model_update(m, &d))) break;
    }
    if (!rc) {
        res->flagged_samples = flagged;
        res->optimizer_steps = global_step;
        res->depth = depth;
        res->frozen_prefix = frozen;
        res->seconds = std::chrono::duration<double>(clock::now() - t_start).count();
        if (params_out) rc = detnet_model_get_params(m, params_out);
    }
    detnet_model_destroy(m);
    release();
    return rc;
}
