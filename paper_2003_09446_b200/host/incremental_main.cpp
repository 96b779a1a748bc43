// incremental_main.cpp -- runs the reference's incremental-depth trainer
// (train_incremental, training.cpp:22-141) unchanged. Linked against the
// B200 seam it trains on the GPU engine; linked against the
// reference's own kernels.cpp/adam.cpp it is the CPU baseline. It then
// round-trips the result through the reference checkpoint format
// (checkpoint.cpp) and re-validates the loaded model. Prints one JSON object.
//
// usage: incremental_main K N start t_step max_layers batches batch_size
//                         val_samples seed ckpt_path
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "unfold/checkpoint.hpp"
#include "unfold/training.hpp"

using namespace unfold;

int main(int argc, char **argv) {
    if (argc < 11) {
        std::fprintf(stderr, "usage: %s K N start t_step max_layers batches batch_size val_samples seed ckpt\n",
                     argv[0]);
        return 2;
    }
    const int K = std::atoi(argv[1]), N = std::atoi(argv[2]);
    IncrementalConfig inc;
    inc.start_layers = std::atoi(argv[3]);
    inc.t_step = std::atoi(argv[4]);
    inc.max_layers = std::atoi(argv[5]);
    inc.halt_epsilon = 0.0; // grow to max_layers: the schedule itself is under test
    inc.val_samples = std::atoi(argv[8]);
    inc.val_snr_db = 10.0;
    TrainConfig cfg;
    cfg.total_batches = std::atoi(argv[6]);
    cfg.batch_size = std::atoi(argv[7]);
    cfg.lr0 = 1e-3;
    cfg.snr_lo_db = 7.0;
    cfg.snr_hi_db = 14.0;
    const uint64_t seed = std::strtoull(argv[9], nullptr, 10);
    const std::string ckpt = argv[10];
    LossSpec spec;
    spec.kind = LossKind::sparse_group;
    spec.lambda1 = 1e-4;
    spec.lambda2 = 0.0;
    ModelSpec model;
    model.n_tx = K;
    model.n_rx = N;
    model.dims = param_dims(K);
    model.init.weight_scale = 1.0;

    const auto t0 = std::chrono::steady_clock::now();
    TrainResult r;
    try {
        r = train_incremental(cfg, spec, inc, model, seed, LossLayers::all, 1000000);
    } catch (const std::exception &e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    save_checkpoint(r.params, "detnet-b200", ckpt);
    const Checkpoint back = load_checkpoint(ckpt);
    bool same = back.params.layers.size() == r.params.layers.size() &&
                back.params.frozen_prefix == r.params.frozen_prefix;
    for (size_t l = 0; same && l < r.params.layers.size(); ++l) {
        const LayerParams &a = r.params.layers[l], &b = back.params.layers[l];
        same = a.W1.data == b.W1.data && a.b1 == b.b1 && a.W2.data == b.W2.data && a.b2 == b.b2 &&
               a.W3.data == b.W3.data && a.b3 == b.b3 && a.t == b.t;
    }
    // validation of the reloaded model on a fresh held-out set
    Rng vr(seed + 17);
    const std::vector<ChannelSample> vs = generate_batch(vr, N, K, inc.val_samples, SnrRange::fixed(10.0));
    const ValidationResult v = validate(back.params, vs);

    std::printf("{\"K\": %d, \"N\": %d, \"seconds\": %.6f, \"halt\": \"%s\", \"flagged\": %lld, "
                "\"ckpt_roundtrip\": %s, \"reloaded_val_loss\": %.17g, \"reloaded_val_ber\": %.17g, "
                "\"optimizer_steps\": %lld, \"steps\": [",
                K, N, secs, r.halt_reason.c_str(), r.flagged_samples, same ? "true" : "false", v.loss,
                v.ber, static_cast<long long>(r.params.train_steps));
    for (size_t i = 0; i < r.steps.size(); ++i) {
        const StepRecord &s = r.steps[i];
        std::printf("%s{\"step\": %d, \"layers\": %d, \"train_loss\": %.17g, \"val_loss\": %.17g, "
                    "\"val_ber\": %.17g}",
                    i ? ", " : "", s.step, s.layer_count, s.train_loss, s.val_loss, s.val_ber);
    }
    std::printf("]}\n");
    return 0;
}
