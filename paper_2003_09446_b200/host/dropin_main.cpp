// dropin_main.cpp -- exercises the drop-in seam exactly as the reference's
// callers do (training.cpp:63-72, harness.cpp:134-138): reference types,
// reference init_params, generate_batch / batch_evaluate / batch_gradient /
// adam_step from the B200 engine. Prints one JSON object that
// tests/test_dropin_gpu.py checks against the oracle.
#include <cstdio>
#include <vector>

#include "unfold/kernels.hpp"

using namespace unfold;

static void arr(const char *name, const std::vector<double> &v, bool last = false) {
    std::printf("\"%s\": [", name);
    for (size_t i = 0; i < v.size(); ++i) std::printf(i ? ",%.17g" : "%.17g", v[i]);
    std::printf("]%s\n", last ? "" : ",");
}

int main(int argc, char **argv) {
    const int K = argc > 1 ? std::atoi(argv[1]) : 3;
    const int N = argc > 2 ? std::atoi(argv[2]) : 5;
    const int L = argc > 3 ? std::atoi(argv[3]) : 4;
    const int n = argc > 4 ? std::atoi(argv[4]) : 157;
    Rng model_rng(100);
    ModelParams params = init_params(model_rng, K, N, L);
    params.frozen_prefix = 1;
    Rng data_rng(200);
    const std::vector<ChannelSample> batch = generate_batch(data_rng, N, K, n, {4.0, 12.0});
    const BatchEval ev = batch_evaluate(params, batch);
    const BatchEval evt = batch_evaluate(params, batch, LossLayers::trainable_only);
    LossSpec spec;
    spec.kind = LossKind::sparse_group;
    spec.lambda1 = 0.04;
    spec.lambda2 = 0.04;
    Gradients g = make_gradients(params);
    bool have_grads = true;
    BatchEval evg{};
    try {
        evg = batch_gradient(params, batch, spec, g);
    } catch (const std::exception &e) {
        have_grads = false;
        std::fprintf(stderr, "batch_gradient: %s\n", e.what());
    }
    std::vector<double> H, x, y, P, G;
    for (const ChannelSample &s : batch) {
        H.insert(H.end(), s.H.data.begin(), s.H.data.end());
        x.insert(x.end(), s.x.begin(), s.x.end());
        y.insert(y.end(), s.y.begin(), s.y.end());
    }
    for (const LayerParams &lp : params.layers) {
        for (const std::vector<double> *v : {&lp.W1.data, &lp.b1, &lp.W2.data, &lp.b2, &lp.W3.data, &lp.b3})
            P.insert(P.end(), v->begin(), v->end());
        P.push_back(lp.t);
    }
    std::vector<double> P2;
    if (have_grads) {
        for (const LayerGrads &gl : g.layers) {
            if (gl.empty()) {
                const size_t sz = P.size() / params.layers.size();
                G.insert(G.end(), sz, 0.0);
                continue;
            }
            for (const std::vector<double> *v : {&gl.W1.data, &gl.b1, &gl.W2.data, &gl.b2, &gl.W3.data, &gl.b3})
                G.insert(G.end(), v->begin(), v->end());
            G.push_back(gl.t);
        }
        TrainConfig cfg;
        cfg.lr0 = 1e-3;
        AdamState st = make_adam_state(params);
        adam_step(params, g, st, cfg);
        for (const LayerParams &lp : params.layers) {
            for (const std::vector<double> *v : {&lp.W1.data, &lp.b1, &lp.W2.data, &lp.b2, &lp.W3.data, &lp.b3})
                P2.insert(P2.end(), v->begin(), v->end());
            P2.push_back(lp.t);
        }
    }
    std::printf("{\"K\": %d, \"N\": %d, \"L\": %d, \"n\": %d,\n", K, N, L, n);
    std::printf("\"eval\": [%.17g, %lld, %lld, %lld],\n", ev.data_loss, ev.symbol_errors, ev.symbols, ev.flagged);
    std::printf("\"eval_trainable\": [%.17g, %lld],\n", evt.data_loss, evt.symbol_errors);
    std::printf("\"grad_eval\": [%.17g, %lld],\n", evg.data_loss, evg.symbol_errors);
    std::printf("\"train_steps\": %lld,\n", static_cast<long long>(params.train_steps));
    arr("params", P);
    arr("grads", G);
    arr("params_after_adam", P2);
    arr("H", H);
    arr("x", x);
    arr("y", y, true);
    std::printf("}\n");
    return 0;
}
