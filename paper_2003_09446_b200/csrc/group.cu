// group.cu -- one seam call over several devices (detnet_ctx_create_group).
//
// The reference's batch_evaluate / batch_gradient use every host core inside
// one call and give the same bits for any worker count, by fixed-order
// reductions (kernels.cpp:93-103, 144, 160-200; README.md:83-91). The device
// analogue: a group context shards each host-buffer batch over its members
// (one context per device, one host thread each) at 8,192-sample chunk
// boundaries, and every reduction is done in the canonical chunked order the
// single-device kernels already use (k_reduce: loss folded per chunk, then
// over chunks; k_grad_sum: gradient splits folded per chunk, then over
// chunks). The group folds the members' chunk sums in global chunk order, so
// BatchEval and gradients are bit-identical for any group size, including a
// group of one (tests/test_group_gpu.py runs 1, 2, 3 and 8 members).
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace detnet {

namespace {

constexpr long kChunk = 8192; // samples per canonical reduction chunk

struct Shard {
    long s0 = 0, cnt = 0;
};

std::vector<Shard> shards(long n, int G) {
    const long C = (n + kChunk - 1) / kChunk;
    std::vector<Shard> out(G);
    for (int g = 0; g < G; ++g) {
        const long c0 = C * g / G, c1 = C * (g + 1) / G;
        out[g].s0 = std::min(n, c0 * kChunk);
        out[g].cnt = std::min(n, c1 * kChunk) - out[g].s0;
    }
    return out;
}

std::vector<detnet_model *> members_of(detnet_model *m) {
    std::vector<detnet_model *> v{m};
    v.insert(v.end(), m->replicas.begin(), m->replicas.end());
    return v;
}

// Run f(g) on one host thread per member; the first failing member's status
// and message win (in member order).
template <class F> int run_members(int G, F f, std::vector<std::string> &msgs) {
    std::vector<int> rc(G, 0);
    msgs.assign(G, std::string());
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)
        th.emplace_back([&, g] {
            rc[g] = f(g);
            if (rc[g]) msgs[g] = detnet_last_error();
        });
    for (auto &t : th) t.join();
    for (int g = 0; g < G; ++g)
        if (rc[g]) return fail(rc[g], "%s", msgs[g].c_str());
    return 0;
}

} // namespace

int sync_replicas(detnet_model *m) {
    if (!m->replicas_stale) return 0;
    const long total = record_size(m->K, m->Z, m->V) * m->L;
    std::vector<double> p(total), mk(total);
    if (int rc = detnet_model_get_params(m, p.data())) return rc;
    if (int rc = detnet_model_get_masks(m, mk.data())) return rc;
    detnet_model_desc d{m->K, m->N, m->Z, m->V, m->L, m->frozen, p.data(),
                        m->has_masks || m->train_ready ? mk.data() : nullptr};
    for (detnet_model *r : m->replicas)
        if (int rc = detnet_model_update(r, &d)) return rc;
    m->replicas_stale = false;
    return 0;
}

int group_batch_evaluate(detnet_model *m, long n, const float *H, const float *y,
                         const int8_t *x, int trainable_only, float *xhat_out, detnet_eval *out) {
    if (int rc = sync_replicas(m)) return rc;
    const auto mem = members_of(m);
    const int G = static_cast<int>(mem.size());
    const auto sh = shards(n, G);
    const int N = m->N, K = m->K, L = m->L;
    std::vector<detnet_eval> ev(G);
    std::vector<std::vector<double>> chunks(G);
    std::vector<std::string> msgs;
    const int rc = run_members(G, [&](int g) -> int {
        if (!sh[g].cnt) return 0;
        mem[g]->ctx->variant_n = n; // launch shapes as for the whole batch
        const long s0 = sh[g].s0;
        const int r = eval_host(mem[g], sh[g].cnt, H + s0 * N * K, y + s0 * N, x + s0 * K,
                                trainable_only, xhat_out ? xhat_out + s0 * L * K : nullptr, &ev[g],
                                &chunks[g]);
        mem[g]->ctx->variant_n = 0;
        if (r == DETNET_ERR_SINGULAR) // sample index relative to the whole batch
            return fail(r, "solve_normal_equations: matrix is singular to working precision "
                           "(in samples [%ld, %ld))", s0, s0 + sh[g].cnt);
        return r;
    }, msgs);
    if (rc) return rc;
    double loss = 0.0; // the canonical fold over chunks (k_reduce's second level)
    long long err = 0, flg = 0;
    for (int g = 0; g < G; ++g) {
        for (double v : chunks[g]) loss += v;
        err += ev[g].symbol_errors;
        flg += ev[g].flagged;
    }
    out->loss_sum = loss;
    out->data_loss = loss / static_cast<double>(n);
    out->symbol_errors = err;
    out->symbols = n * static_cast<long long>(K);
    out->flagged = flg;
    return 0;
}

int group_batch_gradient(detnet_model *m, long n, const float *H, const float *y,
                         const int8_t *x, const detnet_loss_spec *spec, int trainable_only,
                         double *grads_out, detnet_eval *out) {
    if (!m || !out || !grads_out || (n > 0 && (!H || !y || !x)))
        return fail(DETNET_ERR_CONTRACT, "null argument");
    if (n < 1) return fail(DETNET_ERR_CONTRACT, "batch_gradient: empty batch");
    if (int rc = sync_replicas(m)) return rc;
    const auto mem = members_of(m);
    const int G = static_cast<int>(mem.size());
    const auto sh = shards(n, G);
    const int N = m->N, K = m->K;
    const long total = record_size(m->K, m->Z, m->V) * m->L;
    std::vector<detnet_eval> ev(G);
    std::vector<std::vector<double>> craw(G), closs(G);
    std::vector<std::string> msgs;
    const int rc = run_members(G, [&](int g) -> int {
        if (!sh[g].cnt) return 0;
        mem[g]->ctx->variant_n = n;
        const long s0 = sh[g].s0;
        const int r = grad_host_shard(mem[g], sh[g].cnt, H + s0 * N * K, y + s0 * N, x + s0 * K,
                                      trainable_only, craw[g], closs[g], &ev[g]);
        mem[g]->ctx->variant_n = 0;
        return r;
    }, msgs);
    if (rc) return rc;
    // canonical fold over the global chunk sequence (k_grad_sum's second level)
    std::vector<double> raw(total, 0.0);
    double loss = 0.0;
    long long err = 0, flg = 0;
    for (int g = 0; g < G; ++g) {
        const long nc = static_cast<long>(closs[g].size());
        for (long c = 0; c < nc; ++c) {
            const double *src = craw[g].data() + c * total;
            for (long e = 0; e < total; ++e) raw[e] += src[e];
            loss += closs[g][c];
        }
        err += ev[g].symbol_errors;
        flg += ev[g].flagged;
    }
    if (int r = apply_reg_host(m, raw.data(), n, spec, grads_out)) return r;
    out->loss_sum = loss;
    out->data_loss = loss / static_cast<double>(n);
    out->symbol_errors = err;
    out->symbols = n * static_cast<long long>(K);
    out->flagged = flg;
    return 0;
}

} // namespace detnet

using namespace detnet;

extern "C" int detnet_ctx_create_group(const int *devices, int count, detnet_ctx **out) {
    if (!devices || count < 1 || !out) return fail(DETNET_ERR_CONTRACT, "bad device list");
    detnet_ctx *c = nullptr;
    if (int rc = detnet_ctx_create(devices[0], &c)) return rc;
    for (int g = 1; g < count; ++g) {
        detnet_ctx *mbr = nullptr;
        if (int rc = detnet_ctx_create(devices[g], &mbr)) {
            detnet_ctx_destroy(c);
            return rc;
        }
        c->members.push_back(mbr);
    }
    *out = c;
    return 0;
}

extern "C" int detnet_ctx_group_size(const detnet_ctx *c) {
    return c ? 1 + static_cast<int>(c->members.size()) : 0;
}
