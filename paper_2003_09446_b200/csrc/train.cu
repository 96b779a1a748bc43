// train.cu -- the training step on the device (BASELINE config 5):
// batch_gradient (kernels.cpp:160-200) = preprocessing + forward with trace +
// reverse sweep + batch contractions + regularizer gradient, and adam_step
// (adam.cpp:48-79). Exposed through detnet_batch_gradient / detnet_adam_step
// (host arrays, the reference seam) and detnet_train_grad / detnet_train_apply
// (device-resident step; raw gradient sums in a caller buffer so ranks can
// all-reduce them between the two calls).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "engine.hpp"
#include "k_train.cuh"
#include "k_train64.cuh"
#include "k_prune.cuh"

namespace detnet {
namespace {

using BwdFn = void (*)(dim3, dim3, size_t, cudaStream_t, const BwdArgs &);

constexpr int BWD_LARGE = 256; // samples per CTA of k_train_bwd (large batches)
template <int K, int Z, int V> constexpr size_t pair_smem() {
    return (static_cast<size_t>(simt_rec(K, Z, V)) + (3 * K + V - K + K + V) * BWP_SAMPLES) * 4 + 64;
}

template <int K, int Z, int V>
void launch_bwd(dim3 g, dim3 b, size_t sm, cudaStream_t st, const BwdArgs &a) {
    if (b.x == BWP_THREADS) {
        k_train_bwd_pair<K, Z, V><<<g, b, pair_smem<K, Z, V>(), st>>>(a);
    } else {
        k_train_bwd<K, Z, V, BWD_LARGE><<<g, b, sm, st>>>(a);
    }
}
template <int K, int Z, int V> int set_bwd_smem() {
    const int bytes = static_cast<int>(2 * simt_rec(K, Z, V) * 4 + 64);
    const bool ok = cudaFuncSetAttribute(k_train_bwd_pair<K, Z, V>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(pair_smem<K, Z, V>())) == cudaSuccess &&
                    cudaFuncSetAttribute(k_train_bwd<K, Z, V, BWD_LARGE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) ==
                        cudaSuccess;
    return ok ? 0 : -1;
}

struct BwdEntry {
    int K, Z, V;
    BwdFn fn;
    int (*prep)();
};
const BwdEntry kBwd[] = {
    {20, 160, 40, launch_bwd<20, 160, 40>, set_bwd_smem<20, 160, 40>},
    {2, 16, 4, launch_bwd<2, 16, 4>, set_bwd_smem<2, 16, 4>},
    {3, 24, 6, launch_bwd<3, 24, 6>, set_bwd_smem<3, 24, 6>},
    {4, 32, 8, launch_bwd<4, 32, 8>, set_bwd_smem<4, 32, 8>},
    {6, 48, 12, launch_bwd<6, 48, 12>, set_bwd_smem<6, 48, 12>},
    {8, 64, 16, launch_bwd<8, 64, 16>, set_bwd_smem<8, 64, 16>},
};

const BwdEntry *find_bwd(int K, int Z, int V) {
    for (const BwdEntry &e : kBwd)
        if (e.K == K && e.Z == Z && e.V == V) return &e;
    return nullptr;
}

struct TrainWs {
    DBuf tr_in, tr_z, tr_u2, tr_xf, u1bar, g23bar, tbar, p1, p23, jobs, raw, grads, colnorm;
    DBuf bstate; // reverse-sweep state between chunks [K+V][ts]
    DBuf gate;   // tcgen05 sweep relu-gate bits [L][5][ts]
    // FP64 reference-order mode (k_train64.cuh)
    DBuf g64, q64, wb, wf, f_in, f_z, f_u2, f_xh, b_u1, b_u2, b_v, b_t, part, s_loss, s_err;
    DBuf objpart;
    cudaStream_t hi = nullptr; // high-priority stream for the sweep chunks
    cudaEvent_t ev[9] = {};
    cudaEvent_t bev[9] = {}; // gradient buckets final (detnet_train_grad_buckets)
    DBuf in_H, in_y, in_x;
};

// one workspace per context (contexts are single-owner); released with it
std::vector<std::pair<detnet_ctx *, TrainWs *>> &train_ws_all() {
    static std::vector<std::pair<detnet_ctx *, TrainWs *>> all;
    return all;
}

std::mutex &train_ws_mu() {
    static std::mutex mu;
    return mu;
}

TrainWs &ws_for(detnet_ctx *c) {
    std::lock_guard<std::mutex> lk(train_ws_mu()); // device-group members run on threads
    auto &all = train_ws_all();
    for (auto &p : all)
        if (p.first == c) return *p.second;
    all.push_back({c, new TrainWs()});
    return *all.back().second;
}

long rec_size(const detnet_model *m) { return record_size(m->K, m->Z, m->V); }

int ensure_train_state(detnet_model *m) {
    if (m->train_ready) return 0;
    if (int rc = quiesce(m->ctx)) return rc;
    const size_t bytes = sizeof(double) * rec_size(m) * m->L;
    if (m->tparams.ensure(bytes) || m->tmasks.ensure(bytes) || m->tm.ensure(bytes) ||
        m->tv.ensure(bytes))
        return fail(DETNET_ERR_CUDA, "training state allocation failed");
    // ordered on the context stream, where every training kernel runs (a
    // pageable cudaMemcpy may return before its DMA lands); staged from the
    // host buffers before each call returns
    cudaStream_t st = m->ctx->stream;
    CK(cudaMemcpyAsync(m->tparams.p, m->params_host.data(), bytes, cudaMemcpyHostToDevice, st));
    if (m->has_masks) {
        CK(cudaMemcpyAsync(m->tmasks.p, m->masks_host.data(), bytes, cudaMemcpyHostToDevice, st));
    } else {
        std::vector<double> ones(rec_size(m) * m->L, 1.0);
        CK(cudaMemcpyAsync(m->tmasks.p, ones.data(), bytes, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st)); // `ones` goes out of scope
    }
    CK(cudaMemsetAsync(m->tm.p, 0, bytes, st));
    CK(cudaMemsetAsync(m->tv.p, 0, bytes, st));
    if (m->tstatus.ensure(4 * sizeof(double))) return fail(DETNET_ERR_CUDA, "status allocation failed");
    const double st0[4] = {0.0, 0.0, 0.0, 0.0};
    CK(cudaMemcpyAsync(m->tstatus.p, st0, sizeof st0, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(static_cast<double *>(m->tstatus.p) + 2, 0xff, 8, st)); // halt step = -1
    CK(cudaStreamSynchronize(st)); // st0 is a local
    m->diverged_step = -1;
    m->adam_step = 0;
    m->train_ready = true;
    return 0;
}

// FP64 training step in the reference's operation order (k_train64.cuh):
// raw = the merged 16-block gradient sums of batch_gradient before its 1/n
// scaling, raw[total] = the sample-order loss sum; bit-identical to the
// reference on FP32-representable samples.
int grad_raw64(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
               bool trainable_only, double *raw, detnet_eval *out) {
    detnet_ctx *c = m->ctx;
    if (n < 1) return fail(DETNET_ERR_CONTRACT, "batch_gradient: empty batch");
    if (m->K > 32 || m->Z > 256 || m->V > 64)
        return fail(DETNET_ERR_UNSUPPORTED, "FP64 training mode: n_tx <= 32, z <= 256, v <= 64");
    const int K = m->K, Z = m->Z, V = m->V, L = m->L, IN = 3 * K + V, lf = m->frozen;
    const long P = rec_size(m), total = P * L;
    TrainWs &w = ws_for(c);
    const int nb = static_cast<int>(std::min<long>(16, n));
    const size_t d = sizeof(double);
    if (w.g64.ensure(d * n * K * K) || w.q64.ensure(d * n * K) || w.wb.ensure(d * total) ||
        w.wf.ensure(d * f64_fwd_rec(K, Z, V) * L) || w.f_in.ensure(d * L * n * IN) ||
        w.f_z.ensure(d * L * n * Z) || w.f_u2.ensure(d * L * n * K) || w.f_xh.ensure(d * L * n * K) ||
        w.b_u1.ensure(d * L * n * Z) || w.b_u2.ensure(d * L * n * K) || w.b_v.ensure(d * L * n * V) ||
        w.b_t.ensure(d * L * n) || w.part.ensure(d * nb * total) || w.s_loss.ensure(d * n) ||
        w.s_err.ensure(sizeof(long long) * n))
        return fail(DETNET_ERR_CUDA, "FP64 training workspace allocation failed");
    if (int rc = ensure_ws(c, n, K)) return rc;
    cudaStream_t st = c->stream;
    if (int rc = reset_sing(c, st)) return rc;
    if (int rc = run_pre(m, st, 0, n, n, H, y, x, /*exact=*/true, w.g64.as<double>(), w.q64.as<double>()))
        return rc;
    {
        LaunchScope ls(c, DETNET_K_OTHER, st);
        k_pack64<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
            m->tparams.as<double>(), m->has_masks ? m->tmasks.as<double>() : nullptr, K, Z, V, L,
            w.wb.as<double>(), w.wf.as<double>());
    }
    if (int rc = check_launch()) return rc;
    const unsigned grid = static_cast<unsigned>((n + F64_WARPS - 1) / F64_WARPS);
    {
        Fwd64Args fa{w.g64.as<double>(), w.q64.as<double>(), c->denom.as<double>(),
                     c->xmask.as<uint32_t>(), w.wf.as<double>(), m->lnk_all.as<double>(),
                     K, Z, V, L, trainable_only ? lf + 1 : 1, n, w.f_in.as<double>(),
                     w.f_z.as<double>(), w.f_u2.as<double>(), w.f_xh.as<double>(),
                     w.s_loss.as<double>(), w.s_err.as<long long>()};
        const size_t smem = d * F64_WARPS * f64_fwd_scratch(K, Z, V);
        LaunchScope ls(c, DETNET_K_STACK, st);
        k_fwd64<<<grid, 32 * F64_WARPS, smem, st>>>(fa);
    }
    if (int rc = check_launch()) return rc;
    if (lf < L) {
        Bwd64Args ba{w.g64.as<double>(), c->denom.as<double>(), c->xmask.as<uint32_t>(),
                     w.wb.as<double>(), m->lnk_all.as<double>(), K, Z, V, L, lf, n,
                     w.f_in.as<double>(), w.f_z.as<double>(), w.f_u2.as<double>(),
                     w.f_xh.as<double>(), w.b_u1.as<double>(), w.b_u2.as<double>(),
                     w.b_v.as<double>(), w.b_t.as<double>()};
        const size_t smem = d * F64_WARPS * f64_bwd_scratch(K, Z, V);
        {
            LaunchScope ls(c, DETNET_K_BACKWARD, st);
            k_bwd64<<<grid, 32 * F64_WARPS, smem, st>>>(ba);
        }
        if (int rc = check_launch()) return rc;
        Dw64Args da{w.b_u1.as<double>(), w.b_u2.as<double>(), w.b_v.as<double>(), w.f_in.as<double>(),
                    w.f_z.as<double>(), m->has_masks ? m->tmasks.as<double>() : nullptr,
                    K, Z, V, L, lf, n, nb, w.part.as<double>()};
        const int mt = (std::max({Z, K, V}) + DW64_T - 1) / DW64_T;
        const int nt = (std::max(IN, Z) + 1 + DW64_T - 1) / DW64_T;
        {
            LaunchScope ls(c, DETNET_K_BACKWARD, st);
            k_dw64<<<dim3(nt, mt, static_cast<unsigned>((L - lf) * 3 * nb)), 256, 0, st>>>(da);
        }
        if (int rc = check_launch()) return rc;
        {
            LaunchScope ls(c, DETNET_K_BACKWARD, st);
            const int jobs = (L - lf) * nb;
            k_tsum64<<<(jobs + 127) / 128, 128, 0, st>>>(w.b_t.as<double>(), L, lf, n, nb, Z, K, V,
                                                        w.part.as<double>());
        }
        if (int rc = check_launch()) return rc;
    }
    {
        LaunchScope ls(c, DETNET_K_BACKWARD, st);
        k_merge64<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(w.part.as<double>(), L, lf,
                                                                             P, nb, raw);
    }
    if (int rc = check_launch()) return rc;
    double *res = c->result.as<double>();
    {
        LaunchScope ls(c, DETNET_K_REDUCE, st);
        k_reduce64<<<1, 256, 0, st>>>(w.s_loss.as<double>(), w.s_err.as<long long>(),
                                      c->flag.as<uint8_t>(), n, res, reinterpret_cast<long long *>(res + 1),
                                      reinterpret_cast<long long *>(res + 2), raw + total);
    }
    if (int rc = check_launch()) return rc;
    if (!out) return drain_times(c, false), 0;
    CK(cudaMemcpyAsync(res + 3, c->sing.p, 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(c->h_result, res, 32, cudaMemcpyDeviceToHost, st));
    return finish_host(m, n, out);
}

// Forward with trace + reverse sweep + contractions -> raw gradient sums
// (record layout, unscaled, unmasked) in `raw`; local BatchEval in *out.
// Buckets (detnet_train_grad_buckets): raw ranges [lo, hi) final when the
// event fires, in the order the reverse sweep produces them.
struct Buckets {
    int cap = 0, count = 0;
    void **events = nullptr;
    long *ranges = nullptr; // [2 b], [2 b + 1]
};

int grad_raw(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
             bool trainable_only, double *raw, detnet_eval *out, double *chunk_raw = nullptr,
             Buckets *bk = nullptr) {
    detnet_ctx *c = m->ctx;
    if (c->train_fp64) return grad_raw64(m, n, H, y, x, trainable_only, raw, out);
    const BwdEntry *be = find_bwd(m->K, m->Z, m->V);
    if (!be) return fail(DETNET_ERR_UNSUPPORTED, "no backward kernel for these dims");
    if (n < 1) return fail(DETNET_ERR_CONTRACT, "batch_gradient: empty batch");
    const int K = m->K, Z = m->Z, V = m->V, L = m->L, IN = 3 * K + V, O = K + V;
    const int lf = m->frozen;
    const long tiles = (n + TILE - 1) / TILE, ts = tiles * TILE;
    TrainWs &w = ws_for(c);
    const int splits = static_cast<int>((n + DW_SPLIT - 1) / DW_SPLIT);
    // one CTA per SM: small batches use 64-sample CTAs to reach more SMs
    // small batches: two threads per sample, 64 samples per CTA (k_train_bwd_pair)
    // launch shape (and with it the FP32 summation order of the sweep) as for
    // a batch of variant_tiles tiles: device groups pass the global batch
    const long variant_tiles = c->variant_n > 0 ? (c->variant_n + TILE - 1) / TILE : tiles;
    const bool bwd_large = variant_tiles * TILE / BWD_LARGE >= c->sms;
    // one gradient bucket: layers [l0, l1) summed and signalled on the context stream
    auto bucket_sum = [&](int l0, int l1) -> int {
        if (bk->count + 1 >= bk->cap) return fail(DETNET_ERR_CONTRACT, "train_grad_buckets: too few slots");
        const long P = rec_size(m);
        SumArgs sa{w.p1.as<double>(), w.p23.as<double>(), w.tbar.as<double>(),
                   static_cast<int>(ts / 32), splits, K, Z, V, L, lf, raw, chunk_raw, l0, l1};
        const long cnt = P * (l1 - l0);
        {
            LaunchScope ls(c, DETNET_K_BACKWARD, c->stream);
            k_grad_sum<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, c->stream>>>(sa);
        }
        if (int rc = check_launch()) return rc;
        cudaEvent_t &e = w.bev[bk->count];
        if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(e, c->stream));
        bk->events[bk->count] = e;
        bk->ranges[2 * bk->count] = P * l0;
        bk->ranges[2 * bk->count + 1] = P * l1;
        ++bk->count;
        return 0;
    };
    const int bwd_samples = bwd_large ? BWD_LARGE : BWP_SAMPLES;
    const int bwd_per = bwd_large ? BWD_LARGE : BWP_THREADS;
    const int bwd_blocks = static_cast<int>((tiles * TILE + bwd_samples - 1) / bwd_samples);
    if (w.tr_in.ensure(sizeof(float) * L * IN * ts) || w.tr_z.ensure(sizeof(float) * L * Z * ts) ||
        w.tr_u2.ensure(sizeof(float) * L * K * ts) || w.tr_xf.ensure(sizeof(float) * K * ts) ||
        w.u1bar.ensure(sizeof(float) * L * Z * ts) || w.g23bar.ensure(sizeof(float) * L * O * ts) ||
        w.tbar.ensure(sizeof(double) * L * (ts / 32)) ||
        w.p1.ensure(sizeof(double) * L * splits * Z * (IN + 1)) ||
        w.p23.ensure(sizeof(double) * L * splits * O * (Z + 1)) ||
        w.jobs.ensure(sizeof(DwJob) * 2 * L))
        return fail(DETNET_ERR_CUDA, "training workspace allocation failed");
    if (int rc = ensure_ws(c, n, K)) return rc;
    if (int rc = reset_sing(c, c->stream)) return rc;
    // FP32 mode: the one-pass K1 (FP32 Cholesky denominators, <= 1e-4 relative, median
    // 6e-7; flagged samples fall back to the exact LU) -- each sample's gradient is
    // weighted by 1/denom, far inside the FP32 noise of the sweep. The FP64 mode and
    // detnet_ctx_set_exact_preprocess keep the reference's LU for every sample.
    if (int rc = run_pre(m, c->stream, 0, n, n, H, y, x, /*exact=*/false)) return rc;
    TraceBufs tb{w.tr_in.as<float>(), w.tr_z.as<float>(), w.tr_u2.as<float>(), w.tr_xf.as<float>(),
                 ts};
    if (int rc = run_stack(m, c->stream, 0, tiles, n, 0, L, trainable_only, nullptr, nullptr,
                           nullptr, &tb))
        return rc;
    if (lf < L) {
        BwdArgs ba{};
        ba.gp = c->gp.as<float>();
        ba.denom = c->denom.as<double>();
        ba.xmask = c->xmask.as<uint32_t>();
        ba.wrec = m->simt.as<float>();
        ba.rec_floats = m->simt_rec;
        ba.lnk = m->lnk_all.as<double>();
        ba.L = L;
        ba.lf = lf;
        ba.n = n;
        ba.n_tiles = tiles;
        ba.ts = ts;
        ba.tr_in = tb.in;
        ba.tr_z = tb.z;
        ba.tr_u2 = tb.u2;
        ba.tr_xf = tb.xf;
        ba.u1bar = w.u1bar.as<float>();
        ba.g23bar = w.g23bar.as<float>();
        ba.tbar_part = w.tbar.as<double>();
        // the reverse sweep runs on tcgen05 (bwd_tc.cu, 3xTF32) for the
        // BASELINE dims; DETNET_BWD_SIMT=1 keeps the CUDA-core kernels. Its
        // weight images follow the device master params (repacked per call).
        static const bool bwd_simt = std::getenv("DETNET_BWD_SIMT") != nullptr;
        const bool bwd_tc = !bwd_simt && K == 20 && Z == 160 && V == 40;
        if (bwd_tc) {
            if (m->bwd_img.ensure(static_cast<size_t>(bwd_tc_image_bytes(L))) ||
                w.gate.ensure(sizeof(uint32_t) * L * 5 * ts))
                return fail(DETNET_ERR_CUDA, "sweep image allocation failed");
            ba.gate = w.gate.as<uint32_t>();
            LaunchScope ls(c, DETNET_K_OTHER, c->stream);
            if (int rc = bwd_tc_pack(m->tparams.as<double>(), m->has_masks ? m->tmasks.as<double>() : nullptr,
                                     L, m->bwd_img.as<unsigned char>(), c->stream))
                return rc;
        }
        auto sweep = [&](cudaStream_t sst, size_t smem) {
            if (bwd_tc) return bwd_tc_launch(ba, m->bwd_img.as<unsigned char>(), c->sms, sst);
            be->fn(dim3(bwd_blocks), dim3(bwd_per), smem, sst, ba);
            return check_launch();
        };
        std::vector<DwJob> jobs;
        for (int l = lf; l < L; ++l) {
            jobs.push_back({w.u1bar.as<float>() + static_cast<long>(l) * Z * ts,
                            w.tr_in.as<float>() + static_cast<long>(l) * IN * ts, Z, IN,
                            w.p1.as<double>() + static_cast<long>(l) * splits * Z * (IN + 1)});
            jobs.push_back({w.g23bar.as<float>() + static_cast<long>(l) * O * ts,
                            w.tr_z.as<float>() + static_cast<long>(l) * Z * ts, O, Z,
                            w.p23.as<double>() + static_cast<long>(l) * splits * O * (Z + 1)});
        }
        CK(cudaMemcpyAsync(w.jobs.p, jobs.data(), sizeof(DwJob) * jobs.size(),
                           cudaMemcpyHostToDevice, c->stream));
        const int mx = std::max(IN, Z) + 1, my = std::max(Z, O);
        // the contractions run on tcgen05 (dw_tc.cu, 3xTF32) when both job
        // shapes fit its tiles; DETNET_DW_SIMT=1 keeps the CUDA-core kernel
        static const bool dw_simt = std::getenv("DETNET_DW_SIMT") != nullptr;
        const bool dw_tc = !dw_simt && Z <= 256 && O <= 256 && IN + 1 <= 176 && Z + 1 <= 176 &&
                           (Z + IN + 7) / 8 <= 36 && (O + Z + 7) / 8 <= 36;
        auto dw_launch = [&](int j0, int j1) { // jobs [j0, j1) on the context stream
            LaunchScope ls(c, DETNET_K_BACKWARD, c->stream);
            if (dw_tc) {
                dw_tc_launch(w.jobs.as<DwJob>(), j0, j1, n, ts, splits, c->stream);
                return;
            }
            k_dw_gemm<<<dim3((mx + DW_TILE - 1) / DW_TILE, (my + DW_TILE - 1) / DW_TILE,
                             static_cast<unsigned>((j1 - j0) * splits)),
                        256, 0, c->stream>>>(w.jobs.as<DwJob>() + j0, n, ts, splits);
        };
        // Small batches: the sweep runs in chunks of layers on a high-priority
        // stream and the dW contractions of each finished chunk run on the
        // context stream meanwhile, on the SMs the sweep leaves idle (79 of 148
        // at batch 5000). Bit-identical to one sweep + one dW launch.
        static const int env_chunks = std::getenv("DETNET_BWD_CHUNKS") ? std::atoi(std::getenv("DETNET_BWD_CHUNKS")) : 4;
        const int nl = L - lf;
        const int chunks = bwd_large ? 1 : std::max(1, std::min({env_chunks, nl, 8}));
        if (chunks > 1) {
            if (!w.hi) {
                int least = 0, greatest = 0;
                CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
                CK(cudaStreamCreateWithPriority(&w.hi, cudaStreamNonBlocking, greatest));
                for (auto &e : w.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            if (w.bstate.ensure(sizeof(float) * (K + V) * ts))
                return fail(DETNET_ERR_CUDA, "training workspace allocation failed");
            ba.state = w.bstate.as<float>();
            CK(cudaEventRecord(w.ev[8], c->stream)); // forward trace + jobs ready
            CK(cudaStreamWaitEvent(w.hi, w.ev[8], 0));
            for (int j = 0; j < chunks; ++j) {
                ba.it_begin = static_cast<int>(static_cast<long>(nl) * j / chunks);
                ba.it_end = static_cast<int>(static_cast<long>(nl) * (j + 1) / chunks);
                {
                    LaunchScope ls(c, DETNET_K_BACKWARD, w.hi);
                    if (int rc = sweep(w.hi, 0)) return rc;
                }
                CK(cudaEventRecord(w.ev[j], w.hi));
                CK(cudaStreamWaitEvent(c->stream, w.ev[j], 0));
                // layers L-1-it for it in [it_begin, it_end): jobs of layers
                // [L - it_end, L - it_begin) (job index 2 (l - lf))
                dw_launch(2 * (L - ba.it_end - lf), 2 * (L - ba.it_begin - lf));
                if (int rc = check_launch()) return rc;
                if (bk) { // this chunk's layers are final: sum them and signal the bucket
                    if (int rc = bucket_sum(L - ba.it_end, L - ba.it_begin)) return rc;
                }
            }
        } else {
            {
                LaunchScope ls(c, DETNET_K_BACKWARD, c->stream);
                if (int rc = sweep(c->stream, 2 * static_cast<size_t>(m->simt_rec) * 4 + 64)) return rc;
            }
            dw_launch(0, static_cast<int>(jobs.size()));
            if (int rc = check_launch()) return rc;
        }
    }
    const long total = rec_size(m) * L;
    if (!bk || bk->count == 0) { // all layers at once (or the unchunked sweep)
        SumArgs sa{w.p1.as<double>(), w.p23.as<double>(), w.tbar.as<double>(),
                   static_cast<int>(ts / 32), splits, K, Z, V, L, lf, raw, chunk_raw, 0, L};
        LaunchScope ls(c, DETNET_K_BACKWARD, c->stream);
        k_grad_sum<<<static_cast<unsigned>((total + 255) / 256), 256, 0, c->stream>>>(sa);
    } else if (lf > 0) { // frozen layers: zero slots (identical on every rank, no bucket)
        SumArgs sa{w.p1.as<double>(), w.p23.as<double>(), w.tbar.as<double>(),
                   static_cast<int>(ts / 32), splits, K, Z, V, L, lf, raw, chunk_raw, 0, lf};
        const long cnt = rec_size(m) * lf;
        LaunchScope ls(c, DETNET_K_BACKWARD, c->stream);
        k_grad_sum<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, c->stream>>>(sa);
    }
    if (int rc = check_launch()) return rc;
    { // raw[total] = this batch's loss sum (fixed tile order): the objective's data term
        double *res = c->result.as<double>();
        LaunchScope ls(c, DETNET_K_REDUCE, c->stream);
        k_reduce<<<1, 1024, 0, c->stream>>>(c->tile_loss.as<double>(), c->tile_err.as<long long>(),
                                           4 * tiles, c->flag.as<uint8_t>(), n, raw + total,
                                           reinterpret_cast<long long *>(res + 4),
                                           reinterpret_cast<long long *>(res + 5),
                                           c->chunks.as<double>());
    }
    c->last_chunks = (tiles + RED_CHUNK_TILES - 1) / RED_CHUNK_TILES;
    if (int rc = check_launch()) return rc;
    if (bk) { // the last bucket: the loss-sum slot (everything, if the sweep was not chunked)
        if (bk->count >= bk->cap) return fail(DETNET_ERR_CONTRACT, "train_grad_buckets: too few slots");
        cudaEvent_t &e = w.bev[bk->count];
        if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(e, c->stream));
        bk->events[bk->count] = e;
        bk->ranges[2 * bk->count] = bk->count ? total : 0;
        bk->ranges[2 * bk->count + 1] = total + 1;
        ++bk->count;
    }
    if (!out) return drain_times(c, false), 0; // no readback requested: no wait
    return finish(m, n, out); // loss / errors / flagged of the forward pass (syncs)
}

// grads = raw * mask / n_global + regularizer gradient
int apply_reg(detnet_model *m, const double *raw, long n_global, const detnet_loss_spec *spec,
              double *grads, bool norms_ready = false) {
    detnet_ctx *c = m->ctx;
    TrainWs &w = ws_for(c);
    const int K = m->K, Z = m->Z, V = m->V, L = m->L, IN = 3 * K + V;
    const int ng = IN + 1 + 2 * (Z + 1);
    const int kind = spec ? spec->kind : 0;
    if (w.colnorm.ensure(sizeof(double) * L * ng)) return fail(DETNET_ERR_CUDA, "alloc colnorm");
    if (kind == 2 && m->frozen < L && !norms_ready) {
        const long groups = static_cast<long>(L - m->frozen) * ng;
        LaunchScope ls(c, DETNET_K_ADAM, c->stream);
        k_group_norms<<<static_cast<unsigned>((groups + 127) / 128), 128, 0, c->stream>>>(
            m->tparams.as<double>(), m->tmasks.as<double>(), K, Z, V, L, m->frozen,
            w.colnorm.as<double>());
    }
    if (int rc = check_launch()) return rc;
    RegArgs ra{raw, m->tparams.as<double>(), m->tmasks.as<double>(), w.colnorm.as<double>(),
               K, Z, V, L, m->frozen, 1.0 / static_cast<double>(n_global), kind,
               spec ? spec->lambda : 0.0, spec ? spec->lambda1 : 0.0, spec ? spec->lambda2 : 0.0,
               grads};
    const long total = rec_size(m) * L;
    {
        LaunchScope ls(c, DETNET_K_ADAM, c->stream);
        k_grad_apply_reg<<<static_cast<unsigned>((total + 255) / 256), 256, 0, c->stream>>>(ra);
    }
    return check_launch();
}

void adam_coefs(const detnet_adam_config *cfg, int64_t &step, double &lr, double &bc1,
                double &bc2) {
    lr = cfg->lr0 * std::pow(cfg->decay_factor, static_cast<double>(step / cfg->decay_step));
    step += 1;
    bc1 = 1.0 - std::pow(cfg->beta1, static_cast<double>(step));
    bc2 = 1.0 - std::pow(cfg->beta2, static_cast<double>(step));
}

int validate_adam(const detnet_adam_config *cfg) {
    if (!cfg || cfg->lr0 <= 0 || cfg->decay_factor <= 0 || cfg->decay_step <= 0 ||
        cfg->beta1 <= 0 || cfg->beta1 >= 1 || cfg->beta2 <= 0 || cfg->beta2 >= 1 || cfg->eps <= 0)
        return fail(DETNET_ERR_CONFIG,
                    "TrainConfig: all optimizer settings must be positive (betas in (0,1))");
    return 0;
}

} // namespace

// cudaFuncSetAttribute is per device: run for every context's device
// (detnet_ctx_create, after cudaSetDevice)
int train_prepare() {
    for (const BwdEntry &e : kBwd)
        if (e.prep()) return fail(DETNET_ERR_CUDA, "cudaFuncSetAttribute (backward smem) failed");
    if (int rc = dw_tc_prepare()) return rc;
    if (int rc = bwd_tc_prepare()) return rc;
    // FP64 mode: per-warp scratch beyond 48 KB at K=20 (up to K=32 supported)
    const int f64_bytes = static_cast<int>(sizeof(double) * F64_WARPS * f64_bwd_scratch(32, 256, 64));
    if (cudaFuncSetAttribute(k_fwd64, cudaFuncAttributeMaxDynamicSharedMemorySize, f64_bytes) !=
            cudaSuccess ||
        cudaFuncSetAttribute(k_bwd64, cudaFuncAttributeMaxDynamicSharedMemorySize, f64_bytes) !=
            cudaSuccess)
        return fail(DETNET_ERR_CUDA, "cudaFuncSetAttribute (FP64 training smem) failed");
    return 0;
}

int pack_simt_device_from(detnet_model *m, const double *params, const double *masks) {
    const long R = simt_rec(m->K, m->Z, m->V) * m->L;
    LaunchScope ls(m->ctx, DETNET_K_ADAM, m->ctx->stream);
    k_pack_simt<<<static_cast<unsigned>((R + 255) / 256), 256, 0, m->ctx->stream>>>(
        params, masks, m->K, m->Z, m->V, m->L, m->simt.as<float>());
    return check_launch();
}

int pack_simt_device(detnet_model *m) {
    return pack_simt_device_from(m, m->tparams.as<double>(), m->tmasks.as<double>());
}

int train_batch_gradient(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
                         const detnet_loss_spec *spec, int trainable_only, double *grads_out,
                         detnet_eval *out) {
    if (!m || !out || !grads_out || (n > 0 && (!H || !y || !x)))
        return fail(DETNET_ERR_CONTRACT, "null argument");
    if (n < 1) return fail(DETNET_ERR_CONTRACT, "batch_gradient: empty batch");
    detnet_ctx *c = m->ctx;
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_train_state(m)) return rc;
    TrainWs &w = ws_for(c);
    const int N = m->N, K = m->K;
    const long total = rec_size(m) * m->L;
    if (w.in_H.ensure(sizeof(float) * n * N * K) || w.in_y.ensure(sizeof(float) * n * N) ||
        w.in_x.ensure(static_cast<size_t>(n) * K) || w.raw.ensure(sizeof(double) * (total + 1)) ||
        w.grads.ensure(sizeof(double) * total))
        return fail(DETNET_ERR_CUDA, "allocation failed");
    CK(cudaMemcpyAsync(w.in_H.p, H, sizeof(float) * n * N * K, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(w.in_y.p, y, sizeof(float) * n * N, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(w.in_x.p, x, static_cast<size_t>(n) * K, cudaMemcpyHostToDevice, c->stream));
    if (int rc = grad_raw(m, n, w.in_H.as<float>(), w.in_y.as<float>(), w.in_x.as<int8_t>(),
                          trainable_only != 0, w.raw.as<double>(), out))
        return rc;
    if (int rc = apply_reg(m, w.raw.as<double>(), n, spec, w.grads.as<double>())) return rc;
    CK(cudaMemcpyAsync(grads_out, w.grads.p, sizeof(double) * total, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    drain_times(c);
    return 0;
}

int grad_host_shard(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
                    int trainable_only, std::vector<double> &chunk_raw,
                    std::vector<double> &chunk_loss, detnet_eval *out) {
    detnet_ctx *c = m->ctx;
    *out = detnet_eval{};
    chunk_raw.clear();
    chunk_loss.clear();
    if (n <= 0) return 0;
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_train_state(m)) return rc;
    TrainWs &w = ws_for(c);
    const int N = m->N, K = m->K;
    const long total = rec_size(m) * m->L;
    const long nc = (n + 8191) / 8192;
    DBuf craw;
    if (w.in_H.ensure(sizeof(float) * n * N * K) || w.in_y.ensure(sizeof(float) * n * N) ||
        w.in_x.ensure(static_cast<size_t>(n) * K) || w.raw.ensure(sizeof(double) * (total + 1)) ||
        craw.ensure(sizeof(double) * nc * total))
        return fail(DETNET_ERR_CUDA, "allocation failed");
    CK(cudaMemcpyAsync(w.in_H.p, H, sizeof(float) * n * N * K, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(w.in_y.p, y, sizeof(float) * n * N, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(w.in_x.p, x, static_cast<size_t>(n) * K, cudaMemcpyHostToDevice, c->stream));
    int rc = grad_raw(m, n, w.in_H.as<float>(), w.in_y.as<float>(), w.in_x.as<int8_t>(),
                      trainable_only != 0, w.raw.as<double>(), out, craw.as<double>());
    if (rc == 0) {
        chunk_raw.resize(static_cast<size_t>(nc) * total);
        chunk_loss.resize(nc);
        if (cudaMemcpy(chunk_raw.data(), craw.p, sizeof(double) * nc * total,
                       cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(chunk_loss.data(), c->chunks.p, sizeof(double) * nc,
                       cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(DETNET_ERR_CUDA, "gradient chunk copy failed");
    }
    craw.release();
    return rc;
}

int apply_reg_host(detnet_model *m, const double *raw_host, long n, const detnet_loss_spec *spec,
                   double *grads_out) {
    detnet_ctx *c = m->ctx;
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_train_state(m)) return rc;
    TrainWs &w = ws_for(c);
    const long total = rec_size(m) * m->L;
    if (w.raw.ensure(sizeof(double) * (total + 1)) || w.grads.ensure(sizeof(double) * total))
        return fail(DETNET_ERR_CUDA, "allocation failed");
    CK(cudaMemcpyAsync(w.raw.p, raw_host, sizeof(double) * total, cudaMemcpyHostToDevice, c->stream));
    if (int rc = apply_reg(m, w.raw.as<double>(), n, spec, w.grads.as<double>())) return rc;
    CK(cudaMemcpyAsync(grads_out, w.grads.p, sizeof(double) * total, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    drain_times(c);
    return 0;
}

int train_adam_step(detnet_ctx *c, int K, int Z, int V, int L, int lf, double *params,
                    const double *masks, const double *grads, double *m1, double *m2,
                    int64_t *step, const detnet_adam_config *cfg) {
    if (!c || !params || !grads || !m1 || !m2 || !step) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (int rc = validate_adam(cfg)) return rc;
    if (L < 1 || lf < 0 || lf > L) return fail(DETNET_ERR_CONTRACT, "bad depth/frozen_prefix");
    CK(cudaSetDevice(c->device));
    const long P = record_size(K, Z, V), total = P * L;
    const size_t bytes = sizeof(double) * total;
    DBuf buf;
    if (buf.ensure(5 * bytes)) return fail(DETNET_ERR_CUDA, "adam buffers");
    double *dp = buf.as<double>(), *dm = dp + total, *dg = dm + total, *d1 = dg + total,
           *d2 = d1 + total;
    CK(cudaMemcpyAsync(dp, params, bytes, cudaMemcpyHostToDevice, c->stream));
    if (masks) CK(cudaMemcpyAsync(dm, masks, bytes, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dg, grads, bytes, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(d1, m1, bytes, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(d2, m2, bytes, cudaMemcpyHostToDevice, c->stream));
    double lr, bc1, bc2;
    int64_t st = *step;
    adam_coefs(cfg, st, lr, bc1, bc2);
    {
        LaunchScope ls(c, DETNET_K_ADAM, c->stream);
        k_adam<<<static_cast<unsigned>((total + 255) / 256), 256, 0, c->stream>>>(
            dp, masks ? dm : nullptr, dg, d1, d2, total, static_cast<int>(P), lf, lr, cfg->beta1,
            cfg->beta2, cfg->eps, bc1, bc2);
    }
    if (int rc = check_launch()) { buf.release(); return rc; }
    cudaMemcpyAsync(params, dp, bytes, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(m1, d1, bytes, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(m2, d2, bytes, cudaMemcpyDeviceToHost, c->stream);
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    buf.release();
    if (e != cudaSuccess) return fail(DETNET_ERR_CUDA, "adam_step: %s", cudaGetErrorString(e));
    drain_times(c);
    *step = st;
    return 0;
}

} // namespace detnet

using namespace detnet;

extern "C" {

long detnet_model_param_count(const detnet_model *m) {
    return m ? record_size(m->K, m->Z, m->V) * m->L : 0;
}

int detnet_train_grad(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
                      int trainable_only, double *raw_dev, detnet_eval *out) {
    if (!m || !raw_dev) return fail(DETNET_ERR_CONTRACT, "null argument");
    CK(cudaSetDevice(m->ctx->device));
    if (int rc = ensure_train_state(m)) return rc;
    return grad_raw(m, n, H, y, x, trainable_only != 0, raw_dev, out);
}

int detnet_train_grad_buckets(detnet_model *m, long n, const float *H, const float *y,
                              const int8_t *x, int trainable_only, double *raw_dev, void **events,
                              long *ranges, int max_buckets) {
    if (!m || !raw_dev || !events || !ranges || max_buckets < 1)
        return -fail(DETNET_ERR_CONTRACT, "null argument");
    if (m->ctx->train_fp64)
        return -fail(DETNET_ERR_UNSUPPORTED, "train_grad_buckets: the FP64 mode is not bucketed");
    if (cudaSetDevice(m->ctx->device) != cudaSuccess) return -fail(DETNET_ERR_CUDA, "cudaSetDevice");
    if (int rc = ensure_train_state(m)) return -rc;
    Buckets bk;
    bk.cap = std::min(max_buckets, 9);
    bk.events = events;
    bk.ranges = ranges;
    if (int rc = grad_raw(m, n, H, y, x, trainable_only != 0, raw_dev, nullptr, nullptr, &bk)) return -rc;
    return bk.count;
}

int detnet_stream_wait_event(void *stream, void *event) {
    if (!event) return fail(DETNET_ERR_CONTRACT, "null event");
    CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0));
    return 0;
}

long detnet_train_raw_count(const detnet_model *m) {
    return m ? record_size(m->K, m->Z, m->V) * m->L + 1 : 0;
}

int detnet_ctx_set_train_precision(detnet_ctx *c, int fp64) {
    if (!c) return fail(DETNET_ERR_CONTRACT, "null context");
    c->train_fp64 = fp64 != 0;
    for (detnet_ctx *g : c->members) g->train_fp64 = c->train_fp64;
    return 0;
}

int detnet_train_apply(detnet_model *m, const double *raw_dev, long n_global,
                       const detnet_loss_spec *spec, const detnet_adam_config *cfg) {
    if (!m || !raw_dev || n_global < 1) return fail(DETNET_ERR_CONTRACT, "bad argument");
    if (spec && (spec->kind < 0 || spec->kind > 2))
        return fail(DETNET_ERR_CONTRACT, "loss spec kind must be 0, 1 or 2");
    if (m->diverged_step >= 0)
        return fail(DETNET_ERR_DIVERGENCE, "train: objective became non-finite at step %lld",
                    m->diverged_step);
    ++m->version; // packed images / layout may change: drop captured evaluate graphs
    m->replicas_stale = !m->replicas.empty();
    if (int rc = validate_adam(cfg)) return rc;
    detnet_ctx *c = m->ctx;
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_train_state(m)) return rc;
    TrainWs &w = ws_for(c);
    const long total = rec_size(m) * m->L;
    if (w.grads.ensure(sizeof(double) * total)) return fail(DETNET_ERR_CUDA, "alloc grads");
    // objective = data_loss + regularizer(params) before the update
    // (training.cpp:65-70); a non-finite one halts the run on the device
    const int IN = 3 * m->K + m->V, ng = IN + 1 + 2 * (m->Z + 1);
    if (w.objpart.ensure(sizeof(double) * 4 * m->L) || w.colnorm.ensure(sizeof(double) * m->L * ng))
        return fail(DETNET_ERR_CUDA, "alloc objective");
    ObjArgs oa{m->tparams.as<double>(), m->has_masks ? m->tmasks.as<double>() : nullptr,
               w.colnorm.as<double>(), m->K, m->Z, m->V, m->L, spec ? spec->kind : 0,
               spec ? spec->lambda : 0.0, spec ? spec->lambda1 : 0.0, spec ? spec->lambda2 : 0.0,
               w.objpart.as<double>()};
    {
        LaunchScope ls(c, DETNET_K_ADAM, c->stream);
        if (oa.kind == 2) { // column norms of every layer: the value's and the gradient's
            const long groups = static_cast<long>(m->L) * ng;
            k_group_norms<<<static_cast<unsigned>((groups + 127) / 128), 128, 0, c->stream>>>(
                m->tparams.as<double>(), m->tmasks.as<double>(), m->K, m->Z, m->V, m->L, 0,
                w.colnorm.as<double>());
        }
        if (oa.kind != 0) k_reg_layers<<<4 * m->L, REG_THREADS, 0, c->stream>>>(oa);
        k_objective<<<1, 1, 0, c->stream>>>(oa, raw_dev + total, static_cast<double>(n_global),
                                            static_cast<long long>(m->adam_step),
                                            m->tstatus.as<double>());
    }
    if (int rc = check_launch()) return rc;
    if (int rc = apply_reg(m, raw_dev, n_global, spec, w.grads.as<double>(), true)) return rc;
    double lr, bc1, bc2;
    adam_coefs(cfg, m->adam_step, lr, bc1, bc2);
    {
        LaunchScope ls(c, DETNET_K_ADAM, c->stream);
        k_adam<<<static_cast<unsigned>((total + 255) / 256), 256, 0, c->stream>>>(
            m->tparams.as<double>(), m->tmasks.as<double>(), w.grads.as<double>(),
            m->tm.as<double>(), m->tv.as<double>(), total, static_cast<int>(rec_size(m)),
            m->frozen, lr, cfg->beta1, cfg->beta2, cfg->eps, bc1, bc2,
            reinterpret_cast<const long long *>(m->tstatus.as<double>() + 2));
    }
    if (int rc = check_launch()) return rc;
    if (int rc = pack_simt_device(m)) return rc;
    // dense tcgen05 images follow the master weights on the device, repacked
    // lazily before their next use (run_stack); other packings (compacted /
    // sparse) are rebuilt from the host copy on demand
    m->tc_dev_dirty = true;
    m->sparse_ready = false; // the CSR stream no longer matches the weights
    // stream-ordered: the next gradient / evaluation on this stream sees the
    // update; nothing here needs the host to wait
    if (int rc = check_launch()) return rc;
    drain_times(c, false);
    return 0;
}

int detnet_train_status(detnet_model *m, double *objective, double *regularizer) {
    if (!m) return fail(DETNET_ERR_CONTRACT, "null argument");
    double st[3] = {0.0, 0.0, 0.0};
    if (m->train_ready) {
        CK(cudaSetDevice(m->ctx->device));
        if (int rc = quiesce(m->ctx)) return rc;
        CK(cudaMemcpy(st, m->tstatus.p, sizeof st, cudaMemcpyDeviceToHost));
        long long halt;
        std::memcpy(&halt, st + 2, 8);
        m->diverged_step = halt;
    }
    if (objective) *objective = st[0];
    if (regularizer) *regularizer = st[1];
    if (m->diverged_step >= 0) // DivergenceError (training.cpp:68-70)
        return fail(DETNET_ERR_DIVERGENCE, "train: objective became non-finite at step %lld",
                    m->diverged_step);
    return 0;
}

int detnet_model_get_params(detnet_model *m, double *out) {
    if (!m || !out) return fail(DETNET_ERR_CONTRACT, "null argument");
    const long total = record_size(m->K, m->Z, m->V) * m->L;
    if (!m->train_ready) {
        std::memcpy(out, m->params_host.data(), sizeof(double) * total);
        return 0;
    }
    if (int rc = quiesce(m->ctx)) return rc;
    CK(cudaMemcpy(out, m->tparams.p, sizeof(double) * total, cudaMemcpyDeviceToHost));
    return 0;
}


// ---- pruning planner ----------------------------------------
// Prunes the device FP64 master weights in place of the masks (bit-identical to
// compression.cpp:43-94), then rebuilds every packed layout -- SIMT records,
// the tcgen05 images (compacted to the live units when few survive) and the
// sparse stream -- from the result. Adam moments and the step counter survive.
int detnet_model_prune(detnet_model *m, int kind, double eta, double eta1, double eta2) {
    if (!m) return fail(DETNET_ERR_CONTRACT, "null argument");
    ++m->version; // packed images / layout may change: drop captured evaluate graphs
    if (int rc = quiesce(m->ctx)) return rc;
    auto frac = [](double v) { return v >= 0.0 && v < 1.0; };
    if (kind < 0 || kind > 2) return fail(DETNET_ERR_CONTRACT, "prune: kind must be 0, 1 or 2");
    if (!frac(eta) || !frac(eta1) || !frac(eta2))
        return fail(DETNET_ERR_CONFIG, "PruneSpec: thresholds must lie in [0, 1)");
    if (3L * m->K + m->V > 1023 || m->Z > 1023)
        return fail(DETNET_ERR_UNSUPPORTED, "prune: layer widths above 1023");
    CK(cudaSetDevice(m->ctx->device));
    if (int rc = ensure_train_state(m)) return rc;
    const long P = record_size(m->K, m->Z, m->V);
    PruneArgs a{m->tparams.as<double>(), m->tmasks.as<double>(), P, m->K, m->Z, m->V, kind,
                eta, eta1, eta2};
    {
        LaunchScope ls(m->ctx, DETNET_K_OTHER, m->ctx->stream);
        k_prune<<<m->L, 256, 0, m->ctx->stream>>>(a);
    }
    if (int rc = check_launch()) return rc;
    const size_t total = static_cast<size_t>(P) * m->L;
    std::vector<double> params(total), masks(total);
    CK(cudaStreamSynchronize(m->ctx->stream));
    CK(cudaMemcpy(params.data(), m->tparams.p, sizeof(double) * total, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(masks.data(), m->tmasks.p, sizeof(double) * total, cudaMemcpyDeviceToHost));
    // The device master copy already holds the pruned weights and masks: the SIMT
    // records are repacked from it on the device; the tcgen05 images are marked
    // stale, so the next tensor-core evaluation compacts them from the host copy
    // (refresh_tc) while a training step switches to the dense device-packed images
    // instead (run_stack) -- the ~10-20 ms of host packing are paid only if and
    // when a compacted evaluation follows, not by every prune.
    m->params_host = std::move(params);
    m->masks_host = std::move(masks);
    m->has_masks = true;
    if (int rc = pack_simt_device(m)) return rc;
    m->tc_stale = true;
    m->tc_dev_dirty = false;
    m->sparse_ready = false;
    if (std::getenv("DETNET_SPARSE_CSR")) { // the table-driven stream is built only on request
        detnet_model_desc d{m->K, m->N, m->Z, m->V, m->L, m->frozen, m->params_host.data(),
                            m->masks_host.data()};
        const int64_t step = m->adam_step;
        if (int rc = upload_model(m, &d)) return rc;
        m->train_ready = true; // device params / masks already hold exactly these values
        m->adam_step = step;
    } else {
        prepare_jit(m, m->params_host.data(), m->masks_host.data());
    }
    m->replicas_stale = !m->replicas.empty();
    CK(cudaStreamSynchronize(m->ctx->stream));
    drain_times(m->ctx);
    return 0;
}

int detnet_model_get_masks(detnet_model *m, double *out) {
    if (!m || !out) return fail(DETNET_ERR_CONTRACT, "null argument");
    const long total = record_size(m->K, m->Z, m->V) * m->L;
    if (m->train_ready) {
        if (int rc = quiesce(m->ctx)) return rc;
        CK(cudaMemcpy(out, m->tmasks.p, sizeof(double) * total, cudaMemcpyDeviceToHost));
    } else if (m->has_masks) {
        std::memcpy(out, m->masks_host.data(), sizeof(double) * total);
    } else {
        std::fill(out, out + total, 1.0);
    }
    return 0;
}

// cost_report (compression.cpp:131-159) of the model as currently masked
int detnet_model_cost_report(detnet_model *m, detnet_cost_report *r, detnet_layer_cost *per_layer) {
    if (!m || !r) return fail(DETNET_ERR_CONTRACT, "null argument");
    const long P = record_size(m->K, m->Z, m->V);
    std::vector<double> mk(static_cast<size_t>(P) * m->L);
    if (int rc = detnet_model_get_masks(m, mk.data())) return rc;
    const long long k = m->K, n = m->N, IN = 3L * m->K + m->V;
    const long W1n = m->Z * IN, W2n = static_cast<long>(m->K) * m->Z, W3n = static_cast<long>(m->V) * m->Z;
    const long oW1 = 0, ob1 = W1n, oW2 = ob1 + m->Z, ob2 = oW2 + W2n, oW3 = ob2 + m->K, ob3 = oW3 + W3n;
    auto ones = [](const double *p, long cnt) {
        long long c = 0;
        for (long i = 0; i < cnt; ++i) c += p[i] != 0.0;
        return c;
    };
    *r = detnet_cost_report{};
    r->layer_count = m->L;
    r->preprocess_flops = 2 * n * k + 2 * n * k * k;
    long long dense_stored = 0, sparse_stored = 0;
    for (int l = 0; l < m->L; ++l) {
        const double *q = mk.data() + static_cast<size_t>(l) * P;
        const long long wt = W1n + W2n + W3n;
        const long long wn = ones(q + oW1, W1n) + ones(q + oW2, W2n) + ones(q + oW3, W3n);
        const long long bn = ones(q + ob1, m->Z) + ones(q + ob2, m->K) + ones(q + ob3, m->V);
        detnet_layer_cost c;
        c.params_total = wt + m->Z + m->K + m->V + 1;
        c.params_nonzero = wn + bn + 1;
        c.flops = 2 * wn + 2 * k * k;
        r->params_total += c.params_total;
        r->params_nonzero += c.params_nonzero;
        r->flops += c.flops;
        r->flops_dense += 2 * wt + 2 * k * k;
        dense_stored += c.params_total;
        sparse_stored += c.params_nonzero;
        if (per_layer) per_layer[l] = c;
    }
    r->flops += r->preprocess_flops;
    r->flops_dense += r->preprocess_flops;
    r->memory_dense_bytes = 4 * dense_stored;
    r->memory_sparse_bytes = 4 * sparse_stored;
    return 0;
}

int detnet_model_reset_adam(detnet_model *m) {
    if (!m) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (!m->train_ready) return 0;
    if (int rc = quiesce(m->ctx)) return rc;
    const size_t bytes = sizeof(double) * record_size(m->K, m->Z, m->V) * m->L;
    CK(cudaMemset(m->tm.p, 0, bytes));
    CK(cudaMemset(m->tv.p, 0, bytes));
    m->adam_step = 0;
    return 0;
}

} // extern "C"

namespace detnet {
// called by detnet_ctx_destroy: the training workspace of a context
void train_ws_release(detnet_ctx *c) {
    std::lock_guard<std::mutex> lk(train_ws_mu());
    auto &all = train_ws_all();
    for (size_t i = 0; i < all.size(); ++i) {
        if (all[i].first != c) continue;
        TrainWs *w = all[i].second;
        for (DBuf *b : {&w->tr_in, &w->tr_z, &w->tr_u2, &w->tr_xf, &w->u1bar, &w->g23bar, &w->tbar,
                        &w->p1, &w->p23, &w->jobs, &w->raw, &w->grads, &w->colnorm, &w->bstate,
                        &w->in_H, &w->in_y, &w->in_x, &w->g64, &w->q64, &w->wb, &w->wf,
                        &w->f_in, &w->f_z, &w->f_u2, &w->f_xh, &w->b_u1, &w->b_u2, &w->b_v,
                        &w->b_t, &w->part, &w->s_loss, &w->s_err, &w->objpart, &w->gate})
            b->release();
        if (w->hi) {
            cudaStreamDestroy(w->hi);
            for (cudaEvent_t e : w->ev) cudaEventDestroy(e);
            for (cudaEvent_t e : w->bev)
                if (e) cudaEventDestroy(e);
        }
        delete w;
        all.erase(all.begin() + static_cast<long>(i));
        return;
    }
}
} // namespace detnet
