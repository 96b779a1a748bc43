// engine.hpp -- internal host-side state shared by the engine's translation
// units (not part of the C-ABI; see include/detnet_b200.h).
#pragma once

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/detnet_b200.h"
#include "common.cuh"


namespace detnet {

inline thread_local std::string g_err;

inline int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(DETNET_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                  \
    } while (0)

inline long record_size(int K, int Z, int V) {
    const long IN = 3L * K + V;
    return Z * IN + Z + static_cast<long>(K) * Z + K + static_cast<long>(V) * Z + V + 1;
}

// device buffer that only grows
// Bumped on every device (re)allocation: a captured CUDA graph is replayed
// only while no buffer it may reference has moved.
inline std::atomic<long long> g_alloc_epoch{0};

struct DBuf {
    void *p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap) return 0;
        ++g_alloc_epoch;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
        cap = bytes;
        return 0;
    }
    void release() {
        ++g_alloc_epoch;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T> T *as() const { return static_cast<T *>(p); }
};

struct DimsEntry;

// tcgen05 path (stack_tc.cu): packed weights and launch arguments.
struct TcModel {
    bool ready = false;
    int K = 0, Z = 0, V = 0, L = 0;
    int zh = 0;         // hidden rows per packed layer (160 dense | 48 compacted)
    DBuf w;             // [L][rec bytes] pre-laid-out smem images
    long rec_bytes = 0;
    // split-FP16 images (stack_h16.cu): [L][rec16] images, [L][64] bias rows,
    // one int "weight out of FP16 range" flag (set by the device repack)
    bool h16_ready = false;
    int zh16 = 0;       // 160 dense | 64 compacted
    DBuf w16;
    long rec16 = 0;
};

// model-specialised sparse stack (sparse_jit.cu): NVRTC-compiled per model
struct JitModel {
    bool ready = false;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    size_t smem = 0;
    int ctas_per_sm = 1, L = 0, K = 0, attr_device = -1;
    long nnz = 0;           // surviving products per sample over all layers
    double compile_ms = 0;  // NVRTC time of the last build (0 = cache hit)
    std::string log;        // NVRTC / ptxas log (register use)
    long long version = -1; // model version the kernel was generated from
};

struct TcArgs {
    const float *gp;
    const float *q32;
    const double *denom;
    const uint32_t *xmask;
    const double *lnk;
    int l_begin, l_end;
    long n, n_tiles, tile0;
    float *xhat;
    double *tile_loss;    // [global tile][4 lane quadrants]
    long long *tile_err;  // [global tile][4 lane quadrants]
};

int tc_prepare();
int tc_pack(TcModel &tc, int K, int Z, int V, int L, const double *params, const double *masks);
int tc_launch(const TcModel &tc, const TcArgs &a, cudaStream_t st);
struct TraceBufs;
int tc_launch_state(const TcModel &tc, const TcArgs &a, float *xs, float *vs, cudaStream_t st,
                    const TraceBufs *tr = nullptr);
void tc_release(TcModel &tc);
int tc_pack_device(TcModel &tc, const double *params, const double *masks, long P, cudaStream_t st);
// 3xTF32 recompute of the tiles the split-FP16 kernel flagged (redo[tile] = 1);
// returns at once on the device when *redo_count == 0
int tc_launch_redo(const TcModel &tc, const TcArgs &a, float *xs, float *vs, cudaStream_t st,
                   const TraceBufs *tr, const uint8_t *redo, const int *redo_count);

// sparse JIT stack (sparse_jit.cu)
constexpr long kJitMaxNnz = 1500; // path 3: worst layer's surviving products
long jit_layer_nnz(int K, int Z, int V, int L, const double *params, const double *masks, long stop);
int jit_build(JitModel &jm, int K, int Z, int V, int L, const double *params, const double *masks);
int jit_launch(JitModel &jm, const TcArgs &a, cudaStream_t st, int sms, int device);
void jit_release(JitModel &jm);

// split-FP16 layer stack (stack_h16.cu)
int h16_prepare();
int h16_pack(TcModel &tc, int K, int Z, int V, int L, const double *params, const double *masks,
             const std::vector<std::vector<int>> &units, size_t max_alive);
int h16_pack_device(TcModel &tc, const double *params, const double *masks, long P, cudaStream_t st);
int h16_alloc_dense(TcModel &tc, int L, cudaStream_t st);
int tc_pack_dense_device(TcModel &tc, int K, int Z, int V, int L, const double *params,
                         const double *masks, cudaStream_t st);
int h16_launch_state(const TcModel &tc, const TcArgs &a, float *xs, float *vs, cudaStream_t st,
                     const TraceBufs *tr, uint8_t *redo, int *redo_count, int sms);


} // namespace detnet

struct detnet_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    cudaStream_t copy_stream = nullptr;
    int path = 0;
    bool profiling = false;
    long long launches = 0;
    detnet_kernel_times times{};
    struct Pending {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    // workspace
    detnet::DBuf gp, q32, denom, xmask, flag, tile_loss, tile_err, sing, result;
    detnet::DBuf chunks; // per-chunk loss sums of the last reduction (k_reduce)
    long last_chunks = 0; // how many
    detnet::DBuf in_H[2], in_y[2], in_x[2], xhat_dev, state_x, state_v, fb_list, fb_count;
    bool exact_pre = false; // bit-exact reference LU for every sample
    bool train_tc = true;   // training forward on tcgen05 (dense images) instead of SIMT
    bool train_fp64 = false; // FP64 training step in the reference's order (k_train64.cuh)
    // > 0: choose the SIMT forward / reverse-sweep launch shapes as for a
    // batch of this many samples (device-group members use the global batch)
    long variant_n = 0;
    detnet::DBuf redo, redo_count; // split-FP16 range flags per tile + count
    double *h_result = nullptr; // pinned: loss, err, flag, singular
    // asynchronous evaluations (detnet_batch_evaluate_device_async): a ring of
    // pinned result slots, each with the event that marks its copy done
    static constexpr int kSlots = 64;
    double *h_async = nullptr; // [kSlots][4]
    cudaEvent_t async_ev[kSlots] = {};
    struct AsyncSlot {
        long long ticket = -1;
        long n = 0;
        int K = 0;
    } slots[kSlots];
    long long next_ticket = 0;
    cudaEvent_t chunk_done[2] = {nullptr, nullptr};
    cudaEvent_t copy_done[2] = {nullptr, nullptr};
    // live models: destroying the context releases their device state and
    // orphans them (a later detnet_model_destroy only frees the handle)
    std::vector<detnet_model *> models;
    // device group (detnet_ctx_create_group): this context is member 0, the
    // others are owned here; host-buffer batch_evaluate / batch_gradient shard
    // the batch over all members at 8,192-sample chunk boundaries
    std::vector<detnet_ctx *> members;
};

struct detnet_model {
    detnet_ctx *ctx = nullptr;
    int K = 0, N = 0, Z = 0, V = 0, L = 0, frozen = 0;
    const detnet::DimsEntry *dims = nullptr;
    detnet::DBuf simt;          // [L][simt_rec]
    long simt_rec = 0;
    detnet::DBuf lnk_all, lnk_train;
    std::vector<double> masks_nnz; // per layer nnz of W masks (census)
    std::vector<double> params_host, masks_host;
    bool has_masks = false;
    detnet::TcModel tc; // tcgen05 path packing (stack_tc.cu)
    // training state (train.cu): FP64 master params, masks, Adam moments
    detnet::DBuf tparams, tmasks, tm, tv;
    detnet::DBuf bwd_img; // tcgen05 reverse-sweep weight images (bwd_tc.cu)
    int64_t adam_step = 0;
    // [objective, regularizer, diverged step (int64, -1 = none)] of the last
    // detnet_train_apply (device); the host copy of the sticky flag
    detnet::DBuf tstatus;
    long long diverged_step = -1;
    bool train_ready = false;
    bool tc_stale = false;  // tcgen05 images lag the device master params
    bool tc_dev_dirty = false; // dense images to repack on the device before next use
    // sparse path (k_stack_sparse.cuh): CSR-like stream of surviving weights
    detnet::DBuf sparse_stream, sparse_off;
    int sparse_max_words = 0; // largest per-layer stream (shared-memory staging)
    bool sparse_ready = false;
    // model-specialised sparse kernel (sparse_jit.cu): path 3, when the worst
    // layer has at most kJitMaxNnz surviving products
    detnet::JitModel jit;
    long jit_worst_nnz = -1;
    std::vector<double> jit_params, jit_masks; // the weights it is generated from
    long long jit_src_version = -1;
    // CUDA graph of batch_evaluate_device (K1 + fallback + stack + reduce +
    // result copy), replayed while the call, the context settings, the model
    // layout and every device buffer are those it was captured with
    long long version = 0; // bumped when packing / layout / host flags change
    struct EvalGraph {
        long n = -1;
        const void *H = nullptr, *y = nullptr, *x = nullptr, *xhat = nullptr;
        int trainable = 0, path = -1;
        bool exact = false, profiling = false;
        long long version = -1, epoch = -1;
        cudaStream_t st = nullptr;
        cudaGraphExec_t exec = nullptr;
        long long launches = 0;           // kernels per replay
        long long cls_launches[8] = {};   // per class
        std::vector<detnet_ctx::Pending> timers; // captured event pairs
        bool same(const EvalGraph &o) const {
            return n == o.n && H == o.H && y == o.y && x == o.x && xhat == o.xhat &&
                   trainable == o.trainable && path == o.path && exact == o.exact &&
                   profiling == o.profiling && version == o.version && epoch == o.epoch &&
                   st == o.st;
        }
    } graph;
    int graph_seen = 0; // consecutive eager calls with the current key
    // group models: one replica per further group member (same params/masks)
    std::vector<detnet_model *> replicas;
    bool replicas_stale = false; // device training / pruning changed member 0 only
};

namespace detnet {
inline cudaEvent_t take_event(detnet_ctx *c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Bracket a launch with events on the launching stream when profiling.
struct LaunchScope {
    detnet_ctx *c;
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    LaunchScope(detnet_ctx *c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
        c->launches++;
        c->times.launches[cls]++;
        if (c->profiling) {
            a = take_event(c);
            cudaEventRecord(a, st);
        }
    }
    ~LaunchScope() {
        if (c->profiling) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, st);
            c->pending.push_back({cls, a, b});
        }
    }
};

// Kernel timers: block = wait for every pending pair; otherwise only the
// pairs that have completed (asynchronous evaluations keep the rest pending).
inline void drain_times(detnet_ctx *c, bool block = true) {
    size_t keep = 0;
    for (size_t i = 0; i < c->pending.size(); ++i) {
        auto &p = c->pending[i];
        if (!block && cudaEventQuery(p.b) != cudaSuccess) {
            cudaGetLastError(); // cudaErrorNotReady is not an error here
            c->pending[keep++] = p;
            continue;
        }
        float ms = 0.f;
        cudaEventSynchronize(p.b);
        cudaEventElapsedTime(&ms, p.a, p.b);
        c->times.ms[p.cls] += ms;
        c->event_pool.push_back(p.a);
        c->event_pool.push_back(p.b);
    }
    c->pending.resize(keep);
}

// Host-synchronous entry points that read or overwrite device state with
// legacy-stream copies first wait for the context stream (evaluations and
// training steps are only stream-ordered and may still be in flight).
inline int quiesce(detnet_ctx *c) {
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    return e == cudaSuccess ? 0 : fail(DETNET_ERR_CUDA, "stream: %s", cudaGetErrorString(e));
}

inline int check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(DETNET_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return 0;
}

// forward-path helpers (detnet_capi.cu) shared with the training step
struct TraceBufs {
    float *in, *z, *u2, *xf;
    long ts;
};
int ensure_ws(detnet_ctx *c, long n, int K);
int upload_model(detnet_model *m, const detnet_model_desc *d);
void prepare_jit(detnet_model *m, const double *params, const double *masks);
int reset_sing(detnet_ctx *c, cudaStream_t st);
// exact: the reference's FP64 LU for every sample (training: each sample's
// gradient is weighted by 1 / denom, so it gets the reference's denominators)
void train_ws_release(detnet_ctx *c);
int run_pre(detnet_model *m, cudaStream_t st, long s0, long cnt, long n_total, const float *H,
            const float *y, const int8_t *x, bool exact = false, double *g64 = nullptr,
            double *q64 = nullptr);
int run_stack(detnet_model *m, cudaStream_t st, long t0, long nt, long n_local, int l_begin,
              int l_end, bool trainable_only, float *xhat, float *xs, float *vs,
              const TraceBufs *trace = nullptr);
int finish(detnet_model *m, long n, detnet_eval *out);
// the host-buffer evaluation (detnet_batch_evaluate) of one shard; chunks:
// the per-8192-sample-chunk loss sums of the canonical reduction (k_reduce)
int eval_host(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
              int trainable_only, float *xhat_out, detnet_eval *out, std::vector<double> *chunks);
// the FP32 training gradient of one shard: per-chunk raw gradient sums
// [chunks][param_count] and loss chunk sums, copied to the host
int grad_host_shard(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
                    int trainable_only, std::vector<double> &chunk_raw,
                    std::vector<double> &chunk_loss, detnet_eval *out);
// grads = raw * mask / n + regularizer gradient on the model's device
int apply_reg_host(detnet_model *m, const double *raw_host, long n, const detnet_loss_spec *spec,
                   double *grads_out);
int group_batch_evaluate(detnet_model *m, long n, const float *H, const float *y,
                         const int8_t *x, int trainable_only, float *xhat_out, detnet_eval *out);
int group_batch_gradient(detnet_model *m, long n, const float *H, const float *y,
                         const int8_t *x, const detnet_loss_spec *spec, int trainable_only,
                         double *grads_out, detnet_eval *out);
int sync_replicas(detnet_model *m);
int finish_host(detnet_model *m, long n, detnet_eval *out);
int pack_simt_device(detnet_model *m); // FP32 records from the FP64 master copy
int pack_simt_device_from(detnet_model *m, const double *params, const double *masks);
int train_prepare();                   // per-device kernel attributes (train.cu)
struct DwJob; // dw_job.hpp
int dw_tc_prepare();                   // dW contractions on tcgen05 (dw_tc.cu)
int dw_tc_launch(const DwJob *jobs, int j0, int j1, long n, long ts, int splits, cudaStream_t st);
struct BwdArgs;                        // k_train.cuh
int bwd_tc_prepare();                  // reverse sweep on tcgen05 (bwd_tc.cu), K=20 z=160 v=40
long bwd_tc_image_bytes(int L);
int bwd_tc_pack(const double *params, const double *masks, int L, unsigned char *img, cudaStream_t st);
int bwd_tc_launch(const BwdArgs &a, const unsigned char *img, int sms, cudaStream_t st);

// training (train.cu)
int train_batch_gradient(detnet_model *m, long n, const float *H, const float *y,
                         const int8_t *x, const detnet_loss_spec *spec, int trainable_only,
                         double *grads_out, detnet_eval *out);
int train_adam_step(detnet_ctx *c, int n_tx, int z_dim, int v_dim, int depth, int frozen_prefix,
                    double *params, const double *masks, const double *grads, double *m1,
                    double *m2, int64_t *step, const detnet_adam_config *cfg);

} // namespace detnet
