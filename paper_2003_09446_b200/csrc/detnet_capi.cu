// detnet_capi.cu -- implementation of include/detnet_b200.h.
//
// Host runtime for the DetNet layer-stack engine: device context, parameter
// packing (once per params version), workspace management, chunked
// host<->device streaming overlapped with compute, kernel launches with
// per-launch CUDA-event timing, and status/error mapping. No CPU fallback:
// every compute entry point requires an sm_100 device.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "../../include/detnet_b200.h"
#include "common.cuh"
#include "k_generate.cuh"
#include "k_preprocess.cuh"
#include "k_baseline.cuh"
#include "k_prep_fast.cuh"
#include "k_stack_sparse.cuh"
#include "k_stack_simt.cuh"
#include <cudaTypedefs.h>

#include "engine.hpp"

using namespace detnet;

namespace detnet {

// ---- dims dispatch --------------------------------------------------------
using PreFn = void (*)(dim3, dim3, size_t, cudaStream_t, long, int, const float *, const float *,
                       const int8_t *, float *, float *, double *, uint32_t *, uint8_t *,
                       unsigned long long *, const long *, const int *, double *, double *);
using SimtFn = void (*)(dim3, dim3, size_t, cudaStream_t, const StackArgs &);
constexpr int SIMT_LARGE = 256; // samples per CTA of k_stack_simt (large batches)
template <int K, int Z, int V> constexpr size_t simt_pair_smem() {
    return (2 * static_cast<size_t>(simt_rec(K, Z, V)) + (K + V) * SIMTP_SAMPLES) * 4 + 64;
}

template <int K>
void launch_pre(dim3 g, dim3 b, size_t sm, cudaStream_t st, long n, int N, const float *H,
                const float *y, const int8_t *x, float *gp, float *q32, double *dn, uint32_t *xm,
                uint8_t *fl, unsigned long long *sing, const long *list, const int *cnt,
                double *g64, double *q64) {
    k_preprocess<K><<<g, b, sm, st>>>(n, N, H, y, x, gp, q32, dn, xm, fl, sing, list, cnt, g64, q64);
}

using FastFn = void (*)(dim3, dim3, size_t, cudaStream_t, long, int, const float *, const float *,
                        const int8_t *, float *, float *, double *, uint32_t *, uint8_t *, int *,
                        long *, const CUtensorMap *);

// 2-D view of H for the K1 fast path: rows of N*K floats (one sample), box
// {SSTR/4 floats, PS_TILE samples}. The box is 4 floats wider than a 6-row
// chunk so each sample lands on the bank-spreading 496-byte stride; the extra
// floats are the next row (or zero fill past the end of the sample).
int encode_h_map(CUtensorMap *map, const float *H, long n, int N, int K) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return fail(DETNET_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N) * K, static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(N) * K * 4};
    const cuuint32_t box[2] = {PrepStreamSmem<20, PREP_FAST_N>::BOXW, PS_TILE};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(H), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(DETNET_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", r);
    return 0;
}

template <int K>
void launch_fast(dim3 g, dim3 b, size_t sm, cudaStream_t st, long n, int N, const float *H,
                 const float *y, const int8_t *x, float *gp, float *q32, double *dn, uint32_t *xm,
                 uint8_t *fl, int *fbc, long *fbl, const CUtensorMap *map) {
    (void)b;
    (void)sm;
    (void)N; // the fast path is instantiated for N == PREP_FAST_N only
    (void)H;
    k_prep_stream<K, PREP_FAST_N><<<g, PS_THREADS, PrepStreamSmem<K, PREP_FAST_N>::BYTES, st>>>(
        *map, n, y, x, gp, q32, dn, xm, fl, fbc, fbl);
}

template <int K> int set_fast_smem() {
    return cudaFuncSetAttribute(k_prep_stream<K, PREP_FAST_N>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(PrepStreamSmem<K, PREP_FAST_N>::BYTES)) ==
                   cudaSuccess
               ? 0
               : -1;
}

template <int K, int Z, int V>
void launch_simt(dim3 g, dim3 b, size_t sm, cudaStream_t st, const StackArgs &a) {
    if (b.x == SIMTP_THREADS) k_stack_simt_pair<K, Z, V><<<g, b, simt_pair_smem<K, Z, V>(), st>>>(a);
    else k_stack_simt<K, Z, V, SIMT_LARGE><<<g, b, sm, st>>>(a);
}

template <int K, int Z, int V> int set_simt_smem() {
    const int bytes = static_cast<int>(2 * simt_rec(K, Z, V) * 4 + 64);
    const bool ok = cudaFuncSetAttribute(k_stack_simt_pair<K, Z, V>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(simt_pair_smem<K, Z, V>())) ==
                        cudaSuccess &&
                    cudaFuncSetAttribute(k_stack_simt<K, Z, V, SIMT_LARGE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) ==
                        cudaSuccess;
    return ok ? 0 : -1;
}

struct DimsEntry {
    int K, Z, V;
    PreFn pre;
    SimtFn simt;
    int (*prep)();
    FastFn fast;           // nullptr: exact preprocessing only
    int (*prep_fast)();
};

#define DETNET_DIMS(K, Z, V) {K, Z, V, launch_pre<K>, launch_simt<K, Z, V>, set_simt_smem<K, Z, V>, nullptr, nullptr}
const DimsEntry kDims[] = {
    {20, 160, 40, launch_pre<20>, launch_simt<20, 160, 40>, set_simt_smem<20, 160, 40>,
     launch_fast<20>, set_fast_smem<20>},
    DETNET_DIMS(2, 16, 4),  DETNET_DIMS(3, 24, 6),
    DETNET_DIMS(4, 32, 8),    DETNET_DIMS(6, 48, 12), DETNET_DIMS(8, 64, 16),
};
#undef DETNET_DIMS

static const DimsEntry *find_dims(int K, int Z, int V) {
    for (const DimsEntry &d : kDims)
        if (d.K == K && d.Z == Z && d.V == V) return &d;
    return nullptr;
}

} // namespace detnet

namespace detnet {

int pack_simt(detnet_model *m, const double *params, const double *masks, std::vector<float> &out) {
    const int K = m->K, Z = m->Z, V = m->V, IN = 3 * K + V;
    const int IN4 = simt_in4(K, V), O4 = simt_o4(K, V);
    const long P = record_size(K, Z, V);
    const long R = simt_rec(K, Z, V);
    out.assign(static_cast<size_t>(R) * m->L, 0.f);
    for (int l = 0; l < m->L; ++l) {
        const double *p = params + l * P;
        const double *mk = masks ? masks + l * P : nullptr;
        auto w = [&](long off) { return p[off] * (mk ? mk[off] : 1.0); };
        float *r = out.data() + static_cast<size_t>(l) * R;
        const long oW1 = 0, ob1 = oW1 + static_cast<long>(Z) * IN, oW2 = ob1 + Z,
                   ob2 = oW2 + static_cast<long>(K) * Z, oW3 = ob2 + K,
                   ob3 = oW3 + static_cast<long>(V) * Z, ot = ob3 + V;
        for (int i = 0; i < Z; ++i) {
            for (int j = 0; j < IN; ++j) r[i * IN4 + j] = static_cast<float>(w(oW1 + i * IN + j));
            r[i * IN4 + IN] = static_cast<float>(w(ob1 + i));
        }
        float *w23 = r + static_cast<long>(Z) * IN4;
        for (int i = 0; i < Z; ++i) {
            for (int k = 0; k < K; ++k) w23[i * O4 + k] = static_cast<float>(w(oW2 + k * Z + i));
            for (int k = 0; k < V; ++k) w23[i * O4 + K + k] = static_cast<float>(w(oW3 + k * Z + i));
        }
        float *b23 = w23 + static_cast<long>(Z) * O4;
        for (int k = 0; k < K; ++k) b23[k] = static_cast<float>(w(ob2 + k));
        for (int k = 0; k < V; ++k) b23[K + k] = static_cast<float>(w(ob3 + k));
        b23[O4] = static_cast<float>(p[ot]);
        if (!(p[ot] > 0.0)) return fail(DETNET_ERR_CONTRACT, "soft_sign: t must be > 0 (layer %d)", l);
    }
    return 0;
}

// Sparse layer streams for k_stack_sparse (format in k_stack_sparse.cuh).
size_t sparse_smem(int max_words) {
    return sizeof(float) * TILE * (3 * 20 + 40 + 2 * 60 + 20) + 2 * sizeof(int) * max_words + 16;
}

int pack_sparse(detnet_model *m, const double *params, const double *masks) {
    m->sparse_ready = false;
    const int K = m->K, Z = m->Z, V = m->V, IN = 3 * K + V;
    const long P = record_size(K, Z, V);
    std::vector<int> st;
    std::vector<long> offs(m->L + 1);
    auto fbits = [](float f) { int i; std::memcpy(&i, &f, 4); return i; };
    for (int l = 0; l < m->L; ++l) {
        const double *p = params + l * P;
        const double *mk = masks ? masks + l * P : nullptr;
        auto w = [&](long off) { return static_cast<float>(p[off] * (mk ? mk[off] : 1.0)); };
        const long oW1 = 0, ob1 = static_cast<long>(Z) * IN, oW2 = ob1 + Z,
                   ob2 = oW2 + static_cast<long>(K) * Z, oW3 = ob2 + K,
                   ob3 = oW3 + static_cast<long>(V) * Z, ot = ob3 + V;
        std::vector<int> units;
        std::vector<std::vector<std::pair<int, float>>> ins, outs;
        for (int i = 0; i < Z; ++i) {
            std::vector<std::pair<int, float>> o;
            for (int r = 0; r < V; ++r) if (w(oW3 + r * Z + i) != 0.f) o.push_back({r, w(oW3 + r * Z + i)});
            for (int k = 0; k < K; ++k) if (w(oW2 + k * Z + i) != 0.f) o.push_back({V + k, w(oW2 + k * Z + i)});
            std::vector<std::pair<int, float>> in;
            for (int j = 0; j < IN; ++j) if (w(oW1 + i * IN + j) != 0.f) in.push_back({j, w(oW1 + i * IN + j)});
            if (o.empty()) continue;
            units.push_back(i);
            ins.push_back(in);
            outs.push_back(o);
        }
        const int nu = static_cast<int>(units.size());
        long work = 0, half = 0;
        for (int u = 0; u < nu; ++u) work += 1 + ins[u].size() + outs[u].size();
        int split = nu;
        for (int u = 0; u < nu; ++u) {
            half += 1 + ins[u].size() + outs[u].size();
            if (2 * half >= work) { split = u + 1; break; }
        }
        while (st.size() % 4) st.push_back(0);
        const long base = static_cast<long>(st.size());
        offs[l] = base;
        st.resize(base + 4 + 4 * nu + nu, 0);
        if (st.size() & 1) st.push_back(0);
        int e = 0;
        std::vector<int> ent;
        for (int u = 0; u < nu; ++u) {
            st[base + 4 + 4 * u + 0] = e;
            for (auto &pr : ins[u]) { ent.push_back(pr.first); ent.push_back(fbits(pr.second)); ++e; }
            st[base + 4 + 4 * u + 1] = e;
            st[base + 4 + 4 * u + 2] = e;
            for (auto &pr : outs[u]) { ent.push_back(pr.first); ent.push_back(fbits(pr.second)); ++e; }
            st[base + 4 + 4 * u + 3] = e;
            st[base + 4 + 4 * nu + u] = fbits(w(ob1 + units[u]));
        }
        st.insert(st.end(), ent.begin(), ent.end());
        const long tail = static_cast<long>(st.size()) - base;
        std::vector<int> b23(68, 0);
        for (int r = 0; r < V; ++r) b23[r] = fbits(w(ob3 + r));
        for (int k = 0; k < K; ++k) b23[V + k] = fbits(w(ob2 + k));
        b23[64] = fbits(static_cast<float>(p[ot]));
        b23[65] = fbits(static_cast<float>(1.0 / p[ot]));
        st.insert(st.end(), b23.begin(), b23.end());
        st[base + 0] = nu;
        st[base + 1] = split;
        st[base + 2] = static_cast<int>(tail);
    }
    while (st.size() % 4) st.push_back(0);
    offs[m->L] = static_cast<long>(st.size());
    long max_words = 0;
    for (int l = 0; l < m->L; ++l) max_words = std::max(max_words, offs[l + 1] - offs[l]);
    m->sparse_max_words = static_cast<int>((max_words + 3) / 4 * 4);
    if (m->sparse_stream.ensure(st.size() * 4) || m->sparse_off.ensure(offs.size() * 8))
        return fail(DETNET_ERR_CUDA, "sparse stream allocation");
    CK(cudaMemcpy(m->sparse_stream.p, st.data(), st.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(m->sparse_off.p, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice));
    // the kernel stages two layer streams next to its 120 KB of activations
    m->sparse_ready = (K == 20 && V == 40) &&
                      sparse_smem(m->sparse_max_words) <= 232448;
    return 0;
}

// The model-specialised kernel (sparse_jit.cu) is generated and compiled at
// its first use from these weights when every layer is sparse enough; the
// count stops at the first layer over the limit (dense models: a few units).
void prepare_jit(detnet_model *m, const double *params, const double *masks) {
    const long P = record_size(m->K, m->Z, m->V);
    m->jit_worst_nnz =
        m->K <= 32 ? jit_layer_nnz(m->K, m->Z, m->V, m->L, params, masks, kJitMaxNnz) : -1;
    m->jit_params.clear();
    m->jit_masks.clear();
    if (m->jit_worst_nnz >= 0 && m->jit_worst_nnz <= kJitMaxNnz) {
        m->jit_params.assign(params, params + P * m->L);
        if (masks) m->jit_masks.assign(masks, masks + P * m->L);
    }
    m->jit_src_version = m->version;
}

// Every hidden unit of every layer has a surviving outgoing weight (the
// dense tcgen05 images then list the units in natural order).
bool all_units_live(int K, int Z, int V, int L, const double *params, const double *masks) {
    const int IN = 3 * K + V;
    const long P = record_size(K, Z, V);
    const long oW2 = static_cast<long>(Z) * IN + Z, oW3 = oW2 + static_cast<long>(K) * Z + K;
    for (int l = 0; l < L; ++l) {
        const double *pr = params + l * P, *mk = masks ? masks + l * P : nullptr;
        auto nz = [&](long off) { return static_cast<float>(pr[off] * (mk ? mk[off] : 1.0)) != 0.f; };
        for (int i = 0; i < Z; ++i) {
            bool alive = false;
            for (int o = 0; o < K && !alive; ++o) alive = nz(oW2 + static_cast<long>(o) * Z + i);
            for (int o = 0; o < V && !alive; ++o) alive = nz(oW3 + static_cast<long>(o) * Z + i);
            if (!alive) return false;
        }
    }
    return true;
}

// Every weight of W1, b1, W2, W3 fits the split-FP16 images (x16 scale within
// the FP16 range, the host packer's test); otherwise the host packers run and
// the model takes the 3xTF32 images only.
bool h16_weights_in_range(int K, int Z, int V, int L, const double *params, const double *masks) {
    const int IN = 3 * K + V;
    const long P = record_size(K, Z, V);
    const long nW1b1 = static_cast<long>(Z) * IN + Z, oW2 = nW1b1, nW2 = static_cast<long>(K) * Z,
               oW3 = oW2 + nW2 + K, nW3 = static_cast<long>(V) * Z;
    for (int l = 0; l < L; ++l) {
        const double *pr = params + l * P, *mk = masks ? masks + l * P : nullptr;
        auto ok = [&](long off) {
            const float sv = static_cast<float>(pr[off] * (mk ? mk[off] : 1.0)) * 16.f;
            return std::fabs(sv) <= 65000.f;
        };
        for (long e = 0; e < nW1b1; ++e) if (!ok(e)) return false;
        for (long e = 0; e < nW2; ++e) if (!ok(oW2 + e)) return false;
        for (long e = 0; e < nW3; ++e) if (!ok(oW3 + e)) return false;
    }
    return true;
}

int upload_model(detnet_model *m, const detnet_model_desc *d) {
    ++m->version;
    if (int rc = quiesce(m->ctx)) return rc; // in-flight work may read the old buffers
    const long P = record_size(m->K, m->Z, m->V);
    m->params_host.assign(d->params, d->params + P * m->L);
    m->has_masks = d->masks != nullptr;
    if (d->masks) m->masks_host.assign(d->masks, d->masks + P * m->L);
    else m->masks_host.clear();
    m->simt_rec = simt_rec(m->K, m->Z, m->V);
    // Dense models (the BASELINE dims, every unit live): the FP64 records go
    // to the device once and the SIMT records and both tensor-core image sets
    // are packed there (~1 ms instead of ~20 ms of host loops per update)
    const bool dense_dev = m->K == 20 && m->Z == 160 && m->V == 40 &&
                           !std::getenv("DETNET_HOST_PACK") &&
                           all_units_live(m->K, m->Z, m->V, m->L, d->params, d->masks) &&
                           h16_weights_in_range(m->K, m->Z, m->V, m->L, d->params, d->masks);
    if (dense_dev) {
        const size_t bytes = sizeof(double) * P * m->L;
        if (m->tparams.ensure(bytes) || (d->masks && m->tmasks.ensure(bytes)) ||
            m->simt.ensure(sizeof(float) * m->simt_rec * m->L))
            return fail(DETNET_ERR_CUDA, "cudaMalloc weights");
        // on the context stream: a pageable cudaMemcpy may return before its
        // DMA lands, and the packers below run on this (non-blocking) stream
        CK(cudaMemcpyAsync(m->tparams.p, d->params, bytes, cudaMemcpyHostToDevice, m->ctx->stream));
        if (d->masks)
            CK(cudaMemcpyAsync(m->tmasks.p, d->masks, bytes, cudaMemcpyHostToDevice, m->ctx->stream));
        const double *mdev = d->masks ? m->tmasks.as<double>() : nullptr;
        if (int rc = pack_simt_device_from(m, m->tparams.as<double>(), mdev)) return rc;
    } else {
        std::vector<float> packed;
        if (int rc = pack_simt(m, d->params, d->masks, packed)) return rc;
        if (m->simt.ensure(packed.size() * 4)) return fail(DETNET_ERR_CUDA, "cudaMalloc weights");
        CK(cudaMemcpy(m->simt.p, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice));
    }
    std::vector<double> la(m->L), lt(m->L);
    for (int l = 0; l < m->L; ++l) {
        la[l] = std::log(static_cast<double>(l + 1));
        lt[l] = (l + 1 >= m->frozen + 1) ? la[l] : 0.0;
    }
    if (m->lnk_all.ensure(m->L * 8) || m->lnk_train.ensure(m->L * 8))
        return fail(DETNET_ERR_CUDA, "cudaMalloc lnk");
    CK(cudaMemcpy(m->lnk_all.p, la.data(), m->L * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(m->lnk_train.p, lt.data(), m->L * 8, cudaMemcpyHostToDevice));
    if (dense_dev) {
        if (int rc = tc_pack_dense_device(m->tc, m->K, m->Z, m->V, m->L, m->tparams.as<double>(),
                                          d->masks ? m->tmasks.as<double>() : nullptr,
                                          m->ctx->stream))
            return rc;
        if (int rc = check_launch()) return rc;
        CK(cudaStreamSynchronize(m->ctx->stream)); // a host-synchronous API, as the host packers
    } else if (int rc = tc_pack(m->tc, m->K, m->Z, m->V, m->L, d->params, d->masks)) {
        return rc;
    }
    // the table-driven CSR stream only when asked for (DETNET_SPARSE_CSR): it
    // costs a pass over every weight on each update
    m->sparse_ready = false;
    if (std::getenv("DETNET_SPARSE_CSR"))
        if (int rc = pack_sparse(m, d->params, d->masks)) return rc;
    prepare_jit(m, d->params, d->masks);
    // every pageable cudaMemcpy above (host-packed images, records) has landed
    // before any kernel on a non-blocking stream reads the buffers
    CK(cudaStreamSynchronize(cudaStreamLegacy));
    m->train_ready = false; // the device master copy restarts from these params
    m->tc_stale = false;
    m->tc_dev_dirty = false; // the images just packed from the host copy are current
    return 0;
}

// After device-side training steps the tcgen05 images are rebuilt once from
// the FP64 master copy before the next tensor-core evaluation.
int refresh_tc(detnet_model *m) {
    if (!m->tc_stale) return 0;
    const long total = record_size(m->K, m->Z, m->V) * m->L;
    std::vector<double> p(total);
    CK(cudaStreamSynchronize(m->ctx->stream));
    CK(cudaMemcpy(p.data(), m->tparams.p, sizeof(double) * total, cudaMemcpyDeviceToHost));
    m->params_host = p;
    if (int rc = tc_pack(m->tc, m->K, m->Z, m->V, m->L, p.data(),
                         m->has_masks ? m->masks_host.data() : nullptr))
        return rc;
    m->tc_stale = false;
    return 0;
}

// Workspace for n samples (all global per-sample/per-tile arrays).
int ensure_ws(detnet_ctx *c, long n, int K) {
    const long tiles = (n + TILE - 1) / TILE;
    const long np = tiles * TILE;
    const int NG = gram_entries(K);
    if (c->gp.ensure(sizeof(float) * NG * np) || c->q32.ensure(sizeof(float) * K * np) ||
        c->denom.ensure(sizeof(double) * np) || c->xmask.ensure(sizeof(uint32_t) * np) ||
        c->flag.ensure(np) || c->tile_loss.ensure(sizeof(double) * 4 * tiles) ||
        c->chunks.ensure(sizeof(double) * ((tiles + RED_CHUNK_TILES - 1) / RED_CHUNK_TILES)) ||
        c->tile_err.ensure(sizeof(long long) * 4 * tiles) || c->sing.ensure(8) ||
        c->result.ensure(64))
        return fail(DETNET_ERR_CUDA, "workspace allocation failed (n=%ld)", n);
    if (!c->h_result) CK(cudaMallocHost(&c->h_result, 64));
    return 0;
}

// The model-specialised sparse kernel: path 3, for models whose every layer
// has at most kJitMaxNnz surviving products (config 4: ~330 per layer, where
// the compacted tcgen05 kernel is bound by its serial per-layer chain). Not
// on the auto path: its ~13 s compile per weight version pays off only over
// billions of detections with fixed weights (a BER sweep), not for a trainer
// that evaluates after every update. Valid while the weights are those it
// was generated from.
bool use_jit(const detnet_model *m) {
    const int path = m->ctx->path;
    if (path != 3 || std::getenv("DETNET_NO_JIT")) return false;
    // weights changed on the device since pack time (training, pruning in
    // progress) bump the version: the kernel no longer matches them
    if (m->jit_src_version != m->version) return false; // (a device prune re-records the source)
    if (m->jit_params.empty()) return false;
    return true;
}

bool use_tc(const detnet_model *m) {
    const int path = m->ctx->path;
    if (path == 1 || path == 3) return false;
    if (!m->tc.ready) return false;
    return true;
}

// split-FP16 stack (stack_h16.cu) for this model and context (training
// forward: only with the dense images)
bool use_h16(const detnet_model *m, bool trace) {
    const int path = m->ctx->path;
    if (!use_tc(m) || !(path == 0 || path == 4) || !m->tc.h16_ready) return false;
    return !trace || m->tc.zh16 == 160;
}

// K1 (+pad) over samples [s0, s0+cnt) of the global arrays.
int run_pre(detnet_model *m, cudaStream_t st, long s0, long cnt, long n_total, const float *H,
            const float *y, const int8_t *x, bool exact, double *g64, double *q64) {
    detnet_ctx *c = m->ctx;
    const int K = m->K, NG = gram_entries(K);
    const long t0 = s0 / TILE;
    const int N = m->N;
    const size_t smem = static_cast<size_t>(4) * (N * K + N + K * K + K) * sizeof(double);
    const bool aligned = (reinterpret_cast<uintptr_t>(H) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(y) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(x) % 4 == 0);
    if (m->dims->fast && !c->exact_pre && !exact && !g64 && aligned && N == PREP_FAST_N) {
        // fast path + exact LU for the samples it flags (device-side list)
        if (c->fb_list.ensure(sizeof(long) * cnt) || c->fb_count.ensure(sizeof(int)))
            return fail(DETNET_ERR_CUDA, "fallback list allocation failed");
        CK(cudaMemsetAsync(c->fb_count.p, 0, sizeof(int), st));
        {
            LaunchScope ls(c, DETNET_K_PREPROCESS, st);
            const long tiles = (cnt + PS_TILE - 1) / PS_TILE;
            const long grid = std::min<long>(tiles, 2L * c->sms);
            CUtensorMap hmap;
            if (int rc = encode_h_map(&hmap, H, cnt, N, K)) return rc;
            m->dims->fast(dim3(static_cast<unsigned>(grid)),
                          dim3(PS_THREADS), 0, st,
                          cnt, N, H, y, x, c->gp.as<float>() + t0 * NG * TILE,
                          c->q32.as<float>() + t0 * K * TILE, c->denom.as<double>() + s0,
                          c->xmask.as<uint32_t>() + s0, c->flag.as<uint8_t>() + s0,
                          c->fb_count.as<int>(), c->fb_list.as<long>(), &hmap);
        }
        if (int rc = check_launch()) return rc;
        LaunchScope ls(c, DETNET_K_OTHER, st); // exact LU for the flagged samples
        m->dims->pre(dim3(148), dim3(128), smem, st, cnt, m->N, H, y, x,
                     c->gp.as<float>() + t0 * NG * TILE, c->q32.as<float>() + t0 * K * TILE,
                     c->denom.as<double>() + s0, c->xmask.as<uint32_t>() + s0,
                     c->flag.as<uint8_t>() + s0, c->sing.as<unsigned long long>(),
                     c->fb_list.as<long>(), c->fb_count.as<int>(), nullptr, nullptr);
    } else {
        const int blocks = static_cast<int>(std::min<long>((cnt + 3) / 4, 148L * 32));
        LaunchScope ls(c, DETNET_K_PREPROCESS, st);
        m->dims->pre(dim3(blocks), dim3(128), smem, st, cnt, m->N, H, y, x,
                     c->gp.as<float>() + t0 * NG * TILE, c->q32.as<float>() + t0 * K * TILE,
                     c->denom.as<double>() + s0, c->xmask.as<uint32_t>() + s0,
                     c->flag.as<uint8_t>() + s0, c->sing.as<unsigned long long>(), nullptr,
                     nullptr, g64 ? g64 + s0 * K * K : nullptr, q64 ? q64 + s0 * K : nullptr);
    }
    if (int rc = check_launch()) return rc;
    const long end = s0 + cnt;
    if (end == n_total) {
        const long np = (n_total + TILE - 1) / TILE * TILE;
        if (np > n_total) {
            LaunchScope ls(c, DETNET_K_OTHER, st);
            k_pad_tail<<<1, TILE, 0, st>>>(n_total, np, K, c->gp.as<float>(), c->q32.as<float>(),
                                           c->denom.as<double>(), c->xmask.as<uint32_t>(),
                                           c->flag.as<uint8_t>());
            if (int rc = check_launch()) return rc;
        }
    }
    return 0;
}

// K2 over tiles [t0, t0+nt) (samples relative to s_base = t0*TILE).
int run_stack(detnet_model *m, cudaStream_t st, long t0, long nt, long n_local, int l_begin,
              int l_end, bool trainable_only, float *xhat, float *xs, float *vs,
              const TraceBufs *trace) {
    detnet_ctx *c = m->ctx;
    if (!trace && !xs && l_begin == 0 && use_jit(m)) {
        JitModel &jm = m->jit;
        if (!jm.ready || jm.version != m->jit_src_version) {
            const int rc = jit_build(jm, m->K, m->Z, m->V, m->L, m->jit_params.data(),
                                     m->jit_masks.empty() ? nullptr : m->jit_masks.data());
            if (rc) return rc; // NVRTC missing or the compile failed: loud, no fallback
            jm.version = m->jit_src_version;
        }
        if (jm.ready && jm.version == m->jit_src_version) {
            TcArgs ja{};
            ja.gp = c->gp.as<float>();
            ja.q32 = c->q32.as<float>();
            ja.denom = c->denom.as<double>();
            ja.xmask = c->xmask.as<uint32_t>();
            ja.lnk = (trainable_only ? m->lnk_train : m->lnk_all).as<double>();
            ja.l_begin = 0;
            ja.l_end = l_end;
            ja.n = n_local;
            ja.n_tiles = nt;
            ja.tile0 = t0;
            ja.xhat = xhat;
            ja.tile_loss = c->tile_loss.as<double>();
            ja.tile_err = c->tile_err.as<long long>();
            LaunchScope ls(c, DETNET_K_STACK, st);
            if (int rc = jit_launch(jm, ja, st, c->sms, c->device)) return rc;
            return check_launch();
        }
    }
    const bool sparse = !trace && !xs && m->sparse_ready && !m->tc_stale && c->path == 3 &&
                        std::getenv("DETNET_SPARSE_CSR") != nullptr;
    if (sparse) {
        SparseArgs sa{};
        sa.gp = c->gp.as<float>();
        sa.q32 = c->q32.as<float>();
        sa.denom = c->denom.as<double>();
        sa.xmask = c->xmask.as<uint32_t>();
        sa.stream = m->sparse_stream.as<int>();
        sa.lay_off = m->sparse_off.as<long>();
        sa.max_words = m->sparse_max_words;
        sa.lnk = (trainable_only ? m->lnk_train : m->lnk_all).as<double>();
        sa.L = m->L;
        sa.n = n_local;
        sa.n_tiles = nt;
        sa.tile0 = t0;
        sa.xhat = xhat;
        sa.tile_loss = c->tile_loss.as<double>();
        sa.tile_err = c->tile_err.as<long long>();
        const size_t smem = sparse_smem(m->sparse_max_words);
        CK(cudaFuncSetAttribute(k_stack_sparse<20, 40>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        const int grid = static_cast<int>(std::min<long>(nt, c->sms));
        {
            LaunchScope ls(c, DETNET_K_STACK, st);
            k_stack_sparse<20, 40><<<grid, 256, smem, st>>>(sa);
        }
        return check_launch();
    }
    // A masked model whose images were compacted at upload (configs 3/4) and that is
    // now being trained on the device: switch it to the dense ZH = 160 images of
    // W (.) M, which the device repacks after every Adam step (k_pack_tc160 /
    // k_pack_h16_160 read the masks). The compacted images would need a host repack
    // per weight version and have no training-trace variant, which put the training
    // forward of such models on the CUDA-core kernel (0.76 vs 0.22 ms at batch 5000).
    // A later detnet_model_update / detnet_model_prune compacts again.
    if (trace && c->train_tc && c->path != 1 && c->path != 3 && m->tc.ready &&
        (m->tc.zh != 160 || m->tc_stale) && m->K == 20 && m->Z == 160 && m->V == 40 &&
        m->train_ready) { // tc_stale: pruned on the device since the images were packed
        LaunchScope ls(c, DETNET_K_OTHER, st);
        if (int rc = tc_pack_dense_device(m->tc, m->K, m->Z, m->V, m->L, m->tparams.as<double>(),
                                          m->tmasks.as<double>(), st))
            return rc;
        m->tc_stale = false;
        m->tc_dev_dirty = false;
        ++m->version; // captured evaluation graphs hold the old image pointers
    }
    // the training forward (trace) on the SIMT path neither needs nor
    // refreshes the tensor-core images (they are repacked on first use)
    const bool simt_trace = trace && !(c->train_tc && m->tc.zh == 160);
    if (m->ctx->path != 1 && !simt_trace) {
        if (m->tc_dev_dirty) { // after training steps: dense images from the device masters
            LaunchScope ls(c, DETNET_K_OTHER, st);
            const int rc = tc_pack_device(m->tc, m->tparams.as<double>(), m->tmasks.as<double>(),
                                          record_size(m->K, m->Z, m->V), st);
            if (rc > 1) return rc;
            m->tc_stale = rc != 0;
            m->tc_dev_dirty = false;
        }
        if (int rc = refresh_tc(m)) return rc;
    }
    // the training forward (trace) runs on tcgen05 only when asked for
    // (detnet_ctx_set_train_forward): 3xTF32 activations are ~4x noisier than
    // FP32 ones, which shortens the FP32-vs-FP64 tracking of long training runs
    if (use_tc(m) && (!trace || (c->train_tc && m->tc.zh == 160))) {
        TcArgs ta{};
        ta.gp = c->gp.as<float>();
        ta.q32 = c->q32.as<float>();
        ta.denom = c->denom.as<double>();
        ta.xmask = c->xmask.as<uint32_t>();
        ta.lnk = (trainable_only ? m->lnk_train : m->lnk_all).as<double>();
        ta.l_begin = l_begin;
        ta.l_end = l_end;
        ta.n = n_local;
        ta.n_tiles = nt;
        ta.tile0 = t0;
        ta.xhat = xhat;
        ta.tile_loss = c->tile_loss.as<double>();
        ta.tile_err = c->tile_err.as<long long>();
        if (use_h16(m, trace != nullptr)) {
            // split-FP16 stack, then the 3xTF32 recompute of the tiles whose
            // activations left the FP16 range (exits at once when none did)
            if (c->redo.ensure(static_cast<size_t>(t0 + nt)) || c->redo_count.ensure(sizeof(int)))
                return fail(DETNET_ERR_CUDA, "range-flag allocation failed");
            CK(cudaMemsetAsync(c->redo_count.p, 0, sizeof(int), st));
            {
                LaunchScope ls(c, DETNET_K_STACK, st);
                if (int rc = h16_launch_state(m->tc, ta, xs, vs, st, trace, c->redo.as<uint8_t>(),
                                              c->redo_count.as<int>(), c->sms))
                    return rc;
            }
            if (int rc = check_launch()) return rc;
            LaunchScope ls(c, DETNET_K_OTHER, st);
            if (int rc = tc_launch_redo(m->tc, ta, xs, vs, st, trace, c->redo.as<uint8_t>(),
                                        c->redo_count.as<int>()))
                return rc;
            return check_launch();
        }
        LaunchScope ls(c, DETNET_K_STACK, st);
        if (int rc = tc_launch_state(m->tc, ta, xs, vs, st, trace)) return rc;
        return check_launch();
    }
    StackArgs a{};
    a.gp = c->gp.as<float>();
    a.q32 = c->q32.as<float>();
    a.denom = c->denom.as<double>();
    a.xmask = c->xmask.as<uint32_t>();
    a.wrec = m->simt.as<float>();
    a.rec_floats = m->simt_rec;
    a.lnk = (trainable_only ? m->lnk_train : m->lnk_all).as<double>();
    a.l_begin = l_begin;
    a.l_end = l_end;
    a.n = n_local;
    a.n_tiles = nt;
    a.tile0 = t0;
    a.xhat = xhat;
    a.x_state = xs;
    a.v_state = vs;
    a.tile_loss = c->tile_loss.as<double>();
    a.tile_err = c->tile_err.as<long long>();
    if (trace) {
        a.tr_in = trace->in;
        a.tr_z = trace->z;
        a.tr_u2 = trace->u2;
        a.tr_xf = trace->xf;
        a.ts = trace->ts;
    }
    const size_t smem = 2 * static_cast<size_t>(m->simt_rec) * 4 + 64;
    // one CTA per SM: small batches use 64-sample CTAs, two threads per sample
    const long vt = c->variant_n > 0 ? (c->variant_n + TILE - 1) / TILE : nt;
    const bool large = vt * TILE / SIMT_LARGE >= c->sms;
    const int samples = large ? SIMT_LARGE : SIMTP_SAMPLES;
    const int blocks = static_cast<int>((nt * TILE + samples - 1) / samples);
    {
        LaunchScope ls(c, DETNET_K_STACK, st);
        m->dims->simt(dim3(blocks), dim3(large ? SIMT_LARGE : SIMTP_THREADS), smem, st, a);
    }
    return check_launch();
}

// finish_eval (kernels.cpp:93-103), device part: fixed-order reduction and
// the copy of {loss, errors, flagged, singular} to pinned host memory
int finish_device(detnet_model *m, long n, double *dst) {
    detnet_ctx *c = m->ctx;
    const long tiles = (n + TILE - 1) / TILE;
    double *res = c->result.as<double>();
    {
        LaunchScope ls(c, DETNET_K_REDUCE, c->stream);
        k_reduce<<<1, 1024, 0, c->stream>>>(c->tile_loss.as<double>(), c->tile_err.as<long long>(),
                                           4 * tiles, c->flag.as<uint8_t>(), n, res,
                                           reinterpret_cast<long long *>(res + 1),
                                           reinterpret_cast<long long *>(res + 2),
                                           c->chunks.as<double>());
    }
    c->last_chunks = (tiles + RED_CHUNK_TILES - 1) / RED_CHUNK_TILES;
    if (int rc = check_launch()) return rc;
    CK(cudaMemcpyAsync(res + 3, c->sing.p, 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(dst ? dst : c->h_result, res, 32, cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

// decode a finished {loss, errors, flagged, singular} block
int decode_eval(const double *h, long n, int K, detnet_eval *out) {
    unsigned long long sing;
    std::memcpy(&sing, h + 3, 8);
    if (sing != ~0ull)
        return fail(DETNET_ERR_SINGULAR,
                    "solve_normal_equations: matrix is singular to working precision (sample %llu)",
                    sing);
    long long e, f;
    std::memcpy(&e, h + 1, 8);
    std::memcpy(&f, h + 2, 8);
    out->loss_sum = h[0];
    out->data_loss = n ? h[0] / static_cast<double>(n) : 0.0;
    out->symbol_errors = e;
    out->symbols = n * static_cast<long long>(K);
    out->flagged = f;
    return 0;
}

// host part: wait, then decode (SingularMatrixError as linalg.cpp:59-60)
int finish_host(detnet_model *m, long n, detnet_eval *out) {
    detnet_ctx *c = m->ctx;
    CK(cudaStreamSynchronize(c->stream));
    drain_times(c);
    return decode_eval(c->h_result, n, m->K, out);
}

int finish(detnet_model *m, long n, detnet_eval *out) {
    if (int rc = finish_device(m, n, nullptr)) return rc;
    return finish_host(m, n, out);
}

int reset_sing(detnet_ctx *c, cudaStream_t st) {
    CK(cudaMemsetAsync(c->sing.p, 0xff, 8, st));
    return 0;
}

} // namespace detnet

// =========================================================================
// ---- detector baselines -------------------------------------
namespace {
using BaseFn = void (*)(int kind, int blocks, size_t smem, cudaStream_t st, long n, int N,
                        const double *H, const double *y, const double *x, int *errs,
                        unsigned long long *sing);
template <int K>
void launch_baseline(int kind, int blocks, size_t smem, cudaStream_t st, long n, int N,
                     const double *H, const double *y, const double *x, int *errs,
                     unsigned long long *sing) {
    if (kind == 0) {
        cudaFuncSetAttribute(k_zf_errors<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        k_zf_errors<K><<<blocks, 256, smem, st>>>(n, N, H, y, x, errs, sing);
    } else if constexpr (K <= 16) {
        cudaFuncSetAttribute(k_ml_errors<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        k_ml_errors<K><<<blocks, 256, smem, st>>>(n, N, H, y, x, errs);
    }
}
template <int... Ks> constexpr BaseFn base_table(int K, std::integer_sequence<int, Ks...>) {
    BaseFn f = nullptr;
    ((K == Ks + 1 ? (f = launch_baseline<Ks + 1>, 0) : 0), ...);
    return f;
}
} // namespace


extern "C" {

const char *detnet_last_error(void) { return g_err.c_str(); }

int detnet_host_alloc(void **ptr, size_t bytes) {
    if (!ptr) return fail(DETNET_ERR_CONTRACT, "null argument");
    *ptr = nullptr;
    if (bytes == 0) return 0;
    if (cudaMallocHost(ptr, bytes) != cudaSuccess) {
        *ptr = nullptr;
        return fail(DETNET_ERR_CUDA, "pinned host allocation of %zu bytes failed: %s", bytes,
                    cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

int detnet_host_free(void *ptr) {
    if (!ptr) return 0;
    if (cudaFreeHost(ptr) != cudaSuccess)
        return fail(DETNET_ERR_CUDA, "cudaFreeHost: %s", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

long detnet_record_size(int n_tx, int z_dim, int v_dim) { return record_size(n_tx, z_dim, v_dim); }

int detnet_ctx_create(int device, detnet_ctx **out) {
    if (!out) return fail(DETNET_ERR_CONTRACT, "detnet_ctx_create: null out");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return fail(DETNET_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
    if (device < 0 || device >= count) return fail(DETNET_ERR_CONTRACT, "bad device %d", device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(DETNET_ERR_CUDA, "device %d is sm_%d%d; this build targets sm_100a", device,
                    prop.major, prop.minor);
    CK(cudaSetDevice(device));
    auto *c = new detnet_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&c->chunk_done[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->copy_done[i], cudaEventDisableTiming));
    }
    for (const DimsEntry &d : kDims)
        if (d.prep() || (d.prep_fast && d.prep_fast()))
            return fail(DETNET_ERR_CUDA, "cudaFuncSetAttribute (smem) failed");
    if (int rc = tc_prepare()) return rc;
    if (int rc = train_prepare()) return rc; // per device: the backward kernels' smem opt-in
    *out = c;
    return 0;
}

namespace {
void release_model_device(detnet_model *m);
}

void detnet_ctx_destroy(detnet_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    drain_times(c);
    for (detnet_model *m : c->models) { // models outliving their context
        release_model_device(m);
        m->ctx = nullptr;
    }
    c->models.clear();
    for (detnet_ctx *g : c->members) detnet_ctx_destroy(g);
    c->members.clear();
    train_ws_release(c);
    for (DBuf *b : {&c->gp, &c->q32, &c->denom, &c->xmask, &c->flag, &c->tile_loss, &c->tile_err,
                    &c->chunks,
                    &c->sing, &c->result, &c->xhat_dev, &c->state_x, &c->state_v, &c->redo,
                    &c->redo_count, &c->fb_list, &c->fb_count})
        b->release();
    for (int i = 0; i < 2; ++i) {
        c->in_H[i].release(); c->in_y[i].release(); c->in_x[i].release();
        cudaEventDestroy(c->chunk_done[i]);
        cudaEventDestroy(c->copy_done[i]);
    }
    for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
    if (c->h_result) cudaFreeHost(c->h_result);
    if (c->h_async) {
        cudaFreeHost(c->h_async);
        for (cudaEvent_t e : c->async_ev) cudaEventDestroy(e);
    }
    if (c->own_stream) cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->copy_stream);
    delete c;
}

int detnet_ctx_set_path(detnet_ctx *c, int path) {
    if (!c || path < 0 || path > 4) return fail(DETNET_ERR_CONTRACT, "bad path");
    c->path = path;
    for (detnet_ctx *g : c->members) g->path = path;
    return 0;
}

int detnet_ctx_set_train_forward(detnet_ctx *c, int tensor_cores) {
    if (!c) return fail(DETNET_ERR_CONTRACT, "null context");
    c->train_tc = tensor_cores != 0;
    for (detnet_ctx *g : c->members) g->train_tc = c->train_tc;
    return 0;
}

int detnet_ctx_set_exact_preprocess(detnet_ctx *c, int on) {
    if (!c) return fail(DETNET_ERR_CONTRACT, "null ctx");
    c->exact_pre = on != 0;
    for (detnet_ctx *g : c->members) g->exact_pre = c->exact_pre;
    return 0;
}

int detnet_ctx_set_stream(detnet_ctx *c, void *stream) {
    if (!c) return fail(DETNET_ERR_CONTRACT, "null ctx");
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (stream) { c->stream = static_cast<cudaStream_t>(stream); c->own_stream = false; }
    else { CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)); c->own_stream = true; }
    return 0;
}

void *detnet_ctx_stream(detnet_ctx *c) { return c ? c->stream : nullptr; }

int detnet_ctx_set_profiling(detnet_ctx *c, int on) {
    if (!c) return fail(DETNET_ERR_CONTRACT, "null ctx");
    c->profiling = on != 0;
    return 0;
}

int detnet_ctx_kernel_times(detnet_ctx *c, detnet_kernel_times *out, int reset) {
    if (!c || !out) return fail(DETNET_ERR_CONTRACT, "null argument");
    drain_times(c);
    *out = c->times;
    if (reset) c->times = detnet_kernel_times{};
    return 0;
}

long long detnet_ctx_launch_count(detnet_ctx *c) { return c ? c->launches : 0; }

long detnet_ctx_chunk_sums(detnet_ctx *c, double *out, long cap) {
    if (!c) return -fail(DETNET_ERR_CONTRACT, "null context");
    if (cudaSetDevice(c->device) != cudaSuccess || quiesce(c)) return -DETNET_ERR_CUDA;
    const long nc = c->last_chunks;
    if (out && cap > 0 && nc > 0 &&
        cudaMemcpy(out, c->chunks.p, sizeof(double) * std::min(cap, nc), cudaMemcpyDeviceToHost) !=
            cudaSuccess)
        return -fail(DETNET_ERR_CUDA, "chunk sums copy failed");
    return nc;
}

int detnet_model_create(detnet_ctx *c, const detnet_model_desc *d, detnet_model **out) {
    if (!c || !d || !out || !d->params) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (d->n_tx < 1 || d->n_rx < d->n_tx)
        return fail(DETNET_ERR_CONFIG, "need N >= K >= 1 for a full-rank channel");
    if (d->depth < 1 || d->frozen_prefix < 0 || d->frozen_prefix > d->depth)
        return fail(DETNET_ERR_CONTRACT, "bad depth/frozen_prefix");
    const DimsEntry *de = find_dims(d->n_tx, d->z_dim, d->v_dim);
    if (!de)
        return fail(DETNET_ERR_UNSUPPORTED, "dims K=%d z=%d v=%d are not in the compiled kernel set",
                    d->n_tx, d->z_dim, d->v_dim);
    CK(cudaSetDevice(c->device));
    auto *m = new detnet_model();
    m->ctx = c;
    m->K = d->n_tx; m->N = d->n_rx; m->Z = d->z_dim; m->V = d->v_dim;
    m->L = d->depth; m->frozen = d->frozen_prefix; m->dims = de;
    c->models.push_back(m);
    if (int rc = upload_model(m, d)) { detnet_model_destroy(m); return rc; }
    for (detnet_ctx *g : c->members) { // device group: one replica per further member
        detnet_model *r = nullptr;
        if (int rc = detnet_model_create(g, d, &r)) { detnet_model_destroy(m); return rc; }
        m->replicas.push_back(r);
    }
    *out = m;
    return 0;
}

int detnet_model_update(detnet_model *m, const detnet_model_desc *d) {
    if (!m || !d || !d->params) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (d->n_tx != m->K || d->z_dim != m->Z || d->v_dim != m->V || d->n_rx != m->N)
        return fail(DETNET_ERR_CONTRACT, "model_update: dims changed");
    if (d->depth < 1 || d->frozen_prefix < 0 || d->frozen_prefix > d->depth)
        return fail(DETNET_ERR_CONTRACT, "bad depth/frozen_prefix");
    CK(cudaSetDevice(m->ctx->device));
    if (int rc = quiesce(m->ctx)) return rc; // in-flight work may read the buffers released below
    if (d->depth != m->L) {
        m->L = d->depth;
        m->simt.release();
        m->lnk_all.release();
        m->lnk_train.release();
    }
    m->frozen = d->frozen_prefix;
    for (detnet_model *r : m->replicas)
        if (int rc = detnet_model_update(r, d)) return rc;
    m->replicas_stale = false;
    return upload_model(m, d);
}

namespace {
void drop_graph(detnet_model *m);
}

namespace {
void release_model_device(detnet_model *m) {
    cudaSetDevice(m->ctx->device);
    cudaStreamSynchronize(m->ctx->stream); // in-flight work may still read the buffers
    drop_graph(m);
    for (DBuf *b : {&m->simt, &m->lnk_all, &m->lnk_train, &m->tparams, &m->tmasks, &m->tm, &m->tv,
                    &m->sparse_stream, &m->sparse_off, &m->tstatus, &m->bwd_img})
        b->release();
    tc_release(m->tc);
    jit_release(m->jit);
}
} // namespace

void detnet_model_destroy(detnet_model *m) {
    if (!m) return;
    for (detnet_model *r : m->replicas) detnet_model_destroy(r);
    m->replicas.clear();
    if (m->ctx) { // else: orphaned by detnet_ctx_destroy, device state already released
        release_model_device(m);
        auto &v = m->ctx->models;
        v.erase(std::remove(v.begin(), v.end(), m), v.end());
    }
    delete m;
}

int detnet_model_path(const detnet_model *m) {
    if (!m) return 0;
    if (use_jit(m)) return 5;
    if (m->sparse_ready && !m->tc_stale && m->ctx->path == 3 && std::getenv("DETNET_SPARSE_CSR"))
        return 3;
    if (!use_tc(m)) return 1;
    return use_h16(m, false) ? 4 : 2;
}

long long detnet_model_flops_per_detection(const detnet_model *m, int include_pre) {
    if (!m) return -1;
    const long long k = m->K, n = m->N;
    const long P = record_size(m->K, m->Z, m->V);
    const long IN = 3L * m->K + m->V;
    const long spans[3][2] = {{0, m->Z * IN},
                              {m->Z * IN + m->Z, static_cast<long>(m->K) * m->Z},
                              {m->Z * IN + m->Z + static_cast<long>(m->K) * m->Z + m->K,
                               static_cast<long>(m->V) * m->Z}};
    long long flops = 0;
    for (int l = 0; l < m->L; ++l) {
        long long nnz = 0;
        for (auto &sp : spans) {
            if (!m->has_masks) { nnz += sp[1]; continue; }
            const double *mk = m->masks_host.data() + l * P + sp[0];
            for (long i = 0; i < sp[1]; ++i) nnz += mk[i] != 0.0;
        }
        flops += 2 * nnz + 2 * k * k;
    }
    if (include_pre) flops += 2 * n * k + 2 * n * k * k;
    return flops;
}

namespace {
int eval_device_body(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
                     int trainable_only, float *xhat) {
    detnet_ctx *c = m->ctx;
    if (int rc = reset_sing(c, c->stream)) return rc;
    if (int rc = run_pre(m, c->stream, 0, n, n, H, y, x)) return rc;
    const long tiles = (n + TILE - 1) / TILE;
    if (int rc = run_stack(m, c->stream, 0, tiles, n, 0, m->L, trainable_only != 0, xhat, nullptr,
                           nullptr))
        return rc;
    return finish_device(m, n, nullptr);
}

void drop_graph(detnet_model *m) {
    auto &g = m->graph;
    if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto &p : g.timers) {
        m->ctx->event_pool.push_back(p.a);
        m->ctx->event_pool.push_back(p.b);
    }
    g = detnet_model::EvalGraph{};
}

// Capture the body into m->graph (the key is already set). Returns 0 and
// leaves g.exec null when capture is not possible (the caller runs eagerly).
int capture_graph(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
                  int trainable_only, float *xhat) {
    detnet_ctx *c = m->ctx;
    auto &g = m->graph;
    const size_t pend0 = c->pending.size();
    const long long l0 = c->launches;
    long long cl0[8];
    std::memcpy(cl0, c->times.launches, sizeof cl0);
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    const int rc = eval_device_body(m, n, H, y, x, trainable_only, xhat);
    if (g_alloc_epoch != g.epoch) cudaGetLastError(); // allocated while capturing: unusable
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->stream, &graph);
    // the capture pass counted launches and took events but ran nothing
    c->launches = l0;
    std::memcpy(c->times.launches, cl0, sizeof cl0);
    g.timers.assign(c->pending.begin() + static_cast<long>(pend0), c->pending.end());
    c->pending.resize(pend0);
    if (rc || ec != cudaSuccess || !graph || g_alloc_epoch != g.epoch) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return 1; // the caller runs the body eagerly (and reports its errors)
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        cudaGetLastError();
        drop_graph(m);
        return 0;
    }
    g.exec = exec; // g.launches / cls_launches: counted by the eager run of this key
    return 0;
}
} // namespace

int detnet_batch_evaluate_device(detnet_model *m, long n, const float *H, const float *y,
                                 const int8_t *x, int trainable_only, float *xhat,
                                 detnet_eval *out) {
    if (!m || !out || (n > 0 && (!H || !y || !x)))
        return fail(DETNET_ERR_CONTRACT, "null argument");
    detnet_ctx *c = m->ctx;
    *out = detnet_eval{};
    if (n <= 0) return 0; // finish_eval of an empty batch (kernels.cpp:93-103)
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_ws(c, n, m->K)) return rc;
    // Graph replay: a repeated call (same samples, model, settings, buffers)
    // is one cudaGraphLaunch of the whole evaluation. The first call with a
    // key runs eagerly (and allocates what it needs), the second captures.
    static const bool no_graph =
        std::getenv("DETNET_NO_GRAPH") != nullptr || std::getenv("DETNET_TC_TRACE") != nullptr;
    detnet_model::EvalGraph key;
    key.n = n; key.H = H; key.y = y; key.x = x; key.xhat = xhat;
    key.trainable = trainable_only; key.path = c->path; key.exact = c->exact_pre;
    key.profiling = c->profiling; key.version = m->version; key.st = c->stream;
    key.epoch = g_alloc_epoch;
    auto &g = m->graph;
    if (!g.same(key)) {
        drop_graph(m);
        g = key;
        m->graph_seen = 0;
    }
    // (not while profiling: timer events recorded by graph nodes do not time)
    if (!no_graph && !c->profiling && !g.exec && m->graph_seen == 1) {
        if (capture_graph(m, n, H, y, x, trainable_only, xhat) || !g.exec) {
            drop_graph(m); // not capturable here: stay eager for this key
            g = key;
            m->graph_seen = 2;
        }
    }
    if (!no_graph && g.exec) {
        CK(cudaGraphLaunch(g.exec, c->stream));
        c->launches += g.launches;
        for (int k = 0; k < 8; ++k) c->times.launches[k] += g.cls_launches[k];
        return finish_host(m, n, out);
    }
    const long long l0 = c->launches;
    long long cl0[8];
    std::memcpy(cl0, c->times.launches, sizeof cl0);
    if (int rc = eval_device_body(m, n, H, y, x, trainable_only, xhat)) return rc;
    const int rc = finish_host(m, n, out);
    if (rc == 0 && m->graph_seen == 0) {
        g.epoch = g_alloc_epoch; // buffers this call allocated are part of the key
        g.launches = c->launches - l0;
        for (int k = 0; k < 8; ++k) g.cls_launches[k] = c->times.launches[k] - cl0[k];
        m->graph_seen = 1;
    }
    return rc;
}

int detnet_batch_evaluate_device_async(detnet_model *m, long n, const float *H, const float *y,
                                       const int8_t *x, int trainable_only, float *xhat,
                                       long long *ticket) {
    if (!m || !ticket || (n > 0 && (!H || !y || !x)))
        return fail(DETNET_ERR_CONTRACT, "null argument");
    detnet_ctx *c = m->ctx;
    const long long t = c->next_ticket;
    auto &slot = c->slots[t % detnet_ctx::kSlots];
    if (slot.ticket >= 0)
        return fail(DETNET_ERR_CONTRACT, "evaluate_async: %d evaluations in flight (wait first)",
                    detnet_ctx::kSlots);
    CK(cudaSetDevice(c->device));
    if (!c->h_async) {
        CK(cudaMallocHost(&c->h_async, sizeof(double) * 4 * detnet_ctx::kSlots));
        for (auto &e : c->async_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    double *dst = c->h_async + 4 * (t % detnet_ctx::kSlots);
    if (n > 0) {
        if (int rc = ensure_ws(c, n, m->K)) return rc;
        if (int rc = reset_sing(c, c->stream)) return rc;
        if (int rc = run_pre(m, c->stream, 0, n, n, H, y, x)) return rc;
        const long tiles = (n + TILE - 1) / TILE;
        if (int rc = run_stack(m, c->stream, 0, tiles, n, 0, m->L, trainable_only != 0, xhat,
                               nullptr, nullptr))
            return rc;
        if (int rc = finish_device(m, n, dst)) return rc;
    } else {
        dst[0] = 0.0; // finish_eval of an empty batch (kernels.cpp:93-103)
        std::memset(dst + 1, 0, 16);
        std::memset(dst + 3, 0xff, 8);
    }
    CK(cudaEventRecord(c->async_ev[t % detnet_ctx::kSlots], c->stream));
    slot.ticket = t;
    slot.n = n;
    slot.K = m->K;
    ++c->next_ticket;
    *ticket = t;
    drain_times(c, false);
    return 0;
}

int detnet_eval_wait(detnet_ctx *c, long long ticket, detnet_eval *out) {
    if (!c || !out) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (ticket < 0) return fail(DETNET_ERR_CONTRACT, "eval_wait: bad ticket");
    auto &slot = c->slots[ticket % detnet_ctx::kSlots];
    if (slot.ticket != ticket) return fail(DETNET_ERR_CONTRACT, "eval_wait: unknown ticket %lld", ticket);
    CK(cudaEventSynchronize(c->async_ev[ticket % detnet_ctx::kSlots]));
    drain_times(c, false);
    const int rc = decode_eval(c->h_async + 4 * (ticket % detnet_ctx::kSlots), slot.n, slot.K, out);
    slot.ticket = -1;
    return rc;
}

namespace {
// tile-major K1 outputs -> sample-major (one thread per sample)
__global__ void k_untile_pre(long n, int K, const float *gp, const float *q32, float *gram,
                             float *q) {
    const long s = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int NG = gram_entries(K);
    const long tile = s / TILE;
    const int col = static_cast<int>(s % TILE);
    if (gram)
        for (int e = 0; e < NG; ++e) gram[s * NG + e] = gp[(tile * NG + e) * TILE + col];
    if (q)
        for (int k = 0; k < K; ++k) q[s * K + k] = q32[(tile * K + k) * TILE + col];
}
} // namespace

int detnet_preprocess_device(detnet_model *m, long n, const float *H, const float *y,
                             const int8_t *x, float *gram, float *q, double *denom,
                             uint8_t *flag) {
    if (!m || (n > 0 && (!H || !y || !x))) return fail(DETNET_ERR_CONTRACT, "null argument");
    detnet_ctx *c = m->ctx;
    if (n <= 0) return 0;
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_ws(c, n, m->K)) return rc;
    if (int rc = reset_sing(c, c->stream)) return rc;
    if (int rc = run_pre(m, c->stream, 0, n, n, H, y, x)) return rc;
    if (gram || q) {
        LaunchScope ls(c, DETNET_K_OTHER, c->stream);
        k_untile_pre<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(
            n, m->K, c->gp.as<float>(), c->q32.as<float>(), gram, q);
    }
    if (int rc = check_launch()) return rc;
    if (denom) CK(cudaMemcpyAsync(denom, c->denom.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    if (flag) CK(cudaMemcpyAsync(flag, c->flag.p, static_cast<size_t>(n), cudaMemcpyDeviceToDevice, c->stream));
    unsigned long long sing;
    CK(cudaMemcpyAsync(&sing, c->sing.p, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    drain_times(c);
    if (sing != ~0ull)
        return fail(DETNET_ERR_SINGULAR,
                    "solve_normal_equations: matrix is singular to working precision (sample %llu)",
                    sing);
    return 0;
}

int detnet_batch_evaluate(detnet_model *m, long n, const float *H, const float *y,
                          const int8_t *x, int trainable_only, float *xhat_out,
                          detnet_eval *out) {
    if (!m || !out || (n > 0 && (!H || !y || !x)))
        return fail(DETNET_ERR_CONTRACT, "null argument");
    *out = detnet_eval{};
    if (n <= 0) return 0;
    if (!m->replicas.empty()) return group_batch_evaluate(m, n, H, y, x, trainable_only, xhat_out, out);
    return eval_host(m, n, H, y, x, trainable_only, xhat_out, out, nullptr);
}

} // extern "C"

namespace detnet {
int eval_host(detnet_model *m, long n, const float *H, const float *y, const int8_t *x,
              int trainable_only, float *xhat_out, detnet_eval *out, std::vector<double> *chunks) {
    detnet_ctx *c = m->ctx;
    *out = detnet_eval{};
    if (n <= 0) { if (chunks) chunks->clear(); return 0; }
    CK(cudaSetDevice(c->device));
    const int K = m->K, N = m->N, L = m->L;
    if (int rc = ensure_ws(c, n, K)) return rc;
    if (int rc = reset_sing(c, c->stream)) return rc;
    // Chunked streaming: copy chunk i+1 on copy_stream while chunk i computes.
    const long chunk = 1L << 17; // samples, multiple of TILE
    for (int b = 0; b < 2; ++b) {
        const long cs = std::min(chunk, n);
        if (c->in_H[b].ensure(sizeof(float) * cs * N * K) || c->in_y[b].ensure(sizeof(float) * cs * N) ||
            c->in_x[b].ensure(static_cast<size_t>(cs) * K))
            return fail(DETNET_ERR_CUDA, "input staging allocation failed");
    }
    if (xhat_out && c->xhat_dev.ensure(sizeof(float) * std::min(chunk, n) * L * K))
        return fail(DETNET_ERR_CUDA, "xhat staging allocation failed");
    const long nchunks = (n + chunk - 1) / chunk;
    for (long ci = 0; ci < nchunks; ++ci) {
        const int b = static_cast<int>(ci & 1);
        const long s0 = ci * chunk, cnt = std::min(chunk, n - s0);
        if (ci >= 2) CK(cudaStreamWaitEvent(c->copy_stream, c->chunk_done[b], 0));
        CK(cudaMemcpyAsync(c->in_H[b].p, H + s0 * N * K, sizeof(float) * cnt * N * K,
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaMemcpyAsync(c->in_y[b].p, y + s0 * N, sizeof(float) * cnt * N,
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaMemcpyAsync(c->in_x[b].p, x + s0 * K, static_cast<size_t>(cnt) * K,
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaEventRecord(c->copy_done[b], c->copy_stream));
        CK(cudaStreamWaitEvent(c->stream, c->copy_done[b], 0));
        if (int rc = run_pre(m, c->stream, s0, cnt, n, c->in_H[b].as<float>(), c->in_y[b].as<float>(),
                             c->in_x[b].as<int8_t>()))
            return rc;
        const long t0 = s0 / TILE, nt = (cnt + TILE - 1) / TILE;
        if (int rc = run_stack(m, c->stream, t0, nt, cnt, 0, L, trainable_only != 0,
                               xhat_out ? c->xhat_dev.as<float>() : nullptr, nullptr, nullptr))
            return rc;
        if (xhat_out) {
            CK(cudaMemcpyAsync(xhat_out + s0 * L * K, c->xhat_dev.p, sizeof(float) * cnt * L * K,
                               cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaEventRecord(c->chunk_done[b], c->stream));
    }
    if (int rc = finish(m, n, out)) return rc;
    if (chunks) {
        const long nc = ((n + TILE - 1) / TILE + RED_CHUNK_TILES - 1) / RED_CHUNK_TILES;
        chunks->resize(nc);
        CK(cudaMemcpy(chunks->data(), c->chunks.p, sizeof(double) * nc, cudaMemcpyDeviceToHost));
    }
    return 0;
}
} // namespace detnet

extern "C" {

int detnet_forward_range(detnet_model *m, long n, const float *H, const float *y, int l_begin,
                         int l_end, float *x_state, float *v_state, float *xhat_out) {
    if (!m || !H || !y || !x_state || !v_state) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (l_begin < 0 || l_end > m->L || l_begin >= l_end)
        return fail(DETNET_ERR_CONTRACT, "bad layer range [%d,%d)", l_begin, l_end);
    if (n <= 0) return 0;
    detnet_ctx *c = m->ctx;
    CK(cudaSetDevice(c->device));
    const int K = m->K, N = m->N, V = m->V, nl = l_end - l_begin;
    if (int rc = ensure_ws(c, n, K)) return rc;
    if (c->in_H[0].ensure(sizeof(float) * n * N * K) || c->in_y[0].ensure(sizeof(float) * n * N) ||
        c->in_x[0].ensure(static_cast<size_t>(n) * K) || c->state_x.ensure(sizeof(float) * n * K) ||
        c->state_v.ensure(sizeof(float) * n * V) ||
        (xhat_out && c->xhat_dev.ensure(sizeof(float) * n * nl * K)))
        return fail(DETNET_ERR_CUDA, "allocation failed");
    CK(cudaMemcpyAsync(c->in_H[0].p, H, sizeof(float) * n * N * K, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->in_y[0].p, y, sizeof(float) * n * N, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->in_x[0].p, 1, static_cast<size_t>(n) * K, c->stream));
    CK(cudaMemcpyAsync(c->state_x.p, x_state, sizeof(float) * n * K, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->state_v.p, v_state, sizeof(float) * n * V, cudaMemcpyHostToDevice, c->stream));
    if (int rc = reset_sing(c, c->stream)) return rc;
    if (int rc = run_pre(m, c->stream, 0, n, n, c->in_H[0].as<float>(), c->in_y[0].as<float>(),
                         c->in_x[0].as<int8_t>()))
        return rc;
    const long tiles = (n + TILE - 1) / TILE;
    if (int rc = run_stack(m, c->stream, 0, tiles, n, l_begin, l_end, false,
                           xhat_out ? c->xhat_dev.as<float>() : nullptr, c->state_x.as<float>(),
                           c->state_v.as<float>()))
        return rc;
    CK(cudaMemcpyAsync(x_state, c->state_x.p, sizeof(float) * n * K, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(v_state, c->state_v.p, sizeof(float) * n * V, cudaMemcpyDeviceToHost, c->stream));
    if (xhat_out)
        CK(cudaMemcpyAsync(xhat_out, c->xhat_dev.p, sizeof(float) * n * nl * K,
                           cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    drain_times(c);
    return 0;
}

// ---- rng helpers (host) ----------------------------------------------------
uint64_t detnet_rng_seed(uint64_t seed, uint64_t stream_id) {
    return mix64(mix64(seed ^ 0x853c49e6748fea9bULL) + stream_id);
}
uint64_t detnet_rng_stream(uint64_t state, uint64_t id) {
    return mix64(state ^ mix64(id + 0xda3e39cb94b95bdbULL));
}
uint64_t detnet_rng_split(uint64_t *state) {
    *state += kGamma;
    return mix64(mix64(*state));
}

int detnet_generate_device(detnet_ctx *c, uint64_t base, long first, long count, int n_rx,
                           int n_tx, double lo, double hi, double scale, float *H, float *y,
                           int8_t *x, double *sigma2) {
    if (!c || !H || !y || !x) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (count < 1) return fail(DETNET_ERR_CONFIG, "generate_batch: batch size must be >= 1");
    if (n_rx < n_tx || n_tx < 1 || n_tx > 32)
        return fail(DETNET_ERR_CONFIG, "generate_batch: need N >= K >= 1 (K <= 32)");
    CK(cudaSetDevice(c->device));
    const int blocks = static_cast<int>((count + 127) / 128);
    {
        LaunchScope ls(c, DETNET_K_GENERATE, c->stream);
        k_generate<float, int8_t><<<blocks, 128, 0, c->stream>>>(base, first, count, n_rx, n_tx,
                                                                 lo, hi, scale, H, y, x, sigma2);
    }
    if (int rc = check_launch()) return rc;
    CK(cudaStreamSynchronize(c->stream));
    drain_times(c);
    return 0;
}

int detnet_generate_host(detnet_ctx *c, uint64_t base, long first, long count, int n_rx, int n_tx,
                         double lo, double hi, double *H, double *x, double *y, double *sigma2) {
    if (!c || !H || !y || !x) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (count < 1) return fail(DETNET_ERR_CONFIG, "generate_batch: batch size must be >= 1");
    if (n_rx < n_tx || n_tx < 1 || n_tx > 32)
        return fail(DETNET_ERR_CONFIG, "generate_batch: need N >= K >= 1 (K <= 32)");
    CK(cudaSetDevice(c->device));
    const size_t nh = static_cast<size_t>(count) * n_rx * n_tx, ny = static_cast<size_t>(count) * n_rx,
                 nx = static_cast<size_t>(count) * n_tx;
    DBuf buf;
    if (buf.ensure(sizeof(double) * (nh + ny + nx + count)))
        return fail(DETNET_ERR_CUDA, "generator buffer allocation failed");
    double *dH = buf.as<double>(), *dy = dH + nh, *dx = dy + ny, *ds = dx + nx;
    const int blocks = static_cast<int>((count + 127) / 128);
    {
        LaunchScope ls(c, DETNET_K_GENERATE, c->stream);
        k_generate<double, double><<<blocks, 128, 0, c->stream>>>(base, first, count, n_rx, n_tx, lo,
                                                                  hi, 1.0, dH, dy, dx, ds);
    }
    if (int rc = check_launch()) { buf.release(); return rc; }
    cudaMemcpyAsync(H, dH, sizeof(double) * nh, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(y, dy, sizeof(double) * ny, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(x, dx, sizeof(double) * nx, cudaMemcpyDeviceToHost, c->stream);
    if (sigma2) cudaMemcpyAsync(sigma2, ds, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream);
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    buf.release();
    if (e != cudaSuccess) return fail(DETNET_ERR_CUDA, "generate_host: %s", cudaGetErrorString(e));
    drain_times(c);
    return 0;
}


int detnet_batch_baseline_errors(detnet_ctx *c, int kind, long n, int n_rx, int n_tx,
                                 const double *H, const double *y, const double *x,
                                 long long *errors, long long *symbols) {
    if (!c || !errors || !symbols) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (n < 0) return fail(DETNET_ERR_CONTRACT, "batch_baseline_errors: negative batch size");
    *errors = 0;
    *symbols = n * static_cast<long long>(n_tx);
    if (kind == 2 || n == 0) return 0; // oracle baseline: no errors (kernels.cpp:105-106)
    if (kind != 0 && kind != 1) return fail(DETNET_ERR_CONTRACT, "baseline kind must be 0 (zf), 1 (ml) or 2");
    if (!H || !y || !x) return fail(DETNET_ERR_CONTRACT, "null argument");
    if (n_tx < 1 || n_rx < n_tx) return fail(DETNET_ERR_CONTRACT, "baseline: need N >= K >= 1");
    if (kind == 1 && n_tx > 16)
        return fail(DETNET_ERR_UNSUPPORTED, "ml_decode: exhaustive search limited to K <= 16");
    // K <= 20: register-resident instantiations; wider ZF: k_zf_errors_any with
    // the warp's [A | x] in shared memory (up to ~160 transmit antennas)
    const BaseFn fn = base_table(n_tx, std::make_integer_sequence<int, 20>{});
    const size_t any_per = sizeof(double) * static_cast<size_t>(n_tx) * (n_tx + 1);
    const int any_warps = static_cast<int>(std::min<size_t>(4, (200u << 10) / any_per));
    if (!fn && (kind != 0 || any_per > (227u << 10)))
        return fail(DETNET_ERR_UNSUPPORTED, "baseline: K = %d exceeds the device ZF limit", n_tx);
    CK(cudaSetDevice(c->device));
    const long chunk = std::min<long>(n, 1L << 16);
    const size_t nh = static_cast<size_t>(chunk) * n_rx * n_tx, ny = static_cast<size_t>(chunk) * n_rx,
                 nx = static_cast<size_t>(chunk) * n_tx;
    DBuf buf;
    if (buf.ensure(sizeof(double) * (nh + ny + nx) + sizeof(int) * chunk + 16))
        return fail(DETNET_ERR_CUDA, "baseline buffer allocation failed");
    double *dH = buf.as<double>(), *dy = dH + nh, *dx = dy + ny;
    int *de = reinterpret_cast<int *>(dx + nx);
    unsigned long long *ds = reinterpret_cast<unsigned long long *>(de + chunk + (chunk & 1));
    const size_t smem = sizeof(double) * 8 *
                        (static_cast<size_t>(n_rx) * n_tx + n_rx + n_tx * n_tx + n_tx);
    std::vector<int> he(chunk);
    long long total = 0;
    for (long s0 = 0; s0 < n; s0 += chunk) {
        const long cnt = std::min(chunk, n - s0);
        CK(cudaMemcpyAsync(dH, H + s0 * n_rx * n_tx, sizeof(double) * cnt * n_rx * n_tx,
                           cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(dy, y + s0 * n_rx, sizeof(double) * cnt * n_rx, cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaMemcpyAsync(dx, x + s0 * n_tx, sizeof(double) * cnt * n_tx, cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaMemsetAsync(ds, 0xff, 8, c->stream));
        const int blocks = static_cast<int>(std::min<long>((cnt + 7) / 8, 148L * 16));
        {
            LaunchScope ls(c, DETNET_K_OTHER, c->stream);
            if (fn) {
                fn(kind, blocks, smem, c->stream, cnt, n_rx, dH, dy, dx, de, ds);
            } else {
                const int w = std::max(1, any_warps);
                const size_t sm_any = any_per * w;
                cudaFuncSetAttribute(k_zf_errors_any, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm_any));
                const int bl = static_cast<int>(std::min<long>((cnt + w - 1) / w, 148L * 8));
                k_zf_errors_any<<<bl, 32 * w, sm_any, c->stream>>>(cnt, n_rx, n_tx, dH, dy, dx, de, ds);
            }
        }
        if (int rc = check_launch()) { buf.release(); return rc; }
        unsigned long long sing = ~0ull;
        CK(cudaMemcpyAsync(he.data(), de, sizeof(int) * cnt, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&sing, ds, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (sing != ~0ull) {
            buf.release();
            return fail(DETNET_ERR_SINGULAR,
                        "solve_normal_equations: matrix is singular to working precision (sample %llu)",
                        static_cast<unsigned long long>(s0) + sing);
        }
        for (long i = 0; i < cnt; ++i) total += he[i]; // sample order
    }
    buf.release();
    drain_times(c);
    *errors = total;
    return 0;
}

// ---- training ----------------------------------------------------------------
int detnet_batch_gradient(detnet_model *m, long n, const float *H, const float *y,
                          const int8_t *x, const detnet_loss_spec *spec, int trainable_only,
                          double *grads_out, detnet_eval *out) {
    if (m && !m->replicas.empty() && !m->ctx->train_fp64)
        return group_batch_gradient(m, n, H, y, x, spec, trainable_only, grads_out, out);
    return train_batch_gradient(m, n, H, y, x, spec, trainable_only, grads_out, out);
}

int detnet_adam_step(detnet_ctx *c, int n_tx, int z_dim, int v_dim, int depth, int frozen_prefix,
                     double *params, const double *masks, const double *grads, double *m1,
                     double *m2, int64_t *step, const detnet_adam_config *cfg) {
    return train_adam_step(c, n_tx, z_dim, v_dim, depth, frozen_prefix, params, masks, grads, m1,
                           m2, step, cfg);
}

} // extern "C"
