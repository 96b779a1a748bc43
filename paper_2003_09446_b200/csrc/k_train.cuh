// k_train.cuh -- training-step kernels (BASELINE config 5): the reverse sweep
// of backward_data (backward.cpp:105-165), the batch reductions that turn it
// into weight gradients, the regularizer gradient (backward.cpp:169-220) and
// Adam (adam.cpp:48-79).
//
// Data layout: the forward pass (k_stack_simt with trace pointers) records,
// feature-major / sample-minor ([l][feature][ts]), the layer input
// in = [q; x; Gx; v], z = relu(u1) and u2, plus x_hat_L. The backward sweep
// (one thread per sample, all trainable layers, weights double-buffered in
// shared memory in reverse layer order) writes the per-sample adjoints
//   u1bar [l][Z][ts],  g23bar [l][K+V][ts] = [u2bar; vbar]
// and per-CTA partial t-gradients. The weight gradients are then batch
// contractions over the sample axis,
//   dW1 = u1bar . in^T,  dW2|dW3 = [u2bar; vbar] . z^T  (+ bias = row sums),
// computed by a split-K kernel (FP32 inside a split of DW_SPLIT = 1024
// samples, FP64 across splits, fixed order => deterministic; tcgen05 in
// dw_tc.cu, CUDA cores in k_dw_gemm below), scaled by 1/n, masked and
// combined with the regularizer gradient in FP64.
#pragma once

#include "common.cuh"
#include "dw_job.hpp"
#include "k_stack_simt.cuh"

namespace detnet {

// BwdArgs: dw_job.hpp (shared with the tcgen05 sweep, bwd_tc.cu)

// THREADS samples per CTA (one CTA per SM: the double-buffered weights take
// ~210 KB of shared memory): 256 for large batches, 64 for small ones -- at the
// config-5 batch (5,000 samples) that spreads the per-sample reverse sweeps
// over 79 SMs instead of 20.
template <int K, int Z, int V, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_train_bwd(BwdArgs a) {
    constexpr int IN = 3 * K + V;
    constexpr int IN4 = simt_in4(K, V);
    constexpr int O = K + V;
    constexpr int O4 = simt_o4(K, V);
    constexpr int NG = gram_entries(K);
    constexpr int REC = static_cast<int>(simt_rec(K, Z, V));
    extern __shared__ __align__(128) float sw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sw + 2 * REC);

    const int tid = threadIdx.x;
    const long unit = static_cast<long>(blockIdx.x) * THREADS + tid;
    const long tile_l = unit / TILE;
    const bool live_tile = tile_l < a.n_tiles;
    const long tile = live_tile ? tile_l : a.n_tiles - 1;
    const int col = static_cast<int>(unit % TILE);
    const long s = tile * TILE + col;
    const bool live = live_tile && s < a.n;
    DETNET_DASSERT(tile >= 0 && s < a.ts);

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t bytes = static_cast<uint32_t>(REC) * 4u;
    const int nl = a.L - a.lf;
    if (tid == 0) {
        for (int b = 0; b < 2 && b < nl; ++b) {
            mbar_arrive_expect_tx(&bars[b], bytes);
            bulk_g2s_chunked(sw + b * REC, a.wrec + static_cast<long>(a.L - 1 - b) * a.rec_floats,
                             bytes, &bars[b]);
        }
    }
    const uint32_t xm = a.xmask[tile * TILE + col];
    const float dinv2 = static_cast<float>(2.0 / a.denom[tile * TILE + col]);
    const float *gps = a.gp + tile * NG * TILE + col;
    float abar[K], vbar[V];
#pragma unroll
    for (int k = 0; k < K; ++k) abar[k] = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) vbar[k] = 0.f;

    for (int it = 0; it < nl; ++it) {
        const int l = a.L - 1 - it;
        const int b = it & 1;
        mbar_wait(&bars[b], (it >> 1) & 1);
        const float *W = sw + b * REC;
        // a_bar += 2 ln(l+1)/denom (x_hat_{l+1} - x)
        const float w = static_cast<float>(a.lnk[l]) * dinv2;
        const float *xn = l + 1 < a.L ? a.tr_in + (static_cast<long>(l + 1) * IN + K) * a.ts + s
                                      : a.tr_xf + s;
        const float t = W[Z * IN4 + Z * O4 + O4];
        const float tinv = 1.f / t;
        float u2bar[K];
        float tb = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float xk = (xm >> k) & 1u ? 1.f : -1.f;
            abar[k] = fmaf(w, xn[k * a.ts] - xk, abar[k]);
            const float u = a.tr_u2[(static_cast<long>(l) * K + k) * a.ts + s];
            const bool lin = u >= -t && u < t; // model.cpp:45-51
            u2bar[k] = lin ? abar[k] * tinv : 0.f;
            tb += lin ? abar[k] * (-u * tinv * tinv) : 0.f;
        }
        // threads of a clamped (dead) second tile alias a live tile: no writes
        float *g23 = a.g23bar + static_cast<long>(l) * O * a.ts + s;
        if (live_tile) {
#pragma unroll
            for (int k = 0; k < K; ++k) g23[k * a.ts] = live ? u2bar[k] : 0.f;
#pragma unroll
            for (int k = 0; k < V; ++k) g23[(K + k) * a.ts] = live ? vbar[k] : 0.f;
        }
        // z_bar = W2^T u2bar + W3^T vbar; u1bar = z_bar [u1 > 0]; in_bar = W1^T u1bar
        float ibar[IN - K]; // x, Gx, v blocks (the q block is data)
#pragma unroll
        for (int j = 0; j < IN - K; ++j) ibar[j] = 0.f;
        const float *zl = a.tr_z + static_cast<long>(l) * Z * a.ts + s;
        float *u1b = a.u1bar + static_cast<long>(l) * Z * a.ts + s;
        // hidden units in groups of 8: the group's z trace values are loaded
        // up front (8 independent L2 reads in flight instead of one per unit)
        static_assert(Z % 8 == 0, "hidden width in groups of 8");
#pragma unroll 1
        for (int i0 = 0; i0 < Z; i0 += 8) {
            float zg[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) zg[q] = zl[(i0 + q) * a.ts];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int i = i0 + q;
                const float4 *c4 = reinterpret_cast<const float4 *>(W + Z * IN4 + i * O4);
                float zb0 = 0.f, zb1 = 0.f;
#pragma unroll
                for (int m = 0; m < O4 / 4; ++m) {
                    const float4 c = c4[m];
#define DETNET_G(j) ((j) < K ? u2bar[(j) < K ? (j) : 0] : vbar[((j) - K) < V ? (j) - K : 0])
                    if (4 * m + 3 < O) { // the same two chains, as FFMA2 pairs
                        fma_x2(zb0, zb1, c.x, c.y, DETNET_G(4 * m + 0), DETNET_G(4 * m + 1));
                        fma_x2(zb0, zb1, c.z, c.w, DETNET_G(4 * m + 2), DETNET_G(4 * m + 3));
                    } else {
                        if (4 * m + 0 < O) zb0 = fmaf(c.x, DETNET_G(4 * m + 0), zb0);
                        if (4 * m + 1 < O) zb1 = fmaf(c.y, DETNET_G(4 * m + 1), zb1);
                        if (4 * m + 2 < O) zb0 = fmaf(c.z, DETNET_G(4 * m + 2), zb0);
                        if (4 * m + 3 < O) zb1 = fmaf(c.w, DETNET_G(4 * m + 3), zb1);
                    }
#undef DETNET_G
                }
                const float ub = zg[q] > 0.f ? zb0 + zb1 : 0.f;
                if (live_tile) u1b[i * a.ts] = live ? ub : 0.f;
                const float4 *w4 = reinterpret_cast<const float4 *>(W + i * IN4);
#pragma unroll
                for (int m = K / 4; m < IN4 / 4; ++m) {
                    const float4 wv = w4[m];
                    if (4 * m >= K && 4 * m + 3 < IN) {
                        fma_x2(ibar[4 * m - K], ibar[4 * m + 1 - K], wv.x, wv.y, ub, ub);
                        fma_x2(ibar[4 * m + 2 - K], ibar[4 * m + 3 - K], wv.z, wv.w, ub, ub);
                        continue;
                    }
#define DETNET_IB(c, wc)                                                                        \
    if (4 * m + (c) >= K && 4 * m + (c) < IN)                                                    \
        ibar[(4 * m + (c) - K) >= 0 ? 4 * m + (c) - K : 0] =                                    \
            fmaf(wc, ub, ibar[(4 * m + (c) - K) >= 0 ? 4 * m + (c) - K : 0]);
                    DETNET_IB(0, wv.x)
                    DETNET_IB(1, wv.y)
                    DETNET_IB(2, wv.z)
                    DETNET_IB(3, wv.w)
#undef DETNET_IB
                }
            }
        }
        // a_bar <- G gx_bar + x_bar (G symmetric); v_bar <- v block
#pragma unroll
        for (int k = 0; k < K; ++k) abar[k] = ibar[k];
        {
            int e = 0;
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int c = r; c < K; ++c, ++e) {
                    const float g = __ldg(gps + e * TILE);
                    abar[r] = fmaf(g, ibar[K + c], abar[r]);
                    if (c != r) abar[c] = fmaf(g, ibar[K + r], abar[c]);
                }
        }
#pragma unroll
        for (int k = 0; k < V; ++k) vbar[k] = ibar[2 * K + k];
        // t gradient per 32-sample group (deterministic tree; the same groups
        // in every kernel variant, so the sum does not depend on the launch shape)
        double tsum = live ? static_cast<double>(tb) : 0.0;
        tsum = warp_sum(tsum);
        if ((tid & 31) == 0 && live_tile) a.tbar_part[static_cast<long>(l) * (a.ts / 32) + s / 32] = tsum;
        __syncthreads(); // every thread is done reading buffer b
        if (tid == 0) {
            if (it + 2 < nl) {
                mbar_arrive_expect_tx(&bars[b], bytes);
                bulk_g2s_chunked(sw + b * REC,
                                 a.wrec + static_cast<long>(a.L - 1 - (it + 2)) * a.rec_floats,
                                 bytes, &bars[b]);
            }
        }
    }
}

// Small-batch variant of the reverse sweep: two threads per sample. Warps 0-1
// ("A") take hidden units [0, Z/2), warps 2-3 ("B") units [Z/2, Z) of the same
// 64 samples; B's in_bar partial meets A's in shared memory, A forms
// a_bar = G gx_bar + x_bar and v_bar and hands them back. The per-sample serial
// chain halves. Weights are single-buffered (the exchange buffers take the
// second slot); the next layer's copy is issued as soon as the last weight
// read of this layer is done, under the exchange and the next layer's prologue.
constexpr int BWP_SAMPLES = 64, BWP_THREADS = 128;

template <int K, int Z, int V>
__global__ void __launch_bounds__(BWP_THREADS, 1) k_train_bwd_pair(BwdArgs a) {
    constexpr int IN = 3 * K + V;
    constexpr int IN4 = simt_in4(K, V);
    constexpr int O = K + V;
    constexpr int O4 = simt_o4(K, V);
    constexpr int NG = gram_entries(K);
    constexpr int REC = static_cast<int>(simt_rec(K, Z, V));
    constexpr int ZH = Z / 2, NIB = IN - K, P = BWP_SAMPLES;
    constexpr int GRP = ZH % 8 == 0 ? 8 : (ZH % 4 == 0 ? 4 : 1); // z-trace prefetch group
    static_assert(Z % 2 == 0, "hidden units split in halves");
    extern __shared__ __align__(128) float sw[];
    float(*sIB)[P] = reinterpret_cast<float(*)[P]>(sw + REC);       // [NIB][P] B -> A
    float(*sAV)[P] = reinterpret_cast<float(*)[P]>(sw + REC + NIB * P); // [K+V][P] A -> B
    uint64_t *bar = reinterpret_cast<uint64_t *>(sw + REC + (NIB + O) * P);

    const int tid = threadIdx.x, warp = tid >> 5;
    const bool isA = warp < 2;
    const int ls = (warp & 1) * 32 + (tid & 31);
    const int pbar = 1 + (warp & 1);
    const long unit = static_cast<long>(blockIdx.x) * P + ls;
    const long tile_l = unit / TILE;
    const bool live_tile = tile_l < a.n_tiles;
    const long tile = live_tile ? tile_l : a.n_tiles - 1;
    const int col = static_cast<int>(unit % TILE);
    const long s = tile * TILE + col;
    const bool live = live_tile && s < a.n;
    const int i0 = isA ? 0 : ZH;

    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t bytes = static_cast<uint32_t>(REC) * 4u;
    const int nl_all = a.L - a.lf;
    const int it0 = a.it_begin, it1 = a.it_end < 0 ? nl_all : a.it_end;
    if (tid == 0 && it0 < it1) {
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s_chunked(sw, a.wrec + static_cast<long>(a.L - 1 - it0) * a.rec_floats, bytes, bar);
    }
    const uint32_t xm = a.xmask[tile * TILE + col];
    const float dinv2 = static_cast<float>(2.0 / a.denom[tile * TILE + col]);
    const float *gps = a.gp + tile * NG * TILE + col;
    float abar[K], vbar[V];
    if (it0 > 0) { // a later chunk: the state the previous chunk left
#pragma unroll
        for (int k = 0; k < K; ++k) abar[k] = a.state[k * a.ts + s];
#pragma unroll
        for (int k = 0; k < V; ++k) vbar[k] = a.state[(K + k) * a.ts + s];
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) abar[k] = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k) vbar[k] = 0.f;
    }

    for (int it = it0; it < it1; ++it) {
        const int l = a.L - 1 - it;
        mbar_wait(bar, (it - it0) & 1);
        const float *W = sw;
        const float w = static_cast<float>(a.lnk[l]) * dinv2;
        const float *xn = l + 1 < a.L ? a.tr_in + (static_cast<long>(l + 1) * IN + K) * a.ts + s
                                      : a.tr_xf + s;
        const float t = W[Z * IN4 + Z * O4 + O4];
        const float tinv = 1.f / t;
        float u2bar[K];
        float tb = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float xk = (xm >> k) & 1u ? 1.f : -1.f;
            abar[k] = fmaf(w, xn[k * a.ts] - xk, abar[k]);
            const float u = a.tr_u2[(static_cast<long>(l) * K + k) * a.ts + s];
            const bool lin = u >= -t && u < t; // model.cpp:45-51
            u2bar[k] = lin ? abar[k] * tinv : 0.f;
            tb += lin ? abar[k] * (-u * tinv * tinv) : 0.f;
        }
        if (isA && live_tile) {
            float *g23 = a.g23bar + static_cast<long>(l) * O * a.ts + s;
#pragma unroll
            for (int k = 0; k < K; ++k) g23[k * a.ts] = live ? u2bar[k] : 0.f;
#pragma unroll
            for (int k = 0; k < V; ++k) g23[(K + k) * a.ts] = live ? vbar[k] : 0.f;
        }
        // this thread's half of the hidden units: z_bar, u1_bar, in_bar partial
        float ibar[NIB];
#pragma unroll
        for (int j = 0; j < NIB; ++j) ibar[j] = 0.f;
        const float *zl = a.tr_z + static_cast<long>(l) * Z * a.ts + s;
        float *u1b = a.u1bar + static_cast<long>(l) * Z * a.ts + s;
#pragma unroll 1
        for (int g0 = i0; g0 < i0 + ZH; g0 += GRP) {
            float zg[GRP];
#pragma unroll
            for (int q = 0; q < GRP; ++q) zg[q] = zl[(g0 + q) * a.ts];
#pragma unroll
            for (int q = 0; q < GRP; ++q) {
                const int i = g0 + q;
                const float4 *c4 = reinterpret_cast<const float4 *>(W + Z * IN4 + i * O4);
                float zb0 = 0.f, zb1 = 0.f;
#pragma unroll
                for (int m = 0; m < O4 / 4; ++m) {
                    const float4 c = c4[m];
#define DETNET_G(j) ((j) < K ? u2bar[(j) < K ? (j) : 0] : vbar[((j) - K) < V ? (j) - K : 0])
                    if (4 * m + 3 < O) { // the same two chains, as FFMA2 pairs
                        fma_x2(zb0, zb1, c.x, c.y, DETNET_G(4 * m + 0), DETNET_G(4 * m + 1));
                        fma_x2(zb0, zb1, c.z, c.w, DETNET_G(4 * m + 2), DETNET_G(4 * m + 3));
                    } else {
                        if (4 * m + 0 < O) zb0 = fmaf(c.x, DETNET_G(4 * m + 0), zb0);
                        if (4 * m + 1 < O) zb1 = fmaf(c.y, DETNET_G(4 * m + 1), zb1);
                        if (4 * m + 2 < O) zb0 = fmaf(c.z, DETNET_G(4 * m + 2), zb0);
                        if (4 * m + 3 < O) zb1 = fmaf(c.w, DETNET_G(4 * m + 3), zb1);
                    }
#undef DETNET_G
                }
                const float ub = zg[q] > 0.f ? zb0 + zb1 : 0.f;
                if (live_tile) u1b[i * a.ts] = live ? ub : 0.f;
                const float4 *w4 = reinterpret_cast<const float4 *>(W + i * IN4);
#pragma unroll
                for (int m = K / 4; m < IN4 / 4; ++m) {
                    const float4 wv = w4[m];
                    if (4 * m >= K && 4 * m + 3 < IN) {
                        fma_x2(ibar[4 * m - K], ibar[4 * m + 1 - K], wv.x, wv.y, ub, ub);
                        fma_x2(ibar[4 * m + 2 - K], ibar[4 * m + 3 - K], wv.z, wv.w, ub, ub);
                        continue;
                    }
#define DETNET_IB(c, wc)                                                                        \
    if (4 * m + (c) >= K && 4 * m + (c) < IN)                                                    \
        ibar[(4 * m + (c) - K) >= 0 ? 4 * m + (c) - K : 0] =                                    \
            fmaf(wc, ub, ibar[(4 * m + (c) - K) >= 0 ? 4 * m + (c) - K : 0]);
                    DETNET_IB(0, wv.x)
                    DETNET_IB(1, wv.y)
                    DETNET_IB(2, wv.z)
                    DETNET_IB(3, wv.w)
#undef DETNET_IB
                }
            }
        }
        // every weight read of layer l is done: stream layer l-1 in now
        __syncthreads();
        if (tid == 0 && it + 1 < it1) {
            mbar_arrive_expect_tx(bar, bytes);
            bulk_g2s_chunked(sw, a.wrec + static_cast<long>(l - 1) * a.rec_floats, bytes, bar);
        }
        if (!isA) {
#pragma unroll
            for (int j = 0; j < NIB; ++j) sIB[j][ls] = ibar[j];
        }
        named_bar_sync(pbar, 64);
        if (isA) {
#pragma unroll
            for (int j = 0; j < NIB; ++j) ibar[j] += sIB[j][ls];
            // a_bar <- G gx_bar + x_bar (G symmetric); v_bar <- v block
#pragma unroll
            for (int k = 0; k < K; ++k) abar[k] = ibar[k];
            int e = 0;
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int c = r; c < K; ++c, ++e) {
                    const float g = __ldg(gps + e * TILE);
                    abar[r] = fmaf(g, ibar[K + c], abar[r]);
                    if (c != r) abar[c] = fmaf(g, ibar[K + r], abar[c]);
                }
#pragma unroll
            for (int k = 0; k < V; ++k) vbar[k] = ibar[2 * K + k];
#pragma unroll
            for (int k = 0; k < K; ++k) sAV[k][ls] = abar[k];
#pragma unroll
            for (int k = 0; k < V; ++k) sAV[K + k][ls] = vbar[k];
        }
        named_bar_sync(pbar, 64);
        if (!isA) {
#pragma unroll
            for (int k = 0; k < K; ++k) abar[k] = sAV[k][ls];
#pragma unroll
            for (int k = 0; k < V; ++k) vbar[k] = sAV[K + k][ls];
        }
        // t gradient per 32-sample group (A warps; same groups as k_train_bwd)
        double tsum = (isA && live) ? static_cast<double>(tb) : 0.0;
        tsum = warp_sum(tsum);
        if (isA && (tid & 31) == 0 && live_tile)
            a.tbar_part[static_cast<long>(l) * (a.ts / 32) + s / 32] = tsum;
        __syncthreads(); // B is done reading sAV before A rewrites it
    }
    if (it1 < nl_all && isA && live_tile) { // hand the sweep state to the next chunk
#pragma unroll
        for (int k = 0; k < K; ++k) a.state[k * a.ts + s] = abar[k];
#pragma unroll
        for (int k = 0; k < V; ++k) a.state[(K + k) * a.ts + s] = vbar[k];
    }
}

// 64 x 64 output tile per CTA, 4 x 4 per thread (two 128-bit shared loads per
// 16 FMAs), K = samples in chunks of 32; FP32 inside a split of DW_SPLIT
// samples, one FP64 partial per split (summed in fixed order by k_grad_sum).
// (DwJob and DW_SPLIT: dw_job.hpp, shared with the tcgen05 kernel dw_tc.cu.)
constexpr int DW_TILE = 64, DW_KC = 32;
// (FP64 accumulation here was measured not to change the FP32-vs-FP64 training
// drift, which comes from gate flips in the FP32 forward/backward.)
using DW_ACC = float;
__device__ __forceinline__ float dw_fma(float a, float b, float c) { return fmaf(a, b, c); }
// (d0, d1) += a * (b0, b1) as one fma.rn.f32x2
__device__ __forceinline__ void dw_fma2(float &d0, float &d1, float a, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %2};\n\tmov.b64 rb, {%3, %4};\n\tmov.b64 rd, {%0, %1};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rd;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a), "f"(b0), "f"(b1));
}

// grid: (N tiles, M tiles, jobs x splits) -- one (tile, split) per CTA
__global__ void __launch_bounds__(256) k_dw_gemm(const DwJob *jobs, long n, long ts, int splits) {
    const DwJob jb = jobs[blockIdx.z / splits];
    const int m0 = blockIdx.y * DW_TILE, n0 = blockIdx.x * DW_TILE;
    if (m0 >= jb.M || n0 > jb.N) return;
    // rows padded by 4 floats: the transposing stores (32 consecutive samples
    // of a row per warp) spread over 8 banks instead of 1; 128-bit reads stay
    // aligned. Two buffers: chunk c+1 is fetched into registers while chunk c
    // is multiplied, then stored to the other buffer (one barrier per chunk).
    __shared__ __align__(16) float sA[2][DW_KC][DW_TILE + 4], sB[2][DW_KC][DW_TILE + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4; // 16 x 16 threads, 4 x 4 outputs
    const int sp = static_cast<int>(blockIdx.z % splits);
    const long k0 = static_cast<long>(sp) * DW_SPLIT;
    const long k1 = k0 + DW_SPLIT < n ? k0 + DW_SPLIT : n;
    DW_ACC c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = 0;
    // 64 rows x 32 samples of A and of B per chunk: each thread moves 8 + 8
    // floats (consecutive threads -> consecutive samples of a row: coalesced)
    float ra[8], rb[8];
    auto gload = [&](long kc) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int idx = threadIdx.x + 256 * r;
            const int kk = idx % DW_KC, row = idx / DW_KC;
            const long k = kc + kk;
            const bool in = k < k1;
            const int mr = m0 + row, nr = n0 + row;
            ra[r] = (in && mr < jb.M) ? __ldg(jb.A + static_cast<long>(mr) * ts + k) : 0.f;
            rb[r] = (in && nr < jb.N) ? __ldg(jb.B + static_cast<long>(nr) * ts + k)
                                      : ((in && nr == jb.N) ? 1.f : 0.f);
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int idx = threadIdx.x + 256 * r;
            const int kk = idx % DW_KC, row = idx / DW_KC;
            sA[buf][kk][row] = ra[r];
            sB[buf][kk][row] = rb[r];
        }
    };
    gload(k0);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (long kc = k0; kc < k1; kc += DW_KC) {
        const bool more = kc + DW_KC < k1;
        if (more) gload(kc + DW_KC);
        // per output: samples in order, as before (bit-identical partials)
#pragma unroll 8
        for (int kk = 0; kk < DW_KC; ++kk) {
            const float4 a4 = *reinterpret_cast<const float4 *>(&sA[buf][kk][ty * 4]);
            const float4 b4 = *reinterpret_cast<const float4 *>(&sB[buf][kk][tx * 4]);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
            // FFMA2: two fused multiply-adds per instruction, each rounded as fmaf
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; j += 2) dw_fma2(c[i][j], c[i][j + 1], av[i], bv[j], bv[j + 1]);
        }
        if (more) sstore(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int mr = m0 + ty * 4 + i, nc = n0 + tx * 4 + j;
            if (mr < jb.M && nc <= jb.N)
                jb.out[(static_cast<long>(sp) * jb.M + mr) * (jb.N + 1) + nc] = c[i][j];
        }
}

struct SumArgs {
    const double *p1;     // W1 partials [L][splits][Z][IN+1]
    const double *p23;    // W23 partials [L][splits][K+V][Z+1]
    const double *tpart;  // [L][tgroups] (32-sample groups)
    int tgroups, splits;
    int K, Z, V, L, lf;
    double *raw;          // [L][P] unscaled, unmasked data-gradient sums (record layout)
    double *chunk_out;    // optional [chunks][L][P]: the per-chunk sums (device groups)
    int l_lo, l_hi;       // layers this launch finalises (a bucket of the overlapped sweep)
};

// Chunk = 8,192 consecutive samples = 32 dW splits = 256 t groups. The raw
// sums are folded in a canonical two-level order -- within each chunk in
// split order, then the chunk sums in chunk order -- which does not depend on
// how a batch is sharded over launches or devices (shards start at chunk
// boundaries), so a device group reproduces the single-device bits.
constexpr int GRAD_CHUNK_SPLITS = 8192 / DW_SPLIT, GRAD_CHUNK_GROUPS = 8192 / 32;

// Sum the split partials in fixed order (FP64) into record layout. The raw
// sums are what ranks all-reduce (sum) before the update.
__global__ void k_grad_sum(SumArgs a) {
    const int K = a.K, Z = a.Z, V = a.V, IN = 3 * K + V;
    const int P = Z * IN + Z + K * Z + K + V * Z + V + 1;
    const long idx = static_cast<long>(a.l_lo) * P + static_cast<long>(blockIdx.x) * blockDim.x +
                     threadIdx.x;
    if (idx >= static_cast<long>(a.l_hi) * P) return;
    const int l = static_cast<int>(idx / P), e = static_cast<int>(idx % P);
    DETNET_DASSERT(a.splits >= 1 && a.tgroups >= 1 && a.lf >= 0 && a.lf <= a.L);
    if (l < a.lf) { a.raw[idx] = 0.0; return; }
    const int ob1 = Z * IN, oW2 = ob1 + Z, ob2 = oW2 + K * Z, oW3 = ob2 + K, ob3 = oW3 + V * Z, ot = ob3 + V;
    const long total = static_cast<long>(a.L) * P;
    double sum = 0.0;
    if (e == ot) {
        const double *tp = a.tpart + static_cast<long>(l) * a.tgroups;
        for (int c0 = 0, ch = 0; c0 < a.tgroups; c0 += GRAD_CHUNK_GROUPS, ++ch) {
            double cs = 0.0;
            const int c1 = c0 + GRAD_CHUNK_GROUPS < a.tgroups ? c0 + GRAD_CHUNK_GROUPS : a.tgroups;
            for (int g = c0; g < c1; ++g) cs += tp[g];
            if (a.chunk_out) a.chunk_out[ch * total + idx] = cs;
            sum += cs;
        }
    } else {
        const double *src;
        long stride, base;
        if (e < ob1) { // W1[i][j]
            src = a.p1 + static_cast<long>(l) * a.splits * Z * (IN + 1);
            base = static_cast<long>(e / IN) * (IN + 1) + e % IN;
            stride = static_cast<long>(Z) * (IN + 1);
        } else if (e < oW2) { // b1[i]
            src = a.p1 + static_cast<long>(l) * a.splits * Z * (IN + 1);
            base = static_cast<long>(e - ob1) * (IN + 1) + IN;
            stride = static_cast<long>(Z) * (IN + 1);
        } else {
            int r, c;
            if (e < ob2) { r = (e - oW2) / Z; c = (e - oW2) % Z; }          // W2[k][i]
            else if (e < oW3) { r = e - ob2; c = Z; }                        // b2[k]
            else if (e < ob3) { r = K + (e - oW3) / Z; c = (e - oW3) % Z; } // W3[v][i]
            else { r = K + (e - ob3); c = Z; }                               // b3[v]
            src = a.p23 + static_cast<long>(l) * a.splits * (K + V) * (Z + 1);
            base = static_cast<long>(r) * (Z + 1) + c;
            stride = static_cast<long>(K + V) * (Z + 1);
        }
        for (int c0 = 0, ch = 0; c0 < a.splits; c0 += GRAD_CHUNK_SPLITS, ++ch) {
            double cs = 0.0;
            const int c1 = c0 + GRAD_CHUNK_SPLITS < a.splits ? c0 + GRAD_CHUNK_SPLITS : a.splits;
            for (int sp = c0; sp < c1; ++sp) cs += src[sp * stride + base];
            if (a.chunk_out) a.chunk_out[ch * total + idx] = cs;
            sum += cs;
        }
    }
    a.raw[idx] = sum;
}

struct RegArgs {
    const double *raw;     // [L][P] (all-reduced across ranks)
    const double *params;  // FP64 master records [L][P]
    const double *masks;   // [L][P] or null
    const double *colnorm; // [L][ng] group norms (SGL)
    int K, Z, V, L, lf;
    double inv_n;
    int kind;              // 0 plain, 1 element_l1, 2 sparse_group
    double lam, lam1, lam2;
    double *grads;         // [L][P] out
};

// Column-group norms of [W (.) M | b (.) mb] (loss.cpp:43-59, backward.cpp:175-199):
// groups per layer = IN + 1 (W1) + Z + 1 (W2) + Z + 1 (W3).
__global__ void k_group_norms(const double *params, const double *masks, int K, int Z, int V,
                              int L, int lf, double *colnorm) {
    const int IN = 3 * K + V, P = Z * IN + Z + K * Z + K + V * Z + V + 1;
    const int ng = IN + 1 + 2 * (Z + 1);
    const long g = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= static_cast<long>(L - lf) * ng) return;
    const int l = lf + static_cast<int>(g / ng), j = static_cast<int>(g % ng);
    const double *p = params + static_cast<long>(l) * P;
    const double *mk = masks ? masks + static_cast<long>(l) * P : nullptr;
    const int oW1 = 0, ob1 = Z * IN, oW2 = ob1 + Z, ob2 = oW2 + K * Z, oW3 = ob2 + K, ob3 = oW3 + V * Z;
    int off, rows, cols, col;
    bool bias;
    if (j <= IN) { off = j < IN ? oW1 : ob1; rows = Z; cols = IN; col = j; bias = j == IN; }
    else if (j <= IN + 1 + Z) { const int jj = j - IN - 1; off = jj < Z ? oW2 : ob2; rows = K; cols = Z; col = jj; bias = jj == Z; }
    else { const int jj = j - IN - 2 - Z; off = jj < Z ? oW3 : ob3; rows = V; cols = Z; col = jj; bias = jj == Z; }
    // loads batched 16 rows ahead (the sum itself stays sequential in i, as in
    // loss.cpp:43-59): one dependent L2 round trip per 16 rows instead of per row
    double sq = 0.0;
    const long step = bias ? 1 : cols;
    const long e0 = bias ? off : off + col;
    int i = 0;
    for (; i + 16 <= rows; i += 16) {
        double w[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const long e = e0 + static_cast<long>(i + u) * step;
            w[u] = dmul(__ldg(p + e), mk ? __ldg(mk + e) : 1.0);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) sq = dadd(sq, dmul(w[u], w[u]));
    }
    for (; i < rows; ++i) {
        const long e = e0 + static_cast<long>(i) * step;
        const double w = dmul(p[e], mk ? mk[e] : 1.0);
        sq = dadd(sq, dmul(w, w));
    }
    colnorm[static_cast<long>(l) * ng + j] = sqrt(sq);
}

__device__ __forceinline__ double sign0(double w) { return w > 0.0 ? 1.0 : (w < 0.0 ? -1.0 : 0.0); }

// grads = raw * mask / n + regularizer gradient (backward.cpp:169-220 order:
// group term then L1 term; kernels.cpp:195-198 scaling).
__global__ void k_grad_apply_reg(RegArgs a) {
    const int K = a.K, Z = a.Z, V = a.V, IN = 3 * K + V;
    const int P = Z * IN + Z + K * Z + K + V * Z + V + 1;
    const int ng = IN + 1 + 2 * (Z + 1);
    const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long>(a.L) * P) return;
    const int l = static_cast<int>(idx / P), e = static_cast<int>(idx % P);
    if (l < a.lf) { a.grads[idx] = 0.0; return; }
    const int ob1 = Z * IN, oW2 = ob1 + Z, ob2 = oW2 + K * Z, oW3 = ob2 + K, ob3 = oW3 + V * Z, ot = ob3 + V;
    const double mk = (a.masks && e != ot) ? a.masks[idx] : 1.0;
    double g = dmul(dmul(a.raw[idx], mk), a.inv_n);
    if (e != ot && a.kind != 0) {
        int gcol;
        bool weight;
        if (e < ob1) { gcol = e % IN; weight = true; }
        else if (e < oW2) { gcol = IN; weight = false; }
        else if (e < ob2) { gcol = IN + 1 + (e - oW2) % Z; weight = true; }
        else if (e < oW3) { gcol = IN + 1 + Z; weight = false; }
        else if (e < ob3) { gcol = IN + 2 + Z + (e - oW3) % Z; weight = true; }
        else { gcol = IN + 2 + 2 * Z; weight = false; }
        const double w = a.params[idx];
        if (a.kind == 2) {
            const double nrm = a.colnorm[static_cast<long>(l) * ng + gcol];
            if (nrm > 0.0) g = dadd(g, dmul(dmul(ddiv(a.lam1, nrm), w), mk));
            if (weight) g = dadd(g, dmul(dmul(a.lam2, sign0(w)), mk));
        } else if (weight) {
            g = dadd(g, dmul(dmul(a.lam, sign0(w)), mk));
        }
    }
    a.grads[idx] = g;
}

// adam.cpp:30-79 per entry, FP64 without contraction (bit-identical to the
// reference for identical inputs). Masked entries (mask 0) untouched.
// halt (nullable): the sticky divergence slot of k_objective -- a diverged
// run keeps its parameters (the reference throws before adam_step).
__global__ void k_adam(double *params, const double *masks, const double *grads, double *m,
                       double *v, long count, int P, int lf, double lr, double b1, double b2,
                       double eps, double bc1, double bc2, const long long *halt = nullptr) {
    const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= count) return;
    if (halt && *halt >= 0) return;
    const int l = static_cast<int>(idx / P), e = static_cast<int>(idx % P);
    if (l < lf) return;
    const bool is_t = e == P - 1;
    if (!is_t && masks && masks[idx] == 0.0) return;
    const double g = grads[idx];
    const double mi = dadd(dmul(b1, m[idx]), dmul(dsub(1.0, b1), g));
    const double vi = dadd(dmul(b2, v[idx]), dmul(dmul(dsub(1.0, b2), g), g));
    m[idx] = mi;
    v[idx] = vi;
    const double mhat = ddiv(mi, bc1);
    const double vhat = ddiv(vi, bc2);
    double w = dsub(params[idx], ddiv(dmul(lr, mhat), dadd(__dsqrt_rn(vhat), eps)));
    if (is_t && w < 1e-3) w = 1e-3;
    params[idx] = w;
}

// ---- objective = data_loss + regularizer(params, spec) (training.cpp:67-70) --
// The reference's regularizer() (loss.cpp:81-91) in its operation order:
// group_norm_sum (loss.cpp:43-59) folds the column norms of [W (.) M] -- each
// the square root of a row-order sum, exactly k_group_norms' colnorm values,
// computed here for every layer (frozen ones count in the value) -- in
// column order and adds the bias group's; masked_l1 (loss.cpp:35-41) is a
// sequential sum over W, done only when the spec weighs it. One thread per
// layer folds that layer's terms (k_reg_layers), then one thread folds the
// layers in order (k_objective): bit-identical to the reference.
struct ObjArgs {
    const double *params, *masks;
    const double *colnorm;  // [L][ng] (k_group_norms over all L layers)
    int K, Z, V, L;
    int kind;
    double lam, lam1, lam2;
    double *part;           // [L][4]: groups (g1 + g2) + g3, then e1, e2, e3 (masked_l1 of W1, W2, W3)
};

// One CTA per (layer, part = group sums | masked_l1 of W1 | W2 | W3): the terms are staged in shared memory by the whole
// CTA (coalesced loads, the per-element |w| m products in parallel) and folded by
// thread 0 in the reference's order, one chunk behind the loads -- the same
// dadd chain as a single thread walking global memory (bit-identical value),
// without a dependent L2 round trip per term.
constexpr int REG_THREADS = 256, REG_CHUNK = 2048;

__global__ void __launch_bounds__(REG_THREADS) k_reg_layers(ObjArgs a) {
    __shared__ double buf[2][REG_CHUNK];
    const int K = a.K, Z = a.Z, V = a.V, IN = 3 * K + V;
    const long P = static_cast<long>(Z) * IN + Z + static_cast<long>(K) * Z + K +
                   static_cast<long>(V) * Z + V + 1;
    const int ng = IN + 1 + 2 * (Z + 1);
    const int idx = blockIdx.x;
    if (idx >= 4 * a.L) return;
    const int l = idx >> 2;
    const int tid = threadIdx.x;
    if ((idx & 3) == 0) { // group_norm_sum of W1, W2, W3 (with their bias groups)
        double g[3] = {0.0, 0.0, 0.0};
        if (a.kind == 2) { // block-uniform
            const double *cn = a.colnorm + static_cast<long>(l) * ng;
            const bool fits = ng <= 2 * REG_CHUNK; // else thread 0 walks global memory
            double *stage = &buf[0][0];
            if (fits)
                for (int j = tid; j < ng; j += REG_THREADS) stage[j] = cn[j];
            __syncthreads();
            const double *flat = fits ? stage : cn;
            if (tid == 0) {
                const int cols[3] = {IN, Z, Z};
                int off = 0;
                for (int m = 0; m < 3; ++m) {
                    double acc = 0.0;
                    for (int j = 0; j < cols[m]; ++j) acc = dadd(acc, flat[off + j]);
                    g[m] = dadd(acc, flat[off + cols[m]]);
                    off += cols[m] + 1;
                }
            }
        }
        if (tid == 0) a.part[4 * l] = dadd(dadd(g[0], g[1]), g[2]);
    } else { // masked_l1 of W1, W2 or W3: one CTA (one sequential fold) per matrix
        const int m = (idx & 3) - 1;
        double em = 0.0;
        if (a.kind == 1 || (a.kind == 2 && a.lam2 != 0.0)) { // block-uniform
            const double *p = a.params + static_cast<long>(l) * P;
            const double *mk = a.masks ? a.masks + static_cast<long>(l) * P : nullptr;
            const long oW[3] = {0, static_cast<long>(Z) * IN + Z,
                                static_cast<long>(Z) * IN + Z + static_cast<long>(K) * Z + K};
            const long cnt[3] = {static_cast<long>(Z) * IN, static_cast<long>(K) * Z,
                                 static_cast<long>(V) * Z};
            {
                double acc = 0.0;
                const long nch = (cnt[m] + REG_CHUNK - 1) / REG_CHUNK;
                for (long c = 0; c <= nch; ++c) {
                    if (c < nch) { // stage chunk c (every thread; thread 0 first, then it folds)
                        double *dst = buf[c & 1];
                        const long q0 = c * REG_CHUNK;
                        const long qn = cnt[m] - q0 < REG_CHUNK ? cnt[m] - q0 : REG_CHUNK;
                        for (long q = tid; q < qn; q += REG_THREADS) {
                            const long ee = oW[m] + q0 + q;
                            dst[q] = dmul(fabs(p[ee]), mk ? mk[ee] : 1.0);
                        }
                    }
                    if (c > 0 && tid == 0) { // fold chunk c - 1 in element order
                        const double *src = buf[(c - 1) & 1];
                        const long q0 = (c - 1) * REG_CHUNK;
                        const long qn = cnt[m] - q0 < REG_CHUNK ? cnt[m] - q0 : REG_CHUNK;
                        for (long q = 0; q < qn; ++q) acc = dadd(acc, src[q]);
                    }
                    __syncthreads();
                }
                em = acc;
            }
        }
        if (tid == 0) a.part[4 * l + 1 + m] = em;
    }
}

// status: [0] objective, [1] regularizer, [2] diverged step (-1 = none; sticky)
__global__ void k_objective(ObjArgs a, const double *loss_sum, double n_global, long long step,
                            double *status) {
    double reg = 0.0;
    if (a.kind == 1) {
        double acc = 0.0;
        for (int l = 0; l < a.L; ++l)
            acc = dadd(acc, dadd(dadd(a.part[4 * l + 1], a.part[4 * l + 2]), a.part[4 * l + 3]));
        reg = dmul(a.lam, acc);
    } else if (a.kind == 2) {
        double groups = 0.0, elems = 0.0;
        for (int l = 0; l < a.L; ++l) {
            groups = dadd(groups, a.part[4 * l]);
            elems = dadd(elems, dadd(dadd(a.part[4 * l + 1], a.part[4 * l + 2]), a.part[4 * l + 3]));
        }
        reg = dadd(dmul(a.lam1, groups), dmul(a.lam2, elems));
    }
    const double obj = dadd(ddiv(*loss_sum, n_global), reg);
    status[0] = obj;
    status[1] = reg;
    long long *halt = reinterpret_cast<long long *>(status + 2);
    if (*halt < 0 && !isfinite(obj)) *halt = step;
}

// FP64 records -> SIMT FP32 records (same mapping as the host packer).
__global__ void k_pack_simt(const double *params, const double *masks, int K, int Z, int V, int L,
                            float *out) {
    const int IN = 3 * K + V, IN4 = simt_in4(K, V), O4 = simt_o4(K, V);
    const long R = simt_rec(K, Z, V);
    const int P = Z * IN + Z + K * Z + K + V * Z + V + 1;
    const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long>(L) * R) return;
    const int l = static_cast<int>(idx / R);
    const long r = idx % R;
    const double *p = params + static_cast<long>(l) * P;
    const double *mk = masks ? masks + static_cast<long>(l) * P : nullptr;
    auto w = [&](long off) { return static_cast<float>(p[off] * (mk ? mk[off] : 1.0)); };
    const int oW1 = 0, ob1 = Z * IN, oW2 = ob1 + Z, ob2 = oW2 + K * Z, oW3 = ob2 + K, ob3 = oW3 + V * Z, ot = ob3 + V;
    float val = 0.f;
    if (r < static_cast<long>(Z) * IN4) {
        const int i = static_cast<int>(r / IN4), j = static_cast<int>(r % IN4);
        val = j < IN ? w(oW1 + i * IN + j) : (j == IN ? w(ob1 + i) : 0.f);
    } else if (r < static_cast<long>(Z) * IN4 + static_cast<long>(Z) * O4) {
        const long rr = r - static_cast<long>(Z) * IN4;
        const int i = static_cast<int>(rr / O4), k = static_cast<int>(rr % O4);
        val = k < K ? w(oW2 + k * Z + i) : (k < K + V ? w(oW3 + (k - K) * Z + i) : 0.f);
    } else {
        const int k = static_cast<int>(r - static_cast<long>(Z) * IN4 - static_cast<long>(Z) * O4);
        val = k < K ? w(ob2 + k) : (k < K + V ? w(ob3 + (k - K)) : (k == O4 ? static_cast<float>(p[ot]) : 0.f));
    }
    out[idx] = val;
}

} // namespace detnet
