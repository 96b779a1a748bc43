// k_stack_simt.cuh -- K2-SIMT: the fused DetNet layer stack on FP32 CUDA
// cores, one thread per sample, all L layers in one launch.
//
// Restates forward_pre (model.cpp:84-122) + loss_plain (loss.cpp:9-31) + the
// hard-decision error count (kernels.cpp:63-65). Per layer and sample:
//   gx = G x_hat                      (G packed, FP32 from K1, read via L2)
//   u1 = W1 [q; x_hat; gx; v] + b1    (bias folded as input column IN)
//   z  = relu(u1);  [u2; v'] = [W2; W3] z + [b2; b3]
//   x_hat' = psi_t(u2)                (model.cpp:32-41)
//   loss += ln(l+1) * ||x - x_hat'||^2 / denom   (FP64)
// Each layer's weights (W (.) M, FP32, ~105 KB at K=20) are staged into
// shared memory by the bulk-copy engine (cp.async.bulk + mbarrier), double
// buffered so layer l+1 lands while layer l computes; every thread reads
// them as warp-uniform float4 broadcasts. This path is the correctness
// baseline and serves dims the tcgen05 kernel does not cover.
#pragma once

#include "common.cuh"

namespace detnet {

struct SimtDims {
    int K, Z, V;
};

// Packed per-layer record for the SIMT kernel (floats):
//   W1x  [Z][IN4]   row i = W1[i][0..IN) * M1, b1[i]*mb1[i], 0 pad
//   W23T [Z][O4]    row i = (W2[.][i] * M2, W3[.][i] * M3, 0 pad)
//   b23  [O4]       (b2 * mb2, b3 * mb3, 0 pad)
//   tail [4]        (t, 0, 0, 0)
__host__ __device__ constexpr int simt_in4(int K, int V) { return round_up(3 * K + V + 1, 4); }
__host__ __device__ constexpr int simt_o4(int K, int V) { return round_up(K + V, 4); }
__host__ __device__ constexpr long simt_rec(int K, int Z, int V) {
    return static_cast<long>(Z) * simt_in4(K, V) + static_cast<long>(Z) * simt_o4(K, V) +
           simt_o4(K, V) + 4;
}

struct StackArgs {
    const float *gp;        // [tile][NG][TILE]
    const float *q32;       // [tile][K][TILE]
    const double *denom;    // [s]
    const uint32_t *xmask;  // [s]
    const float *wrec;      // [depth][rec]
    long rec_floats;
    const double *lnk;      // [depth] ln(l+1) or 0 when excluded
    int l_begin, l_end;
    long n, n_tiles, tile0; // tile0: global index of this launch's first tile
    float *xhat;            // optional [s][l_end-l_begin][K] (s relative to this launch)
    float *x_state;         // optional [s][K] in/out
    float *v_state;         // optional [s][V] in/out
    double *tile_loss;      // [global tile][4 lane quadrants]
    long long *tile_err;    // [global tile][4 lane quadrants]
    // optional training trace (backward.cpp:105-165 needs in, u1 (via z), z,
    // u2 per layer), feature-major / sample-minor: [l][feature][ts]
    float *tr_in;           // [L][IN][ts]   layer input [q; x; Gx; v]
    float *tr_z;            // [L][Z][ts]    relu(u1)
    float *tr_u2;           // [L][K][ts]
    float *tr_xf;           // [K][ts]       x_hat_L
    long ts;                // trace sample stride (>= padded sample count)
};

// THREADS samples per CTA (one CTA per SM fits: the double-buffered weights
// take ~210 KB of shared memory). 256 (two tiles) for large batches; 64 (half
// a tile) for small ones -- the training batch of 5,000 is 40 tiles -- so they
// still spread over 79 SMs.
template <int K, int Z, int V, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_stack_simt(StackArgs a) {
    constexpr int SIMT_THREADS = THREADS;
    constexpr int IN = 3 * K + V;
    constexpr int IN4 = simt_in4(K, V);
    constexpr int O = K + V;
    constexpr int O4 = simt_o4(K, V);
    constexpr int NG = gram_entries(K);
    constexpr int REC = static_cast<int>(simt_rec(K, Z, V));
    extern __shared__ __align__(128) float sw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sw + 2 * REC);

    const int tid = threadIdx.x;
    // blocks cover tiles in units of THREADS consecutive samples
    const long unit = static_cast<long>(blockIdx.x) * SIMT_THREADS + tid;
    const long tile_l = unit / TILE;
    const bool live_tile = tile_l < a.n_tiles;
    const long tile = live_tile ? tile_l : a.n_tiles - 1;
    const int col = static_cast<int>(unit % TILE);
    const long s = tile * TILE + col;           // sample index within this launch
    DETNET_DASSERT(tile >= 0 && tile < a.n_tiles);
    const bool live = live_tile && s < a.n;
    const long gt = a.tile0 + tile;              // global tile index for SoA buffers

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t bytes = static_cast<uint32_t>(REC) * 4u;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            const int l = a.l_begin + b;
            if (l < a.l_end) {
                mbar_arrive_expect_tx(&bars[b], bytes);
                bulk_g2s_chunked(sw + b * REC, a.wrec + static_cast<long>(l) * a.rec_floats, bytes,
                                 &bars[b]);
            }
        }
    }

    float q[K], x[K], v[V];
#pragma unroll
    for (int k = 0; k < K; ++k) q[k] = a.q32[(gt * K + k) * TILE + col];
    if (a.x_state && live) {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = a.x_state[s * K + k];
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = a.v_state[s * V + k];
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = 0.f;
    }
    const uint32_t xm = a.xmask[gt * TILE + col];
    const double dnm = a.denom[gt * TILE + col];
    double loss = 0.0;
    const int nl = a.l_end - a.l_begin;
    const float *gps = a.gp + gt * NG * TILE + col;

    for (int l = a.l_begin; l < a.l_end; ++l) {
        const int it = l - a.l_begin;
        const int b = it & 1;
        mbar_wait(&bars[b], (it >> 1) & 1);
        const float *W = sw + b * REC;

        float gx[K];
#pragma unroll
        for (int k = 0; k < K; ++k) gx[k] = 0.f;
        {
            int e = 0;
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int c = r; c < K; ++c, ++e) {
                    const float g = __ldg(gps + e * TILE);
                    gx[r] = fmaf(g, x[c], gx[r]);
                    if (c != r) gx[c] = fmaf(g, x[r], gx[c]);
                }
        }

        if (a.tr_in && live_tile) {
            float *ti = a.tr_in + static_cast<long>(l) * IN * a.ts + s;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                ti[k * a.ts] = q[k];
                ti[(K + k) * a.ts] = x[k];
                ti[(2 * K + k) * a.ts] = gx[k];
            }
#pragma unroll
            for (int k = 0; k < V; ++k) ti[(3 * K + k) * a.ts] = v[k];
        }
        float acc[O];
        const float *b23 = W + Z * IN4 + Z * O4;
#pragma unroll
        for (int o = 0; o < O; ++o) acc[o] = b23[o];

#define DETNET_IN(j)                                                                            \
    ((j) < K ? q[(j) < K ? (j) : 0]                                                             \
             : (j) < 2 * K ? x[((j) - K) < K ? (j) - K : 0]                                      \
                           : (j) < 3 * K ? gx[((j) - 2 * K) < K ? (j) - 2 * K : 0]               \
                                         : v[((j) - 3 * K) < V ? (j) - 3 * K : 0])
#pragma unroll 1
        for (int i = 0; i < Z; ++i) {
            const float4 *w4 = reinterpret_cast<const float4 *>(W + i * IN4);
            float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;
#pragma unroll
            for (int m = 0; m < IN4 / 4; ++m) {
                const float4 w = w4[m];
                if (4 * m + 0 < IN) u0 = fmaf(w.x, DETNET_IN(4 * m + 0), u0);
                else if (4 * m + 0 == IN) u0 += w.x;
                if (4 * m + 1 < IN) u1 = fmaf(w.y, DETNET_IN(4 * m + 1), u1);
                else if (4 * m + 1 == IN) u1 += w.y;
                if (4 * m + 2 < IN) u2 = fmaf(w.z, DETNET_IN(4 * m + 2), u2);
                else if (4 * m + 2 == IN) u2 += w.z;
                if (4 * m + 3 < IN) u3 = fmaf(w.w, DETNET_IN(4 * m + 3), u3);
                else if (4 * m + 3 == IN) u3 += w.w;
            }
            const float u = (u0 + u1) + (u2 + u3);
            const float z = u > 0.f ? u : 0.f;
            if (a.tr_z && live_tile) a.tr_z[(static_cast<long>(l) * Z + i) * a.ts + s] = z;
            const float4 *c4 = reinterpret_cast<const float4 *>(W + Z * IN4 + i * O4);
#pragma unroll
            for (int m = 0; m < O4 / 4; ++m) {
                const float4 w = c4[m];
                if (4 * m + 0 < O) acc[4 * m + 0] = fmaf(w.x, z, acc[4 * m + 0]);
                if (4 * m + 1 < O) acc[4 * m + 1] = fmaf(w.y, z, acc[4 * m + 1]);
                if (4 * m + 2 < O) acc[4 * m + 2] = fmaf(w.z, z, acc[4 * m + 2]);
                if (4 * m + 3 < O) acc[4 * m + 3] = fmaf(w.w, z, acc[4 * m + 3]);
            }
        }
#undef DETNET_IN
        const float t = W[Z * IN4 + Z * O4 + O4];
        double err = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float u = acc[k];
            if (a.tr_u2 && live_tile) a.tr_u2[(static_cast<long>(l) * K + k) * a.ts + s] = u;
            const float xn = u <= -t ? -1.f : (u >= t ? 1.f : __fdiv_rn(u, t));
            x[k] = xn;
            const double d = ((xm >> k) & 1u ? 1.0 : -1.0) - static_cast<double>(xn);
            err += d * d;
        }
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = acc[K + k];
        loss += a.lnk[l] * err / dnm;
        if (a.xhat && live) {
            float *o = a.xhat + (s * nl + it) * K;
#pragma unroll
            for (int k = 0; k < K; ++k) o[k] = x[k];
        }
        __syncthreads();  // every thread is done reading buffer b
        if (tid == 0 && l + 2 < a.l_end) {
            mbar_arrive_expect_tx(&bars[b], bytes);
            bulk_g2s_chunked(sw + b * REC, a.wrec + static_cast<long>(l + 2) * a.rec_floats, bytes,
                             &bars[b]);
        }
    }

    if (a.x_state && live) {
#pragma unroll
        for (int k = 0; k < K; ++k) a.x_state[s * K + k] = x[k];
#pragma unroll
        for (int k = 0; k < V; ++k) a.v_state[s * V + k] = v[k];
    }
    if (a.tr_xf && live_tile) {
#pragma unroll
        for (int k = 0; k < K; ++k) a.tr_xf[k * a.ts + s] = x[k];
    }
    long long errs = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) errs += (x[k] >= 0.f) != (((xm >> k) & 1u) != 0);
    if (!live) { loss = 0.0; errs = 0; }

    // per lane-quadrant partials (a warp = one quadrant), summed in fixed order later
    loss = warp_sum(loss);
    errs = warp_sum(errs);
    if ((tid & 31) == 0 && live_tile) {
        a.tile_loss[gt * 4 + col / 32] = loss;
        a.tile_err[gt * 4 + col / 32] = errs;
    }
}

// Small-batch variant: two threads per sample. Warps 0-1 ("A") take hidden
// units [0, Z/2), warps 2-3 ("B") units [Z/2, Z) of the same 64 samples. Each
// forms its units' u1 / z and a partial [u2; v'] over them; B's partial meets
// A's in shared memory, A applies psi_t, the loss and the outputs and hands
// x_hat, v back. Weights stay double-buffered (the exchange is 15 KB).
constexpr int SIMTP_SAMPLES = 64, SIMTP_THREADS = 128;

template <int K, int Z, int V>
__global__ void __launch_bounds__(SIMTP_THREADS, 1) k_stack_simt_pair(StackArgs a) {
    constexpr int IN = 3 * K + V;
    constexpr int IN4 = simt_in4(K, V);
    constexpr int O = K + V;
    constexpr int O4 = simt_o4(K, V);
    constexpr int NG = gram_entries(K);
    constexpr int REC = static_cast<int>(simt_rec(K, Z, V));
    constexpr int ZH = Z / 2, P = SIMTP_SAMPLES;
    static_assert(Z % 2 == 0, "hidden units split in halves");
    extern __shared__ __align__(128) float sw[];
    float(*sX)[P] = reinterpret_cast<float(*)[P]>(sw + 2 * REC); // [O][P] exchange
    uint64_t *bars = reinterpret_cast<uint64_t *>(sw + 2 * REC + O * P);

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
    const long gt = a.tile0 + tile;
    const int i0 = isA ? 0 : ZH;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t bytes = static_cast<uint32_t>(REC) * 4u;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            const int l = a.l_begin + b;
            if (l < a.l_end) {
                mbar_arrive_expect_tx(&bars[b], bytes);
                bulk_g2s_chunked(sw + b * REC, a.wrec + static_cast<long>(l) * a.rec_floats, bytes,
                                 &bars[b]);
            }
        }
    }

    float q[K], x[K], v[V];
#pragma unroll
    for (int k = 0; k < K; ++k) q[k] = a.q32[(gt * K + k) * TILE + col];
    if (a.x_state && live) {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = a.x_state[s * K + k];
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = a.v_state[s * V + k];
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = 0.f;
    }
    const uint32_t xm = a.xmask[gt * TILE + col];
    const double dnm = a.denom[gt * TILE + col];
    double loss = 0.0;
    const int nl = a.l_end - a.l_begin;
    const float *gps = a.gp + gt * NG * TILE + col;

    for (int l = a.l_begin; l < a.l_end; ++l) {
        const int it = l - a.l_begin;
        const int b = it & 1;
        mbar_wait(&bars[b], (it >> 1) & 1);
        const float *W = sw + b * REC;

        float gx[K];
#pragma unroll
        for (int k = 0; k < K; ++k) gx[k] = 0.f;
        {
            int e = 0;
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int c = r; c < K; ++c, ++e) {
                    const float g = __ldg(gps + e * TILE);
                    gx[r] = fmaf(g, x[c], gx[r]);
                    if (c != r) gx[c] = fmaf(g, x[r], gx[c]);
                }
        }
        if (isA && a.tr_in && live_tile) {
            float *ti = a.tr_in + static_cast<long>(l) * IN * a.ts + s;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                ti[k * a.ts] = q[k];
                ti[(K + k) * a.ts] = x[k];
                ti[(2 * K + k) * a.ts] = gx[k];
            }
#pragma unroll
            for (int k = 0; k < V; ++k) ti[(3 * K + k) * a.ts] = v[k];
        }
        float acc[O];
        const float *b23 = W + Z * IN4 + Z * O4;
#pragma unroll
        for (int o = 0; o < O; ++o) acc[o] = isA ? b23[o] : 0.f;

#define DETNET_IN(j)                                                                            \
    ((j) < K ? q[(j) < K ? (j) : 0]                                                             \
             : (j) < 2 * K ? x[((j) - K) < K ? (j) - K : 0]                                      \
                           : (j) < 3 * K ? gx[((j) - 2 * K) < K ? (j) - 2 * K : 0]               \
                                         : v[((j) - 3 * K) < V ? (j) - 3 * K : 0])
        // Same FMA chains per unit as before (u0..u3 over the input columns,
        // acc[o] over the units), issued as FFMA2 pairs: bit-identical.
        // (two units in flight: their chains interleave; still per-unit order)
#pragma unroll 2
        for (int i = i0; i < i0 + ZH; ++i) {
            const float4 *w4 = reinterpret_cast<const float4 *>(W + i * IN4);
            float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;
#pragma unroll
            for (int m = 0; m < IN4 / 4; ++m) {
                const float4 w = w4[m];
                if (4 * m + 3 < IN) {
                    fma_x2(u0, u1, w.x, w.y, DETNET_IN(4 * m + 0), DETNET_IN(4 * m + 1));
                    fma_x2(u2, u3, w.z, w.w, DETNET_IN(4 * m + 2), DETNET_IN(4 * m + 3));
                } else {
                    if (4 * m + 0 < IN) u0 = fmaf(w.x, DETNET_IN(4 * m + 0), u0);
                    else if (4 * m + 0 == IN) u0 += w.x;
                    if (4 * m + 1 < IN) u1 = fmaf(w.y, DETNET_IN(4 * m + 1), u1);
                    else if (4 * m + 1 == IN) u1 += w.y;
                    if (4 * m + 2 < IN) u2 = fmaf(w.z, DETNET_IN(4 * m + 2), u2);
                    else if (4 * m + 2 == IN) u2 += w.z;
                    if (4 * m + 3 < IN) u3 = fmaf(w.w, DETNET_IN(4 * m + 3), u3);
                    else if (4 * m + 3 == IN) u3 += w.w;
                }
            }
            const float u = (u0 + u1) + (u2 + u3);
            const float z = u > 0.f ? u : 0.f;
            if (a.tr_z && live_tile) a.tr_z[(static_cast<long>(l) * Z + i) * a.ts + s] = z;
            const float4 *c4 = reinterpret_cast<const float4 *>(W + Z * IN4 + i * O4);
#pragma unroll
            for (int m = 0; m < O4 / 4; ++m) {
                const float4 w = c4[m];
                if (4 * m + 3 < O) {
                    fma_x2(acc[4 * m + 0], acc[4 * m + 1], w.x, w.y, z, z);
                    fma_x2(acc[4 * m + 2], acc[4 * m + 3], w.z, w.w, z, z);
                } else {
                    if (4 * m + 0 < O) acc[4 * m + 0] = fmaf(w.x, z, acc[4 * m + 0]);
                    if (4 * m + 1 < O) acc[4 * m + 1] = fmaf(w.y, z, acc[4 * m + 1]);
                    if (4 * m + 2 < O) acc[4 * m + 2] = fmaf(w.z, z, acc[4 * m + 2]);
                    if (4 * m + 3 < O) acc[4 * m + 3] = fmaf(w.w, z, acc[4 * m + 3]);
                }
            }
        }
#undef DETNET_IN
        const float t = W[Z * IN4 + Z * O4 + O4];
        __syncthreads(); // every weight read of buffer b is done
        if (tid == 0 && l + 2 < a.l_end) {
            mbar_arrive_expect_tx(&bars[b], bytes);
            bulk_g2s_chunked(sw + b * REC, a.wrec + static_cast<long>(l + 2) * a.rec_floats, bytes,
                             &bars[b]);
        }
        if (!isA) {
#pragma unroll
            for (int o = 0; o < O; ++o) sX[o][ls] = acc[o];
        }
        named_bar_sync(pbar, 64);
        if (isA) {
#pragma unroll
            for (int o = 0; o < O; ++o) acc[o] += sX[o][ls];
            double err = 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float u = acc[k];
                if (a.tr_u2 && live_tile) a.tr_u2[(static_cast<long>(l) * K + k) * a.ts + s] = u;
                const float xn = u <= -t ? -1.f : (u >= t ? 1.f : __fdiv_rn(u, t));
                x[k] = xn;
                const double d = ((xm >> k) & 1u ? 1.0 : -1.0) - static_cast<double>(xn);
                err += d * d;
            }
#pragma unroll
            for (int k = 0; k < V; ++k) v[k] = acc[K + k];
            loss += a.lnk[l] * err / dnm;
            if (a.xhat && live) {
                float *o = a.xhat + (s * nl + it) * K;
#pragma unroll
                for (int k = 0; k < K; ++k) o[k] = x[k];
            }
#pragma unroll
            for (int k = 0; k < K; ++k) sX[k][ls] = x[k];
#pragma unroll
            for (int k = 0; k < V; ++k) sX[K + k][ls] = v[k];
        }
        named_bar_sync(pbar, 64);
        if (!isA) {
#pragma unroll
            for (int k = 0; k < K; ++k) x[k] = sX[k][ls];
#pragma unroll
            for (int k = 0; k < V; ++k) v[k] = sX[K + k][ls];
        }
        named_bar_sync(pbar, 64); // B has read before A overwrites next layer
    }

    if (!isA) return;
    if (a.x_state && live) {
#pragma unroll
        for (int k = 0; k < K; ++k) a.x_state[s * K + k] = x[k];
#pragma unroll
        for (int k = 0; k < V; ++k) a.v_state[s * V + k] = v[k];
    }
    if (a.tr_xf && live_tile) {
#pragma unroll
        for (int k = 0; k < K; ++k) a.tr_xf[k * a.ts + s] = x[k];
    }
    long long errs = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) errs += (x[k] >= 0.f) != (((xm >> k) & 1u) != 0);
    if (!live) { loss = 0.0; errs = 0; }
    loss = warp_sum(loss);
    errs = warp_sum(errs);
    if ((tid & 31) == 0 && live_tile) {
        a.tile_loss[gt * 4 + col / 32] = loss;
        a.tile_err[gt * 4 + col / 32] = errs;
    }
}

// K5: fixed-order reduction of per-tile partials and per-sample flags.
// finish_eval (kernels.cpp:93-103) on the device, in a canonical order that
// does not depend on how the samples were split into launches or devices:
// each chunk of RED_CHUNK_TILES consecutive tiles (8,192 samples) folds its
// tiles' loss partials ((q0 + q1) + (q2 + q3) per tile) in tile order, and
// the chunk sums are folded in chunk order. A device group whose shards
// start at chunk boundaries reproduces the single-device sum exactly from the
// members' chunk sums (chunk_out). Counts are integers (exact in any order).
constexpr int RED_CHUNK_TILES = 64;
static __global__ void __launch_bounds__(1024) k_reduce(const double *tile_loss, const long long *tile_err,
                                                 long n_quads, const uint8_t *flag, long n,
                                                 double *out_loss, long long *out_err,
                                                 long long *out_flag, double *chunk_out) {
    __shared__ long long se[1024], sf[1024];
    const int t = threadIdx.x;
    const long tiles = n_quads / 4;
    const long chunks = (tiles + RED_CHUNK_TILES - 1) / RED_CHUNK_TILES;
    DETNET_DASSERT(n_quads % 4 == 0 && n <= tiles * TILE);
    long long e = 0, f = 0;
    for (long i = t; i < n_quads; i += 1024) e += tile_err[i];
    for (long c = t; c < chunks; c += 1024) {
        double acc = 0.0;
        const long t1 = (c + 1) * RED_CHUNK_TILES < tiles ? (c + 1) * RED_CHUNK_TILES : tiles;
        for (long tt = c * RED_CHUNK_TILES; tt < t1; ++tt) {
            const double *q = tile_loss + tt * 4;
            acc += (q[0] + q[1]) + (q[2] + q[3]);
        }
        chunk_out[c] = acc;
    }
    // flags are 0/1 bytes: 16 per 128-bit load, summed with popc
    long i0 = 0;
    if ((reinterpret_cast<uintptr_t>(flag) & 15) == 0) {
        const uint4 *f16 = reinterpret_cast<const uint4 *>(flag);
        const long n16 = n / 16;
        for (long i = t; i < n16; i += 1024) {
            const uint4 v = __ldg(f16 + i);
            f += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        }
        i0 = n16 * 16;
    }
    for (long i = i0 + t; i < n; i += 1024) f += flag[i];
    se[t] = e; sf[t] = f;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if (t < w) { se[t] += se[t + w]; sf[t] += sf[t + w]; }
        __syncthreads();
    }
    if (t == 0) {
        double l = 0.0;
        for (long c = 0; c < chunks; ++c) l += chunk_out[c];
        *out_loss = l;
        *out_err = se[0];
        *out_flag = sf[0];
    }
}

} // namespace detnet
