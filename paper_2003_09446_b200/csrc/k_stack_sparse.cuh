// k_stack_sparse.cuh -- K4: the DetNet layer stack for sparse-group-pruned
// models (BASELINE config 4): the masked branch of masked_affine
// (model.cpp:69-78) without the zeros.
//
// Per layer only "alive" hidden units are visited -- units with at least one
// surviving outgoing weight in [W2; W3] (a unit with none cannot influence
// anything; model.cpp:114-118). For each alive unit the kernel walks its
// surviving W1 entries (CSR row: (input column, weight)) and, when
// relu(u1) > 0, scatters z into the U2V accumulators along its surviving
// [W2; W3] column entries. Entries are read as warp-uniform broadcasts (all
// samples share the weights) from L1; the per-sample vectors live in shared
// memory, feature-major / sample-minor, so the data-dependent gathers and
// scatters are bank-conflict free. Two threads per sample (warps w and w+4):
// each holds half of the packed Gram matrix in registers (G x_hat without L2
// traffic) and walks half of the alive units (balanced by entry count).
#pragma once

#include "common.cuh"

namespace detnet {

// Sparse layer stream (int32 words), per layer at word offset lay_off[l]:
//   [0] nu  [1] split  [2] unused [3] unused
//   unit table nu x 4: in_begin, in_end, out_begin, out_end (entry indices)
//   b1[nu] (float bits)
//   in entries  (col, w bits) pairs
//   out entries (row, w bits) pairs; row < V -> v (b3 order), else u2[row - V]
//   b23[64] (float bits: b3[0..V) then b2[0..K)), t, 1/t
struct SparseArgs {
    const float *gp;
    const float *q32;
    const double *denom;
    const uint32_t *xmask;
    const int *stream;      // all layers
    const long *lay_off;    // [L + 1] word offsets (16-byte aligned), last = total
    int max_words;          // largest layer stream (shared-memory staging slot)
    const double *lnk;
    int L;
    long n, n_tiles, tile0;
    float *xhat;
    double *tile_loss;
    long long *tile_err;
};

template <int K, int V>
__global__ void __launch_bounds__(256, 1) k_stack_sparse(SparseArgs a) {
    constexpr int IN = 3 * K + V;
    constexpr int O = K + V;
    constexpr int NG = gram_entries(K);
    constexpr int R0 = 6;                                 // rows 0..5 on half 0 (K = 20: 105 + 105)
    constexpr int NA = R0 * K - R0 * (R0 - 1) / 2;
    constexpr int NB = NG - NA;
    constexpr int NMAX = NA > NB ? NA : NB;
    extern __shared__ __align__(16) float smx[];
    float(*sin)[TILE] = reinterpret_cast<float(*)[TILE]>(smx);                  // [IN][TILE]
    float(*acc)[O][TILE] = reinterpret_cast<float(*)[O][TILE]>(smx + IN * TILE); // [2][O][TILE]
    float(*gxp)[TILE] = reinterpret_cast<float(*)[TILE]>(smx + IN * TILE + 2 * O * TILE); // [K][TILE]
    // layer streams staged in shared memory (double-buffered bulk copies), so the
    // warp-uniform entry reads are shared-memory broadcasts instead of L1/L2 trips
    int *stage = reinterpret_cast<int *>(smx + IN * TILE + 2 * O * TILE + K * TILE);
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage + 2 * a.max_words);
    __shared__ double s_loss[4];
    __shared__ long long s_err[4];

    const int tid = threadIdx.x;
    const int half = tid >> 7, col = tid & (TILE - 1);
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const long my_tiles = a.n_tiles > blockIdx.x ? (a.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long total_it = my_tiles * a.L;
    auto load_layer = [&](long itn) { // iteration itn -> layer itn % L into slot itn & 1
        const int l = static_cast<int>(itn % a.L);
        const uint32_t bytes = static_cast<uint32_t>(a.lay_off[l + 1] - a.lay_off[l]) * 4u;
        mbar_arrive_expect_tx(&bars[itn & 1], bytes);
        bulk_g2s_chunked(stage + (itn & 1) * a.max_words, a.stream + a.lay_off[l], bytes,
                         &bars[itn & 1]);
    };
    if (tid == 0) {
        for (long itn = 0; itn < 2 && itn < total_it; ++itn) load_layer(itn);
    }
    long it = 0;
    for (long tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const long gt = a.tile0 + tile;
        const long s = tile * TILE + col;
        const bool live = s < a.n;
        float g[NMAX];
        const float *gps = a.gp + gt * NG * TILE + col;
#pragma unroll
        for (int e = 0; e < NMAX; ++e)
            g[e] = (half == 0 || e < NB) ? __ldg(gps + (half == 0 ? e : NA + e) * TILE) : 0.f;
        // state: q, x = 0, v = 0 in sin
        if (half == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                sin[k][col] = a.q32[(gt * K + k) * TILE + col];
                sin[K + k][col] = 0.f;
            }
        } else {
#pragma unroll
            for (int k = 0; k < V; ++k) sin[3 * K + k][col] = 0.f;
        }
        const uint32_t xm = a.xmask[gt * TILE + col];
        double wsum = 0.0;
        __syncthreads();
        for (int l = 0; l < a.L; ++l, ++it) {
            mbar_wait(&bars[it & 1], static_cast<uint32_t>((it >> 1) & 1));
            const int *ls = stage + (it & 1) * a.max_words;
            // ---- G x_hat: half 0 rows 0..R0-1, half 1 rows R0..K-1 ----
            float x[K], gx[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { x[k] = sin[K + k][col]; gx[k] = 0.f; }
            {
                int e = 0;
                if (half == 0) {
#pragma unroll
                    for (int r = 0; r < R0; ++r)
#pragma unroll
                        for (int c = r; c < K; ++c, ++e) {
                            gx[r] = fmaf(g[e], x[c], gx[r]);
                            if (c != r) gx[c] = fmaf(g[e], x[r], gx[c]);
                        }
                } else {
#pragma unroll
                    for (int r = R0; r < K; ++r)
#pragma unroll
                        for (int c = r; c < K; ++c, ++e) {
                            gx[r] = fmaf(g[e], x[c], gx[r]);
                            if (c != r) gx[c] = fmaf(g[e], x[r], gx[c]);
                        }
                }
            }
            if (half == 1) {
#pragma unroll
                for (int k = 0; k < K; ++k) gxp[k][col] = gx[k];
            }
            // zero both accumulator halves
#pragma unroll
            for (int o = 0; o < O; ++o) acc[half][o][col] = 0.f;
            __syncthreads();
            if (half == 0) {
#pragma unroll
                for (int k = 0; k < K; ++k) sin[2 * K + k][col] = gx[k] + gxp[k][col];
            }
            __syncthreads();
            // ---- alive units of this half ----
            const int nu = ls[0], split = ls[1];
            const int4 *units = reinterpret_cast<const int4 *>(ls + 4);
            const float *b1 = reinterpret_cast<const float *>(ls + 4 + 4 * nu);
            const int2 *ent = reinterpret_cast<const int2 *>(ls + 4 + 5 * nu + ((4 + 5 * nu) & 1));
            const int u0 = half == 0 ? 0 : split, u1 = half == 0 ? split : nu;
            for (int u = u0; u < u1; ++u) {
                const int4 un = units[u];
                float p0 = b1[u], p1 = 0.f, p2 = 0.f, p3 = 0.f;
                int e = un.x;
                // 4 independent gathers in flight per step (entries of a row are distinct)
                for (; e + 4 <= un.y; e += 4) {
                    const int2 c0 = ent[e], c1 = ent[e + 1], c2 = ent[e + 2], c3 = ent[e + 3];
                    p0 = fmaf(__int_as_float(c0.y), sin[c0.x][col], p0);
                    p1 = fmaf(__int_as_float(c1.y), sin[c1.x][col], p1);
                    p2 = fmaf(__int_as_float(c2.y), sin[c2.x][col], p2);
                    p3 = fmaf(__int_as_float(c3.y), sin[c3.x][col], p3);
                }
                for (; e < un.y; ++e) {
                    const int2 c = ent[e];
                    p0 = fmaf(__int_as_float(c.y), sin[c.x][col], p0);
                }
                const float uu = (p0 + p1) + (p2 + p3);
                if (uu > 0.f) {
                    // scatter: the rows of one unit's column are distinct, so the
                    // read-modify-writes of a group of 4 are independent
                    e = un.z;
                    for (; e + 4 <= un.w; e += 4) {
                        const int2 c0 = ent[e], c1 = ent[e + 1], c2 = ent[e + 2], c3 = ent[e + 3];
                        const float a0 = acc[half][c0.x][col], a1 = acc[half][c1.x][col],
                                    a2 = acc[half][c2.x][col], a3 = acc[half][c3.x][col];
                        acc[half][c0.x][col] = fmaf(__int_as_float(c0.y), uu, a0);
                        acc[half][c1.x][col] = fmaf(__int_as_float(c1.y), uu, a1);
                        acc[half][c2.x][col] = fmaf(__int_as_float(c2.y), uu, a2);
                        acc[half][c3.x][col] = fmaf(__int_as_float(c3.y), uu, a3);
                    }
                    for (; e < un.w; ++e) {
                        const int2 c = ent[e];
                        acc[half][c.x][col] = fmaf(__int_as_float(c.y), uu, acc[half][c.x][col]);
                    }
                }
            }
            __syncthreads();
            // ---- outputs: v (rows 0..V-1) -> half 1, u2 (rows V..) -> psi_t on half 0 ----
            const int tail = ls[2];
            const float *b23 = reinterpret_cast<const float *>(ls + tail);
            if (half == 1) {
#pragma unroll
                for (int k = 0; k < V; ++k)
                    sin[3 * K + k][col] = b23[k] + acc[0][k][col] + acc[1][k][col];
            } else {
                const float t = b23[64], tinv = b23[65];
                float err = 0.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float uu = b23[V + k] + acc[0][V + k][col] + acc[1][V + k][col];
                    const float xn = uu <= -t ? -1.f : (uu >= t ? 1.f : uu * tinv);
                    sin[K + k][col] = xn;
                    const float d = ((xm >> k) & 1u ? 1.f : -1.f) - xn;
                    err = fmaf(d, d, err);
                    x[k] = xn;
                }
                wsum += a.lnk[l] * static_cast<double>(err);
                if (a.xhat && live) {
                    float4 *o = reinterpret_cast<float4 *>(a.xhat + (s * a.L + l) * K);
#pragma unroll
                    for (int k = 0; k < K / 4; ++k)
                        o[k] = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
                }
            }
            __syncthreads(); // every thread is done with slot it & 1
            if (tid == 0 && it + 2 < total_it) load_layer(it + 2);
        }
        if (half == 0) {
            long long errs = 0;
#pragma unroll
            for (int k = 0; k < K; ++k)
                errs += (sin[K + k][col] >= 0.f) != (((xm >> k) & 1u) != 0);
            double loss = live ? wsum / a.denom[gt * TILE + col] : 0.0;
            if (!live) errs = 0;
            loss = warp_sum(loss);
            errs = warp_sum(errs);
            if (lane == 0) { s_loss[warp] = loss; s_err[warp] = errs; }
        }
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a.tile_loss[gt * 4 + q] = s_loss[q];
                a.tile_err[gt * 4 + q] = s_err[q];
            }
        }
        __syncthreads();
    }
}

} // namespace detnet
