// k_prep_fast.cuh -- K1 fast path: per-sample preprocessing, one fused
// kernel, a pair of threads per sample (64 samples per 128-thread CTA).
//
// Computes what evaluate_one needs before the layer loop (kernels.cpp:55-58):
//   q = H^T y, G = H^T H                      -> FP32 outputs for the layer stack
//   d = x - x_tilde = G^-1 H^T (H x - y)      -> denom = max(||d||^2, 1e-12)
// Instead of the reference's FP64 LU (linalg.cpp:44-79, kept bit-exact in
// k_preprocess.cuh), d is one FP32 Cholesky solve G d = p with the right-hand
// side p = H^T (H x - y) accumulated in the same pass over H as the Gram
// matrix. H x - y is the channel noise itself (x_j = +-1, x_j h_ij exact), so
// p carries none of the cancellation of the algebraically equal G x - q, and
// d is FP32-accurate (~cond(G) x 2^-24, measured <= 1e-5 relative in ||d||^2).
// Samples whose Cholesky pivots collapse, whose noise is small enough for the
// rounding of H x - y to matter (||H x - y||^2 < 1e-3 ||y||^2, i.e. SNR above
// ~30 dB, which includes the reference's 1e-12 guard, loss.cpp:16-19), or that
// produce NaN are queued for the exact
// reference LU (k_preprocess on an index list), which also owns
// SingularMatrixError.
//
// Work split: warps 0-1 ("A") and 2-3 ("B") hold the same 64 samples, so
// every branch below is warp-uniform. A owns Gram rows 0..R0-1 (upper-triangle
// entries [0, NA)) and q, B rows R0..K-1 and p. The Cholesky factor is
// computed in registers where the Gram halves already live: A factors its
// rows, takes p from B, solves its rows and hands the cross block and the
// folded right-hand side to B through shared memory (one 64-thread named
// barrier per hand-off); B applies the Schur update, factors the trailing
// block and solves it forwards and backwards; A finishes the back
// substitution and forms ||d||^2.
#pragma once

#include <cuda.h>
#include <type_traits>

#include "common.cuh"

namespace detnet {

// Rows [0, R0) of the Gram matrix (and q) belong to thread A, rows [R0, K) (and
// p) to thread B; R0 splits the upper triangle about in half (6 of 20).
template <int K> struct PrepSplit {
    static constexpr int NG = K * (K + 1) / 2;
    static constexpr int r0() {
        int acc = 0;
        for (int r = 0; r < K; ++r) {
            if (2 * (acc + (K - r)) > NG) return r == 0 ? 1 : r;
            acc += K - r;
        }
        return K;
    }
    static constexpr int R0 = r0();
};

__host__ __device__ constexpr int tri_idx(int K, int a, int b) { // a <= b
    return a * K - a * (a - 1) / 2 + (b - a);
}

// ---- streaming layout ------------------------------------------------------
// Persistent CTAs, 2 per SM: 4 consumer warps + 1 producer warp. A tile is 64
// consecutive samples; its H block (64 x N x K floats, contiguous) is streamed
// once through a 2-stage ring of 6-row chunks by a 2-D tensor TMA (box 124
// floats x 64 samples: the per-sample stride in a stage is padded to 496 B so
// the 8-lane phases of a 128-bit shared load hit distinct banks).
#ifndef DETNET_K1_POLICY
#define DETNET_K1_POLICY 1
#endif
#ifndef DETNET_K1_UNROLL
#define DETNET_K1_UNROLL 1
#endif
constexpr int K1_UNROLL = DETNET_K1_UNROLL;
#define K1_BOUNDS __launch_bounds__(PS_THREADS, 2)
constexpr int PS_TILE = 64, PS_ROWS = 6, PS_THREADS = 128;
constexpr int PREP_FAST_N = 30; // n_rx the fast path is instantiated for (K = 20 configs)
template <int K, int N> struct PrepStreamSmem {
    static constexpr int NG = K * (K + 1) / 2;
    static constexpr uint32_t ROWB = K * 4;                          // bytes per H row
    static constexpr uint32_t SSTR = 496;                             // per-sample stride in a stage
    static constexpr uint32_t BOXW = SSTR / 4;                        // TMA box width (floats)
    static constexpr uint32_t STAGE = PS_TILE * SSTR;
    static constexpr uint32_t YTILE = PS_TILE * N * 4;
    static constexpr uint32_t RING = 0;                               // [2][64][SSTR]
    static constexpr uint32_t YB = RING + 2 * STAGE;                  // float [2][64][N]
    static constexpr uint32_t YSLOT = (YTILE + 127) / 128 * 128;
    static constexpr uint32_t XB = YB + 2 * YSLOT;                    // int8 [2][64][K]
    static constexpr uint32_t XSLOT = (PS_TILE * K + 127) / 128 * 128;
    static constexpr uint32_t X1 = XB + 2 * XSLOT;                    // float [K][64]
    static constexpr uint32_t XF = X1 + K * PS_TILE * 4;              // float [64][K] (x = +-1)
    static constexpr uint32_t BAD = XF + K * PS_TILE * 4;             // int [64]
    static constexpr uint32_t BARS = BAD + PS_TILE * 4;               // 8 mbarriers
    static constexpr uint32_t BYTES = BARS + 8 * 8;
    static_assert(PS_ROWS * ROWB <= SSTR && SSTR % 16 == 0 && (SSTR / 16) % 2 == 1,
                  "stage rows must fit; odd 16-byte stride keeps 128-bit loads conflict-free");
    static_assert(N % PS_ROWS == 0, "whole chunks");
};

// Gram entries of one half held as FP32 pairs for fma.rn.f32x2: row a keeps
// columns [a & ~1, K), so an odd row carries one unused lower-triangle slot.
template <int K, int R0> struct PairMap {
    // closed forms only: the indices must fold before scalar replacement of acc[]
    __host__ __device__ static constexpr int len(int a) { return K - (a & ~1); }
    // sum of len(r) for r < a:  a K - sum_{r<a} 2 floor(r / 2)
    __host__ __device__ static constexpr int start0(int a) {
        return a * K - (2 * (a / 2) * (a / 2 - 1) + 2 * (a / 2) * (a & 1));
    }
    __host__ __device__ static constexpr int start(int a) {
        return a < R0 ? start0(a) : start0(a) - start0(R0);
    }
    __host__ __device__ static constexpr int pos(int a, int b) { return start(a) + b - (a & ~1); }
    static constexpr int NA2 = start0(R0);
    static constexpr int NB2 = start0(K) - start0(R0);
    static_assert(start0(1) == K && start0(2) == 2 * K && start0(3) == 3 * K - 2, "closed form");
};

__device__ __forceinline__ void pair_bar(int id) {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

// Compile-time loops (sfor / sfor_rev, common.cuh): triangular nests index
// register arrays, so every index must be a constant before scalar
// replacement; a plain "#pragma unroll" on the outer loop is not enough once
// the nest gets large.

// 2-D tensor TMA load of box {c0 (inner), c1} into shared memory
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)),
                 "l"(policy)
                 : "memory");
}

// d += {a, a} * {b0, b1}
__device__ __forceinline__ void ffma2(float &d0, float &d1, float a, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %2};\n\tmov.b64 rb, {%3, %4};\n\tmov.b64 rd, {%0, %1};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rd;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a), "f"(b0), "f"(b1));
}

// (d0, d1) += (a0, a1) * (b0, b1)
__device__ __forceinline__ void fma2p(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rd, {%0, %1};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rd;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

#ifdef DETNET_PREP_TRACE
#define PTR(ev) \
    if (blockIdx.x == 0 && lane == 0 && it < 3) ptr_t[it][ev] = clock64();
#else
#define PTR(ev)
#endif

// K1 fast path. grid = min(tiles, 2 x SMs), PS_THREADS threads,
// PrepStreamSmem<K, N>::BYTES of dynamic smem.
template <int K, int N>
__global__ void K1_BOUNDS
    k_prep_stream(const __grid_constant__ CUtensorMap tmH, long n, const float *__restrict__ y,
                  const int8_t *__restrict__ x, float *__restrict__ gp, float *__restrict__ q32,
                  double *__restrict__ denom, uint32_t *__restrict__ xmask,
                  uint8_t *__restrict__ flag, int *__restrict__ fb_count,
                  long *__restrict__ fb_list) {
    using S = PrepSplit<K>;
    using SM = PrepStreamSmem<K, N>;
    constexpr int R0 = S::R0, P = PS_TILE;
    using PM = PairMap<K, R0>;
    constexpr int NMAX = PM::NA2 > PM::NB2 ? PM::NA2 : PM::NB2;
    constexpr int NCH = N / PS_ROWS;
    static_assert(K % 4 == 0 && K <= 32 && R0 % 2 == 0, "row pairs / float4 rows / 32-bit mask");
    static_assert(R0 * (K - R0) * 32 * 4 <= 32 * SM::SSTR, "cross block must fit a pair's rows");
    extern __shared__ __align__(128) unsigned char psm[];
    float(*X1)[P] = reinterpret_cast<float(*)[P]>(psm + SM::X1);
    int *badB = reinterpret_cast<int *>(psm + SM::BAD);
    uint64_t *bars = reinterpret_cast<uint64_t *>(psm + SM::BARS);
    uint64_t *full = bars, *empty = bars + 2, *yfull = bars + 4, *yempty = bars + 6;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long ntiles = (n + P - 1) / P;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 4);
            mbar_init(&yfull[i], 1);
            mbar_init(&yempty[i], 4);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // ---- loads: issued by thread 0 (no producer warp: with 4 warps per CTA
    // and 2 CTAs per SM every SM sub-partition runs 2 warps, so each thread can
    // hold 255 registers -- the sample's Gram half, p and an H row -- without
    // spilling). Chunk step cs = (tile iteration) * NCH + chunk goes to ring
    // stage cs & 1; a stage is refilled once all 4 warps released it.
    const bool issuer = threadIdx.x == 0;
    uint64_t pol = 0; // H is read once; evict_normal keeps the 256-B promoted
                      // lines a chunk shares with the next one until it is read
    if (issuer) {
#if DETNET_K1_POLICY == 1
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#elif DETNET_K1_POLICY == 2
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    }
    const long my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long total_cs = my_tiles * NCH;
    auto issue_chunk = [&](long cs) { // thread 0 only; the stage must be free
        if (cs >= total_cs) return;
        const int st = static_cast<int>(cs & 1);
        const long tt = blockIdx.x + (cs / NCH) * gridDim.x;
        const int c = static_cast<int>(cs % NCH);
        mbar_arrive_expect_tx(&full[st], SM::STAGE);
        tma_load_2d(psm + SM::RING + st * SM::STAGE, &tmH, c * PS_ROWS * K, static_cast<int>(tt * P),
                    &full[st], pol);
    };
    auto issue_yx = [&](int itn) { // thread 0 only; y / x of this CTA's tile itn
        if (itn >= my_tiles) return;
        const int yb = itn & 1;
        const long s0 = (blockIdx.x + static_cast<long>(itn) * gridDim.x) * P;
        const int live = static_cast<int>(n - s0 < P ? n - s0 : P);
        float *ybuf = reinterpret_cast<float *>(psm + SM::YB + yb * SM::YSLOT);
        unsigned char *xbuf = psm + SM::XB + yb * SM::XSLOT;
        const uint32_t ybytes = static_cast<uint32_t>(live * N * 4);
        const uint32_t xbytes = static_cast<uint32_t>(live * K);
        if (ybytes % 16 == 0 && xbytes % 16 == 0) {
            mbar_arrive_expect_tx(&yfull[yb], ybytes + xbytes);
            bulk_g2s(ybuf, y + s0 * N, ybytes, &yfull[yb]);
            bulk_g2s(xbuf, x + s0 * K, xbytes, &yfull[yb]);
        } else { // ragged tail: plain loads (one thread, once per launch)
            for (int i = 0; i < live * N; ++i) ybuf[i] = __ldg(y + s0 * N + i);
            for (int i = 0; i < live * K; ++i) xbuf[i] = static_cast<unsigned char>(x[s0 * K + i]);
            mbar_arrive(&yfull[yb]);
        }
    };
    if (issuer) {
        issue_yx(0);
        issue_chunk(0);
        issue_chunk(1);
    }

    // ===================== consumers =====================
    const bool isA = warp < 2;
    const int ls = (warp & 1) * 32 + lane;
    const int bar = 1 + (warp & 1);
    long cstep = 0;
    int it = 0;
#ifdef DETNET_PREP_TRACE
    long long ptr_t[3][12] = {};
#endif
    for (long tt = blockIdx.x; tt < ntiles; tt += gridDim.x, ++it) {
        PTR(0);
        const int yb = it & 1;
        const uint32_t yph = (it >> 1) & 1;
        const long s = tt * P + ls;
        const bool live = s < n;
        const long sc = live ? s : n - 1;
        const long tile = sc / TILE;
        const int col = static_cast<int>(sc % TILE);
        const float *ybuf =
            reinterpret_cast<const float *>(psm + SM::YB + yb * SM::YSLOT) + ls * N;
        mbar_wait_guard(&yfull[yb], yph);
        PTR(1);
        uint32_t mask = 0;
        {
            const int *xw = reinterpret_cast<const int *>(psm + SM::XB + yb * SM::XSLOT + ls * K);
#pragma unroll
            for (int w = 0; w < K / 4; ++w) {
                const int v = xw[w];
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (static_cast<int8_t>(v >> (8 * b)) > 0) mask |= 1u << (4 * w + b);
            }
        }
        auto xs = [&](int j) { return (mask >> j) & 1u ? 1.f : -1.f; };

        // ---- the one pass over H: Gram halves; q = H^T y (A); p = H^T (H x - y) (B) ----
        float acc[NMAX];
#pragma unroll
        for (int e = 0; e < NMAX; ++e) acc[e] = 0.f;
        float pr[K]; // A: q, B: p
#pragma unroll
        for (int j = 0; j < K; ++j) pr[j] = 0.f;
        // B: x as +-1 floats in shared memory (this thread's row only), read
        // back four at a time per H row: keeps 20 registers free for p
        float4 *xf = reinterpret_cast<float4 *>(psm + SM::XF) + ls * (K / 4);
        if (!isA) {
#pragma unroll
            for (int q4 = 0; q4 < K / 4; ++q4)
                xf[q4] = make_float4(xs(4 * q4), xs(4 * q4 + 1), xs(4 * q4 + 2), xs(4 * q4 + 3));
        }
        float rr = 0.f, yy = 0.f; // B: ||H x - y||^2, ||y||^2
        int hold = 0; // stage of the last Gram chunk: released after the Schur hand-off
#pragma unroll 1
        for (int c = 0; c < NCH; ++c, ++cstep) {
            const int st = static_cast<int>(cstep & 1);
            mbar_wait_guard(&full[st], static_cast<uint32_t>((cstep >> 1) & 1));
            const float4 *hrow =
                reinterpret_cast<const float4 *>(psm + SM::RING + st * SM::STAGE + ls * SM::SSTR);
#pragma unroll K1_UNROLL
            for (int r = 0; r < PS_ROWS; ++r) {
                float h[K];
#pragma unroll
                for (int q4 = 0; q4 < K / 4; ++q4) {
                    const float4 v = hrow[r * (K / 4) + q4];
                    h[4 * q4] = v.x; h[4 * q4 + 1] = v.y; h[4 * q4 + 2] = v.z; h[4 * q4 + 3] = v.w;
                }
                auto row = [&](auto ac) {
                    constexpr int a = SF_IDX(ac);
#pragma unroll
                    for (int b = a & ~1; b < K; b += 2)
                        ffma2(acc[PM::pos(a, b)], acc[PM::pos(a, b) + 1], h[a], h[b], h[b + 1]);
                };
                const float yi = ybuf[c * PS_ROWS + r];
                if (isA) {
                    sfor<0, R0>(row);
#pragma unroll
                    for (int j = 0; j < K; j += 2) ffma2(pr[j], pr[j + 1], yi, h[j], h[j + 1]);
                } else {
                    sfor<R0, K>(row);
                    // residual of the transmitted x on this receive row: (H x - y)_i.
                    // x_j h_j is exact; it is the noise itself (y = H x + n), so no
                    // G-sized cancellation enters p, unlike G x - q.
                    float re = -yi, ro = 0.f;
#pragma unroll
                    for (int q4 = 0; q4 < K / 4; ++q4) {
                        const float4 xq = xf[q4];
                        fma2p(re, ro, h[4 * q4], h[4 * q4 + 1], xq.x, xq.y);
                        fma2p(re, ro, h[4 * q4 + 2], h[4 * q4 + 3], xq.z, xq.w);
                    }
                    const float ri = re + ro;
#pragma unroll
                    for (int j = 0; j < K; j += 2) ffma2(pr[j], pr[j + 1], ri, h[j], h[j + 1]);
                    rr = fmaf(ri, ri, rr); // noise energy
                    yy = fmaf(yi, yi, yy); // received energy
                }
            }
            __syncwarp();
            if (c + 1 < NCH) {
                if (lane == 0) mbar_arrive(&empty[st]);
                if (issuer) { // refill the stage two chunk steps ahead
                    mbar_wait_guard(&empty[st], static_cast<uint32_t>((cstep >> 1) & 1));
                    issue_chunk(cstep + 2);
                }
            } else {
                hold = st;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&yempty[yb]); // y / x of this tile consumed
        if (issuer) { // next tile's y / x into the other buffer (released a tile ago)
            if (it >= 1) mbar_wait_guard(&yempty[yb ^ 1], static_cast<uint32_t>(((it - 1) >> 1) & 1));
            issue_yx(it + 1);
        }
        PTR(2);
        // The cross block of a warp pair goes into the pair's OWN sample rows of
        // the held stage: the other pair's B may still be reading its rows of
        // that chunk (B has more work per H row than A).
        float *ub = reinterpret_cast<float *>(psm + SM::RING + hold * SM::STAGE +
                                              (warp & 1) * 32 * SM::SSTR) + lane;
        // G entries of row a (upper triangle) to the tile-major gp layout
        auto put_row = [&](auto ac) {
            constexpr int a = SF_IDX(ac);
#pragma unroll
            for (int b = a; b < K; ++b)
                gp[(tile * S::NG + tri_idx(K, a, b)) * TILE + col] = acc[PM::pos(a, b)];
        };
        // right-looking Cholesky step k on rows (k, LAST): diag slot <- 1/L_kk
        bool bad = false;
        auto chol_step = [&](auto kc, auto lastc, auto gdiag) {
            constexpr int k = SF_IDX(kc), LAST = SF_IDX(lastc);
            const float p = acc[PM::pos(k, k)];
            if (!(p > 1e-5f * gdiag(k))) bad = true;
            const float dinv = rsqrtf(fmaxf(p, 1e-30f));
            acc[PM::pos(k, k)] = dinv;
#pragma unroll
            for (int j = k + 1; j < K; ++j) acc[PM::pos(k, j)] *= dinv;
            sfor<k + 1, LAST>([&](auto ic) {
                constexpr int i = SF_IDX(ic);
#pragma unroll
                for (int j = i; j < K; ++j)
                    acc[PM::pos(i, j)] = fmaf(-acc[PM::pos(k, i)], acc[PM::pos(k, j)], acc[PM::pos(i, j)]);
            });
        };
        if (live) {
            if (isA) {
                sfor<0, R0>(put_row);
#pragma unroll
                for (int j = 0; j < K; ++j) q32[(tile * K + j) * TILE + col] = pr[j];
                xmask[s] = mask;
            } else {
                sfor<R0, K>(put_row);
            }
        }
        PTR(3);

        // ---- d = x - x_tilde = G^-1 p: FP32 Cholesky G = R^T R, split A | B ----
        float z[K];
        if (isA) {
            float gd[R0];
#pragma unroll
            for (int k = 0; k < R0; ++k) gd[k] = acc[PM::pos(k, k)];
            sfor<0, R0>([&](auto kc) {
                chol_step(kc, std::integral_constant<int, R0>{}, [&](int k) { return gd[k]; });
            });
            pair_bar(bar); // (0) B -> A: p
            PTR(4);
            // forward solve R^T z = p on rows [0, R0), fold them into rows [R0, K)
            sfor<0, R0>([&](auto kc) {
                constexpr int k = SF_IDX(kc);
                float t = X1[k][ls];
#pragma unroll
                for (int m = 0; m < k; ++m) t = fmaf(-acc[PM::pos(m, k)], z[m], t);
                z[k] = t * acc[PM::pos(k, k)];
            });
#pragma unroll
            for (int j = R0; j < K; ++j) {
                float t = X1[j][ls];
#pragma unroll
                for (int m = 0; m < R0; ++m) t = fmaf(-acc[PM::pos(m, j)], z[m], t);
                X1[j][ls] = t;
            }
#pragma unroll
            for (int m = 0; m < R0; ++m)
#pragma unroll
                for (int j = R0; j < K; ++j)
                    ub[(m * (K - R0) + (j - R0)) * 32] = acc[PM::pos(m, j)];
            pair_bar(bar); // (1) A -> B: cross block, folded rhs
            PTR(5);
            pair_bar(bar); // (2) B -> A: d[R0..K); B is done with the cross block
            PTR(6);
            // the cross block was written through the generic proxy into a ring
            // stage the TMA (async proxy) refills next: order the two
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[hold]);
            if (issuer) { // the held stage (this tile's last chunk) -> chunk step + 2
                mbar_wait_guard(&empty[hold], static_cast<uint32_t>(((cstep - 1) >> 1) & 1));
                issue_chunk(cstep + 1);
            }
            float d[K];
#pragma unroll
            for (int j = R0; j < K; ++j) d[j] = X1[j][ls];
            sfor_rev<0, R0>([&](auto kc) {
                constexpr int k = SF_IDX(kc);
                float t = z[k];
#pragma unroll
                for (int j = k + 1; j < K; ++j) t = fmaf(-acc[PM::pos(k, j)], d[j], t);
                d[k] = t * acc[PM::pos(k, k)];
            });
            if (badB[ls]) bad = true;
            double dn = 0.0;
#pragma unroll
            for (int j = 0; j < K; ++j) dn = fma(static_cast<double>(d[j]), static_cast<double>(d[j]), dn);
            // near-noise-free samples (the reference's 1e-12 guard,
            // loss.cpp:16-19; also caught by B's energy test) and NaN take the exact LU
            if (!(dn >= 1e-6)) bad = true;
            PTR(7);
            if (live) {
                if (bad) {
                    const int slot = atomicAdd(fb_count, 1);
                    fb_list[slot] = s;
                    flag[s] = 0;
                    denom[s] = 1.0;
                } else {
                    flag[s] = 0;
                    denom[s] = dn;
                }
            }
        } else {
            float gd[K - R0];
#pragma unroll
            for (int k = R0; k < K; ++k) gd[k - R0] = acc[PM::pos(k, k)];
#pragma unroll
            for (int j = 0; j < K; ++j) X1[j][ls] = pr[j];
            pair_bar(bar); // (0)
            PTR(4);
            pair_bar(bar); // (1)
            PTR(5);
            sfor<0, R0>([&](auto mc) {
                constexpr int m = SF_IDX(mc);
                float u[K];
#pragma unroll
                for (int j = R0; j < K; ++j) u[j] = ub[(m * (K - R0) + (j - R0)) * 32];
                sfor<R0, K>([&](auto ic) {
                    constexpr int i = SF_IDX(ic);
#pragma unroll
                    for (int j = i; j < K; ++j) acc[PM::pos(i, j)] = fmaf(-u[i], u[j], acc[PM::pos(i, j)]);
                });
            });
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[hold]);
            sfor<R0, K>([&](auto kc) {
                chol_step(kc, std::integral_constant<int, K>{}, [&](int k) { return gd[k - R0]; });
            });
            sfor<R0, K>([&](auto kc) {
                constexpr int k = SF_IDX(kc);
                float t = X1[k][ls];
#pragma unroll
                for (int m = R0; m < k; ++m) t = fmaf(-acc[PM::pos(m, k)], z[m], t);
                z[k] = t * acc[PM::pos(k, k)];
            });
            sfor_rev<R0, K>([&](auto kc) {
                constexpr int k = SF_IDX(kc);
                float t = z[k];
#pragma unroll
                for (int j = k + 1; j < K; ++j) t = fmaf(-acc[PM::pos(k, j)], z[j], t);
                z[k] = t * acc[PM::pos(k, k)];
            });
#pragma unroll
            for (int k = R0; k < K; ++k) X1[k][ls] = z[k];
            // H x - y is formed in FP32 from y ~ H x: once the noise is below
            // ~1e-3 of the signal (SNR above ~30 dB) its rounding error reaches
            // 1e-5 of ||d||^2 -- such samples take the exact LU.
            if (!(rr >= 1e-3f * yy)) bad = true;
            badB[ls] = bad ? 1 : 0;
            pair_bar(bar); // (2)
            PTR(6);
            PTR(7);
        }
    }
#ifdef DETNET_PREP_TRACE
    if (blockIdx.x == 0 && lane == 0 && (warp == 0 || warp == 2))
        for (int t = 0; t < 3; ++t)
            printf("prep trace warp %d tile %d: %lld %lld %lld %lld %lld %lld %lld\n", warp, t,
                   ptr_t[t][1] - ptr_t[t][0], ptr_t[t][2] - ptr_t[t][0], ptr_t[t][3] - ptr_t[t][0],
                   ptr_t[t][4] - ptr_t[t][0], ptr_t[t][5] - ptr_t[t][0], ptr_t[t][6] - ptr_t[t][0],
                   ptr_t[t][7] - ptr_t[t][0]);
#endif
}

} // namespace detnet
