// bwd_tc.cu -- the training step's reverse sweep (backward_data,
// backward.cpp:105-165) on tcgen05 tensor cores, K=20, z=160, v=40.
//
// The sweep is the forward's transpose: for every 128-sample tile (TMEM lane
// = sample) and every trainable layer l = L-1 .. lf,
//   a_bar += w_l (x_hat_{l+1} - x),  u2_bar = a_bar psi'(u2),  t_bar += ...
//   Zbar[128 x 160]  = [u2_bar | v_bar | 0][128 x 64] . [W2 (.) M2; W3 (.) M3]
//   u1_bar = Zbar [z > 0]
//   Inbar[128 x 80]  = u1_bar[128 x 160] . (W1 (.) M1)[:, x gx v columns]
//   a_bar <- G gx_bar + x_bar,  v_bar <- v block
// both contractions as 3xTF32 (Ahi.Bhi + Ahi.Blo + Alo.Bhi, hi = rna_tf32,
// FP32 accumulate; kind::tf32 keeps FP32's exponent range, which the adjoints
// -- scaled by 2 ln(k) / ||x - x_tilde||^2 -- need). The per-sample chain
// (a_bar, psi', the relu gate, G gx_bar) runs on CUDA cores, two threads per
// sample as in the forward (thread A: Gram rows 0-5 and a_bar[0, 10); thread
// B: rows 6-19, a_bar[10, 20) and v_bar). The adjoints the weight gradients
// need (u1_bar, [u2_bar; v_bar], t_bar per 32-sample group) go to HBM in the
// layout k_train_bwd writes, so dW (dw_tc.cu) and k_grad_sum are unchanged.
//
// TMEM (lane = sample): [0, 160) Zbar accumulator, overwritten in place by
// u1_bar hi; [160, 224) A1 hi = [u2_bar | v_bar | 0], [224, 288) A1 lo, reused
// for u1_bar lo of units 0-127 once the first contraction is done;
// [288, 320) u1_bar lo of units 128-159; [320, 400) Inbar accumulator.
// SMEM: the layer's B operands (hi + lo, 180 KB), refilled by the bulk-copy
// engine as soon as the contraction reading the previous copy has completed.
#include <cstdio>
#include <cstdlib>

#include "dw_job.hpp"
#include "engine.hpp"
#include "gram.cuh"
#include "tc_ptx.cuh"

namespace detnet {
namespace {

using gram::gram_mv;
constexpr int KX = 20, VV = 40, ZZ = 160, IN = 3 * KX + VV, OO = KX + VV, NG = 210, NA = 105;
constexpr int A1K = 64;  // [u2_bar (20) | v_bar (40) | pad (4)]
constexpr int IBN = 80;  // in_bar entries needed: x (20), gx (20), v (40)
constexpr int C_Z = 0, C_A1 = 160, C_A1LO = 224, C_ULO2 = 288, C_IB = 320;
constexpr uint32_t B1_HALF = ZZ * A1K * 4, B2_HALF = IBN * ZZ * 4; // 40 KB, 50 KB
constexpr uint32_t B1_BYTES = 2 * B1_HALF, B2_BYTES = 2 * B2_HALF;
constexpr uint32_t LAYER_BYTES = B1_BYTES + B2_BYTES;             // 180 KB
constexpr uint32_t SM_B1 = 0, SM_B2 = B1_BYTES, SM_X = LAYER_BYTES,
                   SM_TR = SM_X + KX * 128 * 4, SM_T = SM_TR + (2 * KX + 5) * 128 * 4,
                   SM_BAR = SM_T + 4 * 8, SM_TMEM = SM_BAR + 16 * 8, SM_TOTAL = SM_TMEM + 16;
constexpr int NTHREADS = 384;
// B_TRF: the tile's x_hat_{l+1} and u2_l rows of the forward trace (bulk copies
// by the producer warp, one layer ahead, so the chain never waits on HBM)
// The trace rows (B_TRF) include the layer's relu gates (z > 0 <=> u1 > 0) as
// five bit-mask words per sample, built once per step by k_gate_bits.
enum { B_B1F = 0, B_B2F = 1, B_A1 = 2, B_Z = 3, B_UA = 4, B_UB = 5, B_IB = 6, B_TRF = 7 };

// Offsets of the no-swizzle K-major TF32 images (core matrices of 8 rows x 4)
__host__ __device__ inline uint32_t b_off(int n, int k, int R) {
    return static_cast<uint32_t>((k / 4) * R * 16 + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4);
}

struct BtcArgs {
    BwdArgs b;
    const unsigned char *w; // [L][LAYER_BYTES] images
    const float *tval;      // [L] t
    long long *trace;       // debug timeline (EXTRA=-DDETNET_TC_TRACE, env DETNET_BWD_TRACE)
};

// Debug timeline: clock64 stamps of CTA 0's first 8 layer iterations, 16
// events each. Compiled out by default.
#ifdef DETNET_TC_TRACE
#define BTRACE(ev, it, cond)                                                                   \
    do {                                                                                       \
        if (p.trace && blockIdx.x == 0 && (it) < 8 && (cond)) p.trace[(it) * 16 + (ev)] = clock64(); \
    } while (0)
#else
#define BTRACE(ev, it, cond)                                                                   \
    do {                                                                                       \
    } while (0)
#endif

__device__ __forceinline__ void split(float v, uint32_t &hi, uint32_t &lo) {
    const float h = tc::tf32_rna(v);
    hi = __float_as_uint(h);
    lo = __float_as_uint(v - h);
}

template <int N> __device__ __forceinline__ void st_cols(uint32_t taddr, const uint32_t *v) {
    static_assert(N % 4 == 0, "column count");
#pragma unroll
    for (int c = 0; c + 8 <= N; c += 8) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         taddr + c),
                     "r"(v[c]), "r"(v[c + 1]), "r"(v[c + 2]), "r"(v[c + 3]), "r"(v[c + 4]),
                     "r"(v[c + 5]), "r"(v[c + 6]), "r"(v[c + 7])
                     : "memory");
    }
    if constexpr (N % 8) {
        constexpr int c = N / 8 * 8;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr + c),
                     "r"(v[c]), "r"(v[c + 1]), "r"(v[c + 2]), "r"(v[c + 3])
                     : "memory");
    }
}

__global__ void __launch_bounds__(NTHREADS, 1) k_bwd_tc(BtcArgs p) {
    const BwdArgs &a = p.b;
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + SM_BAR);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(sm + SM_TMEM);
    float *sX = reinterpret_cast<float *>(sm + SM_X);        // [20][128] G gx partial exchange
    double *sT = reinterpret_cast<double *>(sm + SM_T);      // [4] B-side t group sums
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nl_all = a.L - a.lf;
    const int it0 = a.it_begin, it1 = a.it_end < 0 ? nl_all : a.it_end;
    const int NL = it1 - it0;
    const long my_tiles = a.n_tiles > blockIdx.x ? (a.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long total_it = my_tiles * NL;

    if (threadIdx.x == 0) {
        mbar_init(&bars[B_B1F], 1);
        mbar_init(&bars[B_B2F], 1);
        mbar_init(&bars[B_A1], 256);
        mbar_init(&bars[B_Z], 1);
        mbar_init(&bars[B_UA], 128);
        mbar_init(&bars[B_UB], 128);
        mbar_init(&bars[B_IB], 1);
        mbar_init(&bars[B_TRF], 1);
        fence_mbar_init();
    }
    if (warp == 8) {
        tc::tmem_alloc(tslot, 512);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tslot;

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
        if (warp == 8) {
            // ================= MMA issuer (one elected lane) =================
            const uint32_t sb1 = smem_u32(sm + SM_B1), sb2 = smem_u32(sm + SM_B2);
            // GEMM1 as two N = 80 halves (units [0, 80) and [80, 160)): measured
            // ~3.5x faster than single N = 160 instructions
            constexpr uint32_t id1 = tc::idesc_tf32(128, ZZ / 2), id2 = tc::idesc_tf32(128, IBN);
            for (long it = 0; it < total_it; ++it) {
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                mbar_wait_guard(&bars[B_B1F], ph);
                BTRACE(0, it, lane == 0);
                mbar_wait_guard(&bars[B_A1], ph);
                BTRACE(1, it, lane == 0);
                tc::fence_after();
                if (tc::elect_one()) {
                    const uint32_t tb = tc::opaque32(tbase);
#pragma unroll 1
                    for (int ks = 0; ks < A1K / 8; ++ks) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t ro = h * (ZZ / 2 / 8) * 128; // rows [80 h, 80 h + 80)
                            const uint64_t bh = tc::smem_desc(sb1 + ro + ks * 2 * ZZ * 16, ZZ * 16, 128);
                            const uint64_t bl =
                                tc::smem_desc(sb1 + B1_HALF + ro + ks * 2 * ZZ * 16, ZZ * 16, 128);
                            const uint32_t d = tb + C_Z + h * (ZZ / 2);
                            tc::mma_tf32_ts(d, tb + C_A1 + 8 * ks, bh, id1, ks > 0);
                            tc::mma_tf32_ts(d, tb + C_A1 + 8 * ks, bl, id1, 1);
                            tc::mma_tf32_ts(d, tb + C_A1LO + 8 * ks, bh, id1, 1);
                        }
                    }
                    tc::commit(&bars[B_Z]);
                }
                __syncwarp();
                mbar_wait_guard(&bars[B_B2F], ph);
                BTRACE(2, it, lane == 0);
                auto gemm2 = [&](int k0, int k1) {
                    if (tc::elect_one()) {
                        const uint32_t tb = tc::opaque32(tbase);
#pragma unroll 1
                        for (int ks = k0; ks < k1; ++ks) {
                            const uint64_t bh = tc::smem_desc(sb2 + ks * 2 * IBN * 16, IBN * 16, 128);
                            const uint64_t bl =
                                tc::smem_desc(sb2 + B2_HALF + ks * 2 * IBN * 16, IBN * 16, 128);
                            const uint32_t ahi = C_Z + 8 * ks;
                            const uint32_t alo = ks < 16 ? C_A1 + 8 * ks : C_ULO2 + 8 * (ks - 16);
                            tc::mma_tf32_ts(tb + C_IB, tb + ahi, bh, id2, ks > 0);
                            tc::mma_tf32_ts(tb + C_IB, tb + ahi, bl, id2, 1);
                            tc::mma_tf32_ts(tb + C_IB, tb + alo, bh, id2, 1);
                        }
                        if (k1 == ZZ / 8) tc::commit(&bars[B_IB]);
                    }
                    __syncwarp();
                };
                mbar_wait_guard(&bars[B_UA], ph);
                BTRACE(3, it, lane == 0);
                tc::fence_after();
                gemm2(0, 10); // u1_bar units 0-79 (A side)
                mbar_wait_guard(&bars[B_UB], ph);
                BTRACE(4, it, lane == 0);
                tc::fence_after();
                gemm2(10, 20); // units 80-159 (B side)
            }
        } else if (warp == 9) {
            // ============ weight producer (bulk copies, one elected lane) ============
            const bool leader = tc::elect_one();
            auto layer_of = [&](long it) { return a.L - 1 - (it0 + static_cast<int>(it % NL)); };
            auto load = [&](int which, int l) {
                if (leader) {
                    const uint32_t bytes = which == 0 ? B1_BYTES : B2_BYTES;
                    uint64_t *bar = &bars[which == 0 ? B_B1F : B_B2F];
                    mbar_arrive_expect_tx(bar, bytes);
                    bulk_g2s_chunked(sm + (which == 0 ? SM_B1 : SM_B2),
                                     p.w + static_cast<size_t>(l) * LAYER_BYTES + (which == 0 ? 0 : B1_BYTES),
                                     bytes, bar);
                }
                __syncwarp();
            };
            // the tile's trace rows of iteration it: x_hat_{l+1} (20 rows) and u2_l (20)
            auto load_trace = [&](long it) {
                if (leader) {
                    const long tile = blockIdx.x + (it / NL) * gridDim.x;
                    const int l = layer_of(it);
                    float *dst = reinterpret_cast<float *>(sm + SM_TR);
                    mbar_arrive_expect_tx(&bars[B_TRF], (2 * KX + 5) * TILE * 4);
                    for (int i = 0; i < 5; ++i)
                        bulk_g2s(dst + (2 * KX + i) * TILE,
                                 a.gate + (static_cast<long>(l) * 5 + i) * a.ts + tile * TILE,
                                 TILE * 4, &bars[B_TRF]);
                    for (int i = 0; i < KX; ++i) {
                        const float *xr = l + 1 < a.L
                                              ? a.tr_in + (static_cast<long>(l + 1) * IN + KX + i) * a.ts
                                              : a.tr_xf + static_cast<long>(i) * a.ts;
                        bulk_g2s(dst + i * TILE, xr + tile * TILE, TILE * 4, &bars[B_TRF]);
                        bulk_g2s(dst + (KX + i) * TILE,
                                 a.tr_u2 + (static_cast<long>(l) * KX + i) * a.ts + tile * TILE,
                                 TILE * 4, &bars[B_TRF]);
                    }
                }
                __syncwarp();
            };
            if (total_it > 0) {
                load_trace(0);
                load(0, layer_of(0));
                load(1, layer_of(0));
            }
            for (long it = 0; it + 1 < total_it; ++it) {
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                mbar_wait_guard(&bars[B_Z], ph);  // the first contraction read B1
                load(0, layer_of(it + 1));
                // both sides have used this layer's trace rows and gate words
                mbar_wait_guard(&bars[B_UA], ph);
                mbar_wait_guard(&bars[B_UB], ph);
                load_trace(it + 1);
                mbar_wait_guard(&bars[B_IB], ph); // the second read B2
                load(1, layer_of(it + 1));
            }
        }
    } else {
        // ======================= per-sample chain ========================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory");
        const bool isA = warp >= 4;
        const int quad = warp & 3;
        const int col = quad * 32 + lane;
        const uint32_t trow = tbase + (static_cast<uint32_t>(quad * 32) << 16);
        const int bar_x = 1 + quad;
        const int i0 = isA ? 0 : KX / 2; // this side's half of a_bar / u2_bar
        long it = 0;
        for (long ti = 0; ti < my_tiles; ++ti) {
            const long tile = blockIdx.x + ti * gridDim.x;
            const long s = tile * TILE + col;
            DETNET_DASSERT(tile < a.n_tiles && s < a.ts && it0 >= 0 && it1 <= nl_all && a.lf >= 0);
            const bool live = s < a.n;
            float g[NA];
            const float *gps = a.gp + tile * NG * TILE + col;
#pragma unroll
            for (int e = 0; e < NA; ++e) g[e] = __ldg(gps + ((isA ? 0 : NA) + e) * TILE);
            const uint32_t xm = a.xmask[s];
            const float dinv2 = static_cast<float>(2.0 / a.denom[s]);
            float ab[KX / 2], vb[VV];
            if (it0 > 0) {
#pragma unroll
                for (int k = 0; k < KX / 2; ++k) ab[k] = a.state[(i0 + k) * a.ts + s];
#pragma unroll
                for (int k = 0; k < VV; ++k) vb[k] = isA ? 0.f : a.state[(KX + k) * a.ts + s];
            } else {
#pragma unroll
                for (int k = 0; k < KX / 2; ++k) ab[k] = 0.f;
#pragma unroll
                for (int k = 0; k < VV; ++k) vb[k] = 0.f;
            }
            for (int j = it0; j < it1; ++j, ++it) {
                const int l = a.L - 1 - j;
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                // ---- a_bar += w (x_hat_{l+1} - x); u2_bar; t_bar (this side's half) ----
                const float w = static_cast<float>(a.lnk[l]) * dinv2;
                const float t = p.tval[l], tinv = 1.f / t;
                const float *str = reinterpret_cast<const float *>(sm + SM_TR);
                [[maybe_unused]] const bool tA = threadIdx.x == 128, tB = threadIdx.x == 0;
                BTRACE(isA ? 5 : 11, it, tA || tB);
                mbar_wait_guard(&bars[B_TRF], ph);
                float u2b[KX / 2];
                float tb = 0.f;
#pragma unroll
                for (int k = 0; k < KX / 2; ++k) {
                    const int i = i0 + k;
                    const float xk = (xm >> i) & 1u ? 1.f : -1.f;
                    ab[k] = fmaf(w, str[i * TILE + col] - xk, ab[k]);
                    const float u = str[(KX + i) * TILE + col];
                    const bool lin = u >= -t && u < t; // model.cpp:45-51
                    u2b[k] = lin ? ab[k] * tinv : 0.f;
                    tb += lin ? ab[k] * (-u * tinv * tinv) : 0.f;
                }
                float *g23 = a.g23bar + static_cast<long>(l) * OO * a.ts + s;
                {
                    uint32_t hi[KX / 2], lo[KX / 2];
#pragma unroll
                    for (int k = 0; k < KX / 2; ++k) {
                        g23[(i0 + k) * a.ts] = live ? u2b[k] : 0.f;
                        split(u2b[k], hi[k], lo[k]);
                    }
                    // 10 columns: x8 + a pair via two x4 stores would overlap; use x8 + x2
                    st_cols<8>(trow + C_A1 + i0, hi);
                    st_cols<8>(trow + C_A1LO + i0, lo);
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(
                                     trow + C_A1 + i0 + 8),
                                 "r"(hi[8]), "r"(hi[9])
                                 : "memory");
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(
                                     trow + C_A1LO + i0 + 8),
                                 "r"(lo[8]), "r"(lo[9])
                                 : "memory");
                }
                if (!isA) {
#pragma unroll
                    for (int c0 = 0; c0 < VV; c0 += 8) {
                        uint32_t hi[8], lo[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            g23[(KX + c0 + k) * a.ts] = live ? vb[c0 + k] : 0.f;
                            split(vb[c0 + k], hi[k], lo[k]);
                        }
                        st_cols<8>(trow + C_A1 + KX + c0, hi);
                        st_cols<8>(trow + C_A1LO + KX + c0, lo);
                    }
                    // A1 pad [60, 64): zeros (the region held u1_bar lo last layer)
                    const uint32_t z4[4] = {0u, 0u, 0u, 0u};
                    st_cols<4>(trow + C_A1 + OO, z4);
                    st_cols<4>(trow + C_A1LO + OO, z4);
                }
                tc::wait_st();
                tc::fence_before();
                mbar_arrive(&bars[B_A1]);
                BTRACE(isA ? 6 : 12, it, tA || tB);
                // t_bar per 32-sample group: (A half + B half), B's via smem
                {
                    double ts_ = live ? static_cast<double>(tb) : 0.0;
                    ts_ = warp_sum(ts_);
                    if (!isA && lane == 0) sT[quad] = ts_;
                    tc::named_bar(bar_x, 64);
                    if (isA && lane == 0)
                        a.tbar_part[static_cast<long>(l) * (a.ts / 32) + s / 32] = ts_ + sT[quad];
                }
                // relu gate of this side's 80 units: bits [0, 80) (A) or [80, 160) (B)
                // of the sample's five gate words (trace rows 40-44), as 3 words
                uint32_t gate[3];
                {
                    const uint32_t *gw = reinterpret_cast<const uint32_t *>(str) + 2 * KX * TILE + col;
                    if (isA) {
                        gate[0] = gw[0];
                        gate[1] = gw[TILE];
                        gate[2] = gw[2 * TILE] & 0xffffu;
                    } else { // units 80-159 = word 2 bits 16-31, words 3, 4
                        const uint32_t w2 = gw[2 * TILE], w3 = gw[3 * TILE], w4 = gw[4 * TILE];
                        gate[0] = (w2 >> 16) | (w3 << 16);
                        gate[1] = (w3 >> 16) | (w4 << 16);
                        gate[2] = w4 >> 16;
                    }
                }
                // ---- u1_bar = Zbar [z > 0] (this side's 80 units) -> HBM, TMEM (hi in place, lo) ----
                mbar_wait_guard(&bars[B_Z], ph);
                BTRACE(isA ? 7 : 13, it, tA || tB);
                tc::fence_after();
                float *u1b = a.u1bar + (static_cast<long>(l) * ZZ + (isA ? 0 : 80)) * a.ts + s;
#pragma unroll
                for (int b0 = 0; b0 < 80; b0 += 16) { // 16 columns per TMEM round trip
                    uint32_t r[16];
#pragma unroll
                    for (int c0 = 0; c0 < 16; c0 += 8) tc::ld8_nw(trow + C_Z + (isA ? 0 : 80) + b0 + c0, r + c0);
                    tc::wait_ld();
#pragma unroll
                    for (int c0 = 0; c0 < 16; c0 += 8) {
                        uint32_t hi[8], lo[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int u = b0 + c0 + k;
                            const float ub =
                                (gate[u >> 5] >> (u & 31)) & 1u ? __uint_as_float(r[c0 + k]) : 0.f;
                            u1b[u * a.ts] = live ? ub : 0.f;
                            split(ub, hi[k], lo[k]);
                        }
                        const int unit = (isA ? 0 : 80) + b0 + c0; // global unit index
                        st_cols<8>(trow + C_Z + unit, hi);
                        st_cols<8>(trow + (unit < 128 ? C_A1 + unit : C_ULO2 + unit - 128), lo);
                    }
                }
                tc::wait_st();
                tc::fence_before();
                mbar_arrive(&bars[isA ? B_UA : B_UB]);
                BTRACE(isA ? 8 : 14, it, tA || tB);
                // ---- a_bar <- G gx_bar + x_bar; v_bar <- v block ----
                mbar_wait_guard(&bars[B_IB], ph);
                BTRACE(isA ? 9 : 15, it, tA || tB);
                tc::fence_after();
                uint32_t rg[KX], rx[KX / 2];
                tc::ld_cols_nw<KX>(trow + C_IB + KX, rg);     // gx_bar
                tc::ld_cols_nw<8>(trow + C_IB + i0, rx);      // x_bar (this half)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                             : "=r"(rx[8]), "=r"(rx[9])
                             : "r"(trow + C_IB + i0 + 8));
                tc::wait_ld();
                // part = this side's rows of G gx_bar, with x_bar folded into its own half
                float gxb[KX], part[KX];
#pragma unroll
                for (int k = 0; k < KX; ++k) {
                    gxb[k] = __uint_as_float(rg[k]);
                    part[k] = 0.f;
                }
                if (isA) { // (compile-time register indices on both sides)
#pragma unroll
                    for (int k = 0; k < KX / 2; ++k) part[k] = __uint_as_float(rx[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < KX / 2; ++k) part[KX / 2 + k] = __uint_as_float(rx[k]);
                }
                if (isA) gram_mv<0, 6>(g, gxb, part);
                else gram_mv<6, KX>(g, gxb, part);
                // exchange: A needs B's part[0, 10) (rows 10-19 of sX), B needs
                // A's part[10, 20) (rows 0-9)
#pragma unroll
                for (int k = 0; k < KX / 2; ++k) {
                    if (isA) sX[k * 128 + col] = part[KX / 2 + k];
                    else sX[(KX / 2 + k) * 128 + col] = part[k];
                }
                tc::named_bar(bar_x, 64);
                if (isA) {
#pragma unroll
                    for (int k = 0; k < KX / 2; ++k) ab[k] = part[k] + sX[(KX / 2 + k) * 128 + col];
                } else {
#pragma unroll
                    for (int k = 0; k < KX / 2; ++k) ab[k] = part[KX / 2 + k] + sX[k * 128 + col];
                }
                if (!isA) {
                    uint32_t rv[VV];
                    tc::ld_cols_nw<VV>(trow + C_IB + 2 * KX, rv);
                    tc::wait_ld();
#pragma unroll
                    for (int k = 0; k < VV; ++k) vb[k] = __uint_as_float(rv[k]);
                }
                tc::named_bar(bar_x, 64); // sX is free for the next layer
                BTRACE(10, it, tA);
            }
            if (it1 < nl_all && live) { // hand the sweep state to the next layer chunk
#pragma unroll
                for (int k = 0; k < KX / 2; ++k) a.state[(i0 + k) * a.ts + s] = ab[k];
                if (!isA) {
#pragma unroll
                    for (int k = 0; k < VV; ++k) a.state[(KX + k) * a.ts + s] = vb[k];
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 8) tc::tmem_dealloc(tbase, 512);
}

// Relu gates of the forward trace as bit masks: gate[l][w][ts] bit b = z[l][32 w + b] > 0
// (z = relu(u1), so z > 0 <=> u1 > 0, backward.cpp:148-150).
__global__ void k_gate_bits(const float *tr_z, long ts, long n_cols, int lf, int L, uint32_t *gate) {
    const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long per = n_cols * 5;
    if (idx >= static_cast<long>(L - lf) * per) return;
    const int l = lf + static_cast<int>(idx / per);
    const int w = static_cast<int>((idx % per) / n_cols);
    const long s = idx % n_cols;
    DETNET_DASSERT(l >= lf && l < L && w < 5);
    const float *z = tr_z + (static_cast<long>(l) * ZZ + 32 * w) * ts + s;
    float v[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) v[b] = __ldg(z + b * ts);
    uint32_t bits = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) bits |= (v[b] > 0.f ? 1u : 0u) << b;
    gate[(static_cast<long>(l) * 5 + w) * ts + s] = bits;
}

// Device repack of the sweep's B images from the FP64 master records (after
// every Adam step): B1 [160 units][64] = [W2 (.) M2 | W3 (.) M3 | 0]^T,
// B2 [80][160 units] = (W1 (.) M1)[:, 20 + j]^T, each as TF32 hi / lo.
__global__ void k_pack_bwd_tc(const double *params, const double *masks, int L, unsigned char *w,
                              float *tval) {
    constexpr long P = static_cast<long>(ZZ) * IN + ZZ + KX * ZZ + KX + VV * ZZ + VV + 1;
    constexpr long oW1 = 0, ob1 = static_cast<long>(ZZ) * IN, oW2 = ob1 + ZZ,
                   ob2 = oW2 + KX * ZZ, oW3 = ob2 + KX, ob3 = oW3 + VV * ZZ, ot = ob3 + VV;
    constexpr int E1 = ZZ * A1K, E2 = IBN * ZZ;
    const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long>(L) * (E1 + E2)) return;
    const int l = static_cast<int>(idx / (E1 + E2));
    const int e = static_cast<int>(idx % (E1 + E2));
    const double *p = params + l * P;
    const double *mk = masks ? masks + l * P : nullptr;
    auto wm = [&](long off) { return static_cast<float>(p[off] * (mk ? mk[off] : 1.0)); };
    unsigned char *base = w + static_cast<size_t>(l) * LAYER_BYTES;
    float v;
    uint32_t off, half;
    if (e < E1) {
        const int n = e / A1K, k = e % A1K; // unit n, K index k
        v = k < KX ? wm(oW2 + static_cast<long>(k) * ZZ + n)
                   : (k < OO ? wm(oW3 + static_cast<long>(k - KX) * ZZ + n) : 0.f);
        off = SM_B1 + b_off(n, k, ZZ);
        half = B1_HALF;
    } else {
        const int n = (e - E1) / ZZ, k = (e - E1) % ZZ; // in_bar entry n, unit k
        v = wm(oW1 + static_cast<long>(k) * IN + KX + n);
        off = SM_B2 + b_off(n, k, IBN);
        half = B2_HALF;
    }
    const float h = tc::tf32_rna(v);
    *reinterpret_cast<float *>(base + off) = h;
    *reinterpret_cast<float *>(base + off + half) = v - h;
    if (e == 0) tval[l] = static_cast<float>(p[ot]);
}

} // namespace

int bwd_tc_prepare() {
    return cudaFuncSetAttribute(k_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(SM_TOTAL)) == cudaSuccess
               ? 0
               : fail(DETNET_ERR_CUDA, "cudaFuncSetAttribute (tcgen05 sweep smem) failed");
}

long bwd_tc_image_bytes(int L) { return static_cast<long>(L) * LAYER_BYTES + 4L * L + 256; }

int bwd_tc_pack(const double *params, const double *masks, int L, unsigned char *img,
                cudaStream_t st) {
    const long total = static_cast<long>(L) * (ZZ * A1K + IBN * ZZ);
    float *tval = reinterpret_cast<float *>(img + static_cast<size_t>(L) * LAYER_BYTES);
    k_pack_bwd_tc<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(params, masks, L, img,
                                                                             tval);
    return check_launch();
}

int bwd_tc_launch(const BwdArgs &a, const unsigned char *img, int sms, cudaStream_t st) {
    BtcArgs p{a, img, reinterpret_cast<const float *>(img + static_cast<size_t>(a.L) * LAYER_BYTES),
              nullptr};
    static long long *trace_buf = nullptr;
    static const bool tracing = std::getenv("DETNET_BWD_TRACE") != nullptr;
    if (tracing) {
        if (!trace_buf) cudaMalloc(&trace_buf, 8 * 16 * sizeof(long long));
        cudaMemsetAsync(trace_buf, 0, 8 * 16 * sizeof(long long), st);
        p.trace = trace_buf;
    }
    if (a.it_begin == 0) { // the gates of every layer this sweep visits, once
        const long cnt = static_cast<long>(a.L - a.lf) * 5 * a.ts;
        k_gate_bits<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(a.tr_z, a.ts, a.ts, a.lf,
                                                                              a.L, a.gate);
        if (int rc = check_launch()) return rc;
    }
    const int grid = static_cast<int>(std::min<long>(a.n_tiles, sms));
    k_bwd_tc<<<grid, NTHREADS, SM_TOTAL, st>>>(p);
    if (int rc = check_launch()) return rc;
    if (tracing) {
        long long h[8 * 16];
        cudaMemcpyAsync(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        static const char *nm[16] = {"m_b1", "m_a1", "m_b2", "m_ua", "m_ub", "A_st", "A_a1",
                                     "A_z", "A_u", "A_ib", "A_end", "B_st", "B_a1", "B_z", "B_u",
                                     "B_ib"};
        const long long t0 = h[5];
        for (int l = 0; l < 8; ++l) {
            std::fprintf(stderr, "bwd_tc it %d:", l);
            for (int e = 0; e < 16; ++e) std::fprintf(stderr, " %s=%lld", nm[e], h[l * 16 + e] - t0);
            std::fprintf(stderr, "\n");
        }
    }
    return 0;
}

} // namespace detnet
