// stack_tc.cu -- K2-TC: the fused DetNet layer stack on tcgen05 tensor cores
// (3xTF32 split), K=20, z=160, v=40 (the BASELINE.json dims).
//
// Restates forward_pre (model.cpp:84-122) + loss_plain (loss.cpp:9-31) + the
// error count (kernels.cpp:63-65) for a persistent loop over 128-sample
// tiles; every layer of a tile is two dense contractions over the batch:
//   U1[128 x 160]  = [q 1 | x gx v][128 x 104] . W1'^T     (bias b1 folded)
//   U2V[128 x 64]  = relu(U1)[128 x 160] . [W3; W2]^T + [b3; b2]
// each evaluated as Ahi.Bhi + Ahi.Blo + Alo.Bhi with hi = rna_tf32(a),
// lo = rna_tf32(a - hi) (error ~2^-22 relative per product, FP32 accumulate).
//
// On-chip residency (one CTA per SM, 384 threads):
//  * TMEM (512 cols x 128 lanes; lane = sample of the tile):
//      [  0,160) U1 accumulator (two N=80 halves), overwritten in place by z_hi
//      [160,240) A_dyn hi = [x | gx | v] hi   } z_lo of units 80-159 reuses
//      [240,320) A_dyn lo                      } [160,240) once W1 is done
//      z_lo of units 0-79: [408,416) + [440,512) (written during W1 half 2)
//      [320,384) U2V accumulator: [v' (40) | u2 (20) | pad]
//      [384,408) [q | 1 | 0 0 0] hi,  [416,440) lo   (constant per tile)
//  * SMEM: the current layer's W1 (hi+lo, 130 KB) and [W3;W2] (hi+lo, 80 KB)
//    in the no-swizzle K-major core-matrix layout, each streamed in by the
//    bulk-copy engine as soon as the MMAs reading the previous layer's copy
//    have completed (single slot per matrix = natural double buffering,
//    since W1(l+1) lands during the W23 phase of layer l and vice versa).
//  * Registers: each sample's packed Gram matrix (210 FP32) split over two
//    threads (warps w and w+4, the same TMEM lane quadrant): thread A holds
//    rows 0-5 (105 entries) and x_hat, thread B rows 6-19 and v. G x_hat is
//    formed on FP32 CUDA cores with a 14-float smem exchange per layer.
// Warp roles: 4-7 "A" epilogue, 0-3 "B" epilogue, 8 TMEM alloc + weight
// producer + single-thread MMA issuer (warps 9-11 complete its warpgroup so
// setmaxnreg can move registers to the epilogue warpgroups).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "engine.hpp"
#include "tc_ptx.cuh"

namespace detnet {
namespace {

constexpr int KX = 20, VV = 40, NG = 210;
constexpr int NA = 105; // Gram entries held by thread A (rows 0..5)
constexpr int W1_K = 104, W23_ROWS = 64, TMEM_COLS = 512;
constexpr uint32_t W23_LBO = W23_ROWS * 16;
constexpr int BT = 64; // per-layer [b3 (40) | b2 (20) | t | 1/t | pad]
constexpr int NTHREADS = 384; // 2 epilogue warpgroups + 1 control warpgroup

// Shape of one instantiation: ZH hidden units per layer after compaction
// (160 = dense DetNet, 48 = group-pruned configs 3/4 with <= 48 live units).
template <int ZH> struct TcCfg {
    static_assert(ZH % 16 == 0 && ZH <= 160, "hidden width");
    static constexpr int NH = ZH >= 128 ? 2 : 1;   // W1 issued as NH N-groups
    static constexpr int GW = ZH / NH;             // group width (80 | 48)
    static constexpr int EW = GW / 2;              // epilogue-1 columns per thread per group
    static constexpr int C_U1 = 0, C_DYN = ZH, C_DYNLO = ZH + 80, C_U2 = ZH + 160,
                         C_QHI = ZH + 224, C_QLO = ZH + 248;
    // z_lo column of hidden unit j (contiguous per W1 group). With two groups,
    // units of group 0 are written while group 1 still reads A_dyn, so they
    // live in the free columns [C_QLO+24, 512); group 1 reuses A_dyn hi. With
    // one group every W1 MMA has completed, so z_lo reuses A_dyn hi directly.
    __host__ __device__ static constexpr int zlo_col(int j) {
        return NH == 1 ? C_DYN + j : (j >= GW ? C_DYN + (j - GW) : C_QLO + 24 + j);
    }
    static constexpr uint32_t W1_HALF = ZH * W1_K * 4, W23_HALF = W23_ROWS * ZH * 4;
    static constexpr uint32_t W1_BYTES = 2 * W1_HALF, W23_BYTES = 2 * W23_HALF;
    static constexpr uint32_t LAYER_BYTES = W1_BYTES + W23_BYTES;
    static constexpr uint32_t W1_LBO = ZH * 16;
    static constexpr uint32_t SM_W1 = 0, SM_W23 = W1_BYTES, SM_GX = W1_BYTES + W23_BYTES,
                              SM_RED = SM_GX + KX * 128 * 4, SM_BAR = SM_RED + 128,
                              SM_TMEM = SM_BAR + 16 * 8, SM_BT = SM_TMEM + 16,
                              SM_TOTAL = SM_BT + 2 * BT * 4;
    static_assert(C_QLO + 24 <= TMEM_COLS, "TMEM budget");
    static_assert(NH == 1 || zlo_col(GW - 1) < TMEM_COLS, "TMEM budget (z_lo)");
    static_assert(NH == 1 || zlo_col(0) >= C_QLO + 24, "z_lo clear of q");
};

struct TcKArgs {
    TcArgs a;
    const unsigned char *w; // [L][LAYER_BYTES]
    const float *bt;        // [L][BT]
    float *x_state, *v_state;
    long long *trace; // optional debug timeline (DETNET_TC_TRACE): CTA 0, tile 0
    // training trace (TR instantiation, ZH == 160), the k_stack_simt layout:
    // [l][feature][ts] of in = [q; x; Gx; v], z = relu(u1), u2; x_hat_L [K][ts]
    float *tr_in, *tr_z, *tr_u2, *tr_xf;
    long ts;
    // recompute mode (after the split-FP16 kernel): only tiles with redo[tile]
    // set, nothing at all when *redo_count == 0
    const uint8_t *redo;
    const int *redo_count;
};

// Debug timeline (build with EXTRA=-DDETNET_TC_TRACE, run with DETNET_TC_TRACE=1):
// clock64 stamps of CTA 0's first tile, 8 layers x 32 events. Compiled out by
// default -- the checks alone cost a few hundred cycles per layer.
#ifdef DETNET_TC_TRACE
#define TRACE(ev, l)                                                                           \
    do {                                                                                       \
        if (p.trace && blockIdx.x == 0 && (l) - L0 < 8 && trace_on)                            \
            p.trace[((l) - L0) * 32 + (ev)] = clock64();                                       \
    } while (0)
#define TRACE_ON 1
#else
#define TRACE(ev, l)                                                                           \
    do {                                                                                       \
    } while (0)
#define TRACE_ON 0
#endif

// B_VX: v (B warps) and x (A warps) of the next layer are in A_dyn; B_G: G x_hat
// (A warps) is too. W1 is issued in K stages as its inputs become ready:
// [q 1] right after the previous layer's W23, [v x] at B_VX, [gx] at B_G.
// B_E2L: the epilogue has read U2V (so the next layer's [q 1] MMAs do not
// compete with those TMEM loads).
enum { B_W1F = 0, B_W23F = 1, B_U1A = 2, B_U1B = 3, B_U2 = 4, B_VX = 5, B_ZA = 6, B_ZB = 7, B_G = 8,
       B_E2L = 9, NBARS = 10 };

// Store N (multiple of 8) contiguous columns: x16 pieces, then one x8.
template <int N> __device__ __forceinline__ void st_cols(uint32_t taddr, const float *v) {
#pragma unroll
    for (int c = 0; c + 16 <= N; c += 16)
        tc::st16(taddr + c, *reinterpret_cast<const float(*)[16]>(v + c));
    if constexpr (N % 16 != 0) tc::st8(taddr + (N / 16) * 16, v + (N / 16) * 16);
}

// 3xTF32 split: hi = rna_tf32(v); lo = v - hi is exact in FP32 and the tensor
// core drops its low 13 bits (|lo| <= 2^-11 |v|, so the error is <= 2^-21 |v|).
__device__ __forceinline__ void split(float v, float &hi, float &lo) {
    hi = tc::tf32_rna(v);
    lo = v - hi;
}

// Epilogue 2 for one layer: load the whole U2V row (64 columns, one wait),
// x_hat = psi_t(u2 + b2) from columns [40, 60) and, on the B side, v = v' + b3
// from columns [0, 40).
// Epilogue 2 for one layer. A threads: x_hat = psi_t(u2 + b2) from U2V
// columns [40, 60); B threads: v = v' + b3 from columns [0, 40). Only the
// columns a side needs are read (TMEM reads are the epilogue's scarcest
// resource); B gets x_hat from A through shared memory afterwards.
template <bool SIDE_A, int C_U2>
__device__ __forceinline__ void epi2_layer(uint32_t trow, const float *bt, float (&x)[KX],
                                           float (&v)[VV], uint64_t *e2l, long long *tr,
                                           float *tu2 = nullptr, long ts = 0) {
    if (SIDE_A) {
        if (tr) tr[2] = clock64(); // slot 27
        uint32_t r[KX];
        tc::ld_cols_nw<KX>(trow + C_U2 + VV, r);
        float b[KX];
#pragma unroll
        for (int k = 0; k < KX / 4; ++k) {
            const float4 q = reinterpret_cast<const float4 *>(bt + VV)[k];
            b[4 * k] = q.x; b[4 * k + 1] = q.y; b[4 * k + 2] = q.z; b[4 * k + 3] = q.w;
        }
        const float2 tt = *reinterpret_cast<const float2 *>(bt + 60); // (t, 1/t)
        if (tr) tr[3] = clock64();
        tc::wait_ld();
        if (tr) tr[4] = clock64();
        mbar_arrive(e2l);
        if (tr) *tr = clock64();
#pragma unroll
        for (int k = 0; k < KX; ++k) {
            const float uu = __uint_as_float(r[k]) + b[k];
            if (tu2) tu2[k * ts] = uu;
            x[k] = uu <= -tt.x ? -1.f : (uu >= tt.x ? 1.f : uu * tt.y);
        }
    } else {
        uint32_t r[VV];
        tc::ld_cols_nw<VV>(trow + C_U2, r);
        float b[VV];
#pragma unroll
        for (int k = 0; k < VV / 4; ++k) {
            const float4 q = reinterpret_cast<const float4 *>(bt)[k];
            b[4 * k] = q.x; b[4 * k + 1] = q.y; b[4 * k + 2] = q.z; b[4 * k + 3] = q.w;
        }
        tc::wait_ld();
        mbar_arrive(e2l);
#pragma unroll
        for (int k = 0; k < VV; ++k) v[k] = __uint_as_float(r[k]) + b[k];
    }
}

template <int ZH, bool TR>
__global__ void __launch_bounds__(NTHREADS, 1) k_stack_tc(TcKArgs p) {
    static_assert(!TR || ZH == 160, "the training trace is written in the dense unit layout");
    constexpr int IN = 3 * KX + VV;
    using C = TcCfg<ZH>;
    constexpr int NH = C::NH, GW = C::GW, EW = C::EW;
    constexpr int C_U1 = C::C_U1, C_DYN = C::C_DYN, C_DYNLO = C::C_DYNLO, C_U2 = C::C_U2,
                  C_QHI = C::C_QHI, C_QLO = C::C_QLO;
    constexpr uint32_t SM_W1 = C::SM_W1, SM_W23 = C::SM_W23, SM_GX = C::SM_GX,
                       SM_BAR = C::SM_BAR, SM_TMEM = C::SM_TMEM,
                       SM_BT = C::SM_BT;
    constexpr uint32_t W1_HALF = C::W1_HALF, W23_HALF = C::W23_HALF, W1_BYTES = C::W1_BYTES,
                       W23_BYTES = C::W23_BYTES, LAYER_BYTES = C::LAYER_BYTES,
                       W1_LBO = C::W1_LBO;
    constexpr int U1_LAST = NH == 2 ? 3 : 2; // B_U1B : B_U1A
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + SM_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + SM_TMEM);
    float *sGX = reinterpret_cast<float *>(sm + SM_GX);
    const TcArgs &a = p.a;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L0 = a.l_begin, L1 = a.l_end, NL = L1 - L0;
    if (p.redo_count && *p.redo_count == 0) return; // recompute mode, nothing flagged

    if (threadIdx.x == 0) {
        mbar_init(&bars[B_W1F], 1);
        mbar_init(&bars[B_W23F], 1);
        mbar_init(&bars[B_U1A], 1);
        mbar_init(&bars[B_U1B], 1);
        mbar_init(&bars[B_U2], 1);
        mbar_init(&bars[B_VX], 256);
        mbar_init(&bars[B_G], 128);
        mbar_init(&bars[B_E2L], 256);
        mbar_init(&bars[B_ZA], 256);
        mbar_init(&bars[B_ZB], 256);
        fence_mbar_init();
    }
    if (warp == 8) {
        tc::tmem_alloc(tmem_slot, TMEM_COLS);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tmem_slot;
    const long cand_tiles = a.n_tiles > blockIdx.x ? (a.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    long my_tiles = cand_tiles;
    if (p.redo) { // recompute mode: the flagged tiles among this CTA's candidates
        my_tiles = 0;
        for (long ti = 0; ti < cand_tiles; ++ti)
            my_tiles += p.redo[a.tile0 + blockIdx.x + ti * gridDim.x] != 0;
    }
    const long total_it = my_tiles * NL;

    // Registers: the control warpgroup needs few, the epilogue warpgroups hold
    // each sample's Gram matrix (105 floats per thread) + state. setmaxnreg is
    // the first statement of each role branch so ptxas allocates per role.
    if (warp >= 8) {
        // 4 x 40 + 8 x 232 registers per lane = the 384 x 168 the CTA launches with
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
        if (warp == 8) {
            // ============ MMA issuer (warp-uniform loop, one elected lane) ============
            const uint32_t sw1 = smem_u32(sm + SM_W1), sw23 = smem_u32(sm + SM_W23);
            const uint32_t id1 = tc::idesc_tf32(128, GW);
            const uint32_t id2 = tc::idesc_tf32(128, W23_ROWS);
            const uint64_t d1 = tc::smem_desc(sw1, W1_LBO, 128);
            const uint64_t d23 = tc::smem_desc(sw23, W23_LBO, 128);
            constexpr uint64_t S1 = (2 * W1_LBO) >> 4, S23 = (2 * W23_LBO) >> 4;
            constexpr uint64_t H1 = W1_HALF >> 4, H23 = W23_HALF >> 4, NB = (GW / 8 * 128) >> 4;
            for (long it = 0; it < total_it; ++it) {
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                const int l = L0 + static_cast<int>(it % NL);
                [[maybe_unused]] const bool trace_on = it < NL && lane == 0;
                // K steps of W1 (8 columns each): 0-2 [q 1 0 0 0], 3-7 v, 8-9 x, 10-12 [x gx]
                auto w1_steps = [&](int h, int k0, int k1, bool commit) {
                    if (tc::elect_one()) {
                        const uint32_t tb = tc::opaque32(tbase);
                        const uint64_t d1h = tc::opaque64(d1 + h * NB);
                        const uint32_t dcol = tb + C_U1 + GW * h;
#pragma unroll 1
                        for (int kk = k0; kk < k1; ++kk) {
                            const uint32_t ahi = kk < 3 ? C_QHI + 8 * kk : C_DYN + 8 * (kk - 3);
                            const uint32_t alo = kk < 3 ? C_QLO + 8 * kk : C_DYNLO + 8 * (kk - 3);
                            const uint64_t bhi = d1h + kk * S1;
                            tc::mma_tf32_ts(dcol, tb + ahi, bhi, id1, kk > 0);
                            tc::mma_tf32_ts(dcol, tb + ahi, bhi + H1, id1, 1);
                            tc::mma_tf32_ts(dcol, tb + alo, bhi, id1, 1);
                        }
                        if (commit) tc::commit(&bars[h == 0 ? B_U1A : B_U1B]);
                    }
                    __syncwarp();
                };
                mbar_wait_guard(&bars[B_W1F], ph);
                TRACE(11, l);
                // U1 is overwritten: the previous layer's W23 (reading z_hi there)
                // must be complete; a tile's first layer also needs its q columns.
                if (l == L0) mbar_wait_guard(&bars[B_VX], ph);
                else mbar_wait_guard(&bars[B_E2L], ph ^ 1);
                tc::fence_after();
                for (int h = 0; h < NH; ++h) w1_steps(h, 0, 3, false);
                if (l != L0) mbar_wait_guard(&bars[B_VX], ph);
                TRACE(7, l);
                tc::fence_after();
                // group 0 complete first (its epilogue then overlaps group 1's MMAs)
                w1_steps(0, 3, 10, false);
                mbar_wait_guard(&bars[B_G], ph);
                TRACE(13, l);
                tc::fence_after();
                w1_steps(0, 10, 13, true);
                for (int h = 1; h < NH; ++h) w1_steps(h, 3, 13, true);
                TRACE(8, l);
                mbar_wait_guard(&bars[B_W23F], ph);
                TRACE(12, l);
                // U2V = z . [W3; W2]^T, K split by the z groups
                constexpr int KG = GW / 8; // k-steps per group
#pragma unroll 1
                for (int h = 0; h < NH; ++h) {
                    mbar_wait_guard(&bars[h == 0 ? B_ZA : B_ZB], ph);
                    if (h == 0) TRACE(9, l);
                    tc::fence_after();
                    if (tc::elect_one()) {
                        const uint32_t tb = tc::opaque32(tbase);
                        const uint64_t d23h = tc::opaque64(d23 + h * KG * S23);
#pragma unroll
                        for (int k2 = 0; k2 < KG; ++k2) {
                            const int kk = KG * h + k2;
                            const uint64_t bhi = d23h + k2 * S23;
                            const uint32_t zl = h == 0 ? C::zlo_col(8 * k2) : C::zlo_col(GW + 8 * k2);
                            tc::mma_tf32_ts(tb + C_U2, tb + C_U1 + 8 * kk, bhi, id2, kk > 0);
                            tc::mma_tf32_ts(tb + C_U2, tb + C_U1 + 8 * kk, bhi + H23, id2, 1);
                            tc::mma_tf32_ts(tb + C_U2, tb + zl, bhi, id2, 1);
                        }
                        if (h == NH - 1) tc::commit(&bars[B_U2]);
                    }
                    __syncwarp();
                }
                TRACE(10, l);
            }
        } else if (warp == 9) {
            // ================ weight producer (one elected lane) ================
            const bool leader = tc::elect_one();
            auto load_w1 = [&](int l) {
                if (leader) {
                    mbar_arrive_expect_tx(&bars[B_W1F], W1_BYTES);
                    bulk_g2s_chunked(sm + SM_W1, p.w + static_cast<size_t>(l) * LAYER_BYTES,
                                     W1_BYTES, &bars[B_W1F]);
                }
                __syncwarp();
            };
            // [W3; W2] images + the layer's bias row (double-buffered by iteration)
            auto load_w23 = [&](int l, long itn) {
                if (leader) {
                    mbar_arrive_expect_tx(&bars[B_W23F], W23_BYTES + BT * 4);
                    bulk_g2s_chunked(sm + SM_W23,
                                     p.w + static_cast<size_t>(l) * LAYER_BYTES + W1_BYTES,
                                     W23_BYTES, &bars[B_W23F]);
                    bulk_g2s(sm + SM_BT + (itn & 1) * BT * 4, p.bt + static_cast<size_t>(l) * BT,
                             BT * 4, &bars[B_W23F]);
                }
                __syncwarp();
            };
            if (total_it > 0) { load_w1(L0); load_w23(L0, 0); }
            for (long it = 0; it + 1 < total_it; ++it) {
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                [[maybe_unused]] const int l = L0 + static_cast<int>(it % NL);
                const int lnext = L0 + static_cast<int>((it + 1) % NL);
                [[maybe_unused]] const bool trace_on = it < NL && lane == 0;
                mbar_wait_guard(&bars[U1_LAST], ph); // every W1 group consumed
                TRACE(14, l);
                load_w1(lnext);
                // W23 consumed, and the epilogue has read U2V and its bias row: the
                // 80 KB fill now no longer competes with that epilogue for smem
                mbar_wait_guard(&bars[B_E2L], ph);
                TRACE(15, l);
                load_w23(lnext, it + 1);
            }
        }
    } else {
        // ========================= epilogue warps ==========================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory");
        // the x_hat / G x_hat role gets the higher warp ids: the scheduler favours them
        const bool isA = warp >= 4;
        const int quad = warp & 3;
        const int col = quad * 32 + lane; // sample within the tile == TMEM lane
        const uint32_t trow = tbase + (static_cast<uint32_t>(quad * 32) << 16);
        // one-way hand-offs between the two threads of a sample (producer
        // arrives, consumer syncs): x_hat A -> B, G x_hat partial B -> A
        const int bar_x = 1 + quad, bar_g = 6 + quad;
        long it = 0;
        for (long ti = 0; ti < cand_tiles; ++ti) {
            const long tile = blockIdx.x + ti * gridDim.x;
            const long gt = a.tile0 + tile;
            if (p.redo && !p.redo[gt]) continue;
            const long s = tile * TILE + col;
            DETNET_DASSERT(tile < a.n_tiles && gt >= 0);
            const bool live = s < a.n;
            // ---- tile init: Gram entries into registers, state, q ----
            float g[NA];
            const float *gps = a.gp + gt * NG * TILE + col;
            const int e0 = isA ? 0 : NA;
#pragma unroll
            for (int e = 0; e < NA; ++e) g[e] = __ldg(gps + (e0 + e) * TILE);
            float x[KX], v[VV];
#pragma unroll
            for (int k = 0; k < KX; ++k) x[k] = (p.x_state && live) ? p.x_state[s * KX + k] : 0.f;
            if (!isA) {
#pragma unroll
                for (int k = 0; k < VV; ++k) v[k] = (p.v_state && live) ? p.v_state[s * VV + k] : 0.f;
            }
            double wsum = 0.0; // sum_l ln(l+1) ||x - x_hat_l||^2 (divided by denom at the end)
            uint32_t xm = 0;
            if (isA) {
                xm = a.xmask[gt * TILE + col];
            } else {
                float qh[24], ql[24];
#pragma unroll
                for (int k = 0; k < KX; ++k) split(a.q32[(gt * KX + k) * TILE + col], qh[k], ql[k]);
                qh[20] = 1.f; ql[20] = 0.f;
#pragma unroll
                for (int k = 21; k < 24; ++k) { qh[k] = 0.f; ql[k] = 0.f; }
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    tc::st8(trow + C_QHI + 8 * c, qh + 8 * c);
                    tc::st8(trow + C_QLO + 8 * c, ql + 8 * c);
                }
            }
            int lpend = -1;       // layer whose loss / x_hat output is still due (A side)
            double lw_pend = 0.0;
            auto settle = [&]() {
                float err = 0.f;
#pragma unroll
                for (int k = 0; k < KX; ++k) {
                    const float d = ((xm >> k) & 1u ? 1.f : -1.f) - x[k];
                    err = fmaf(d, d, err);
                }
                wsum += lw_pend * static_cast<double>(err);
                if (a.xhat && live) {
                    float4 *o = reinterpret_cast<float4 *>(a.xhat + (s * NL + (lpend - L0)) * KX);
#pragma unroll
                    for (int k = 0; k < KX / 4; ++k)
                        o[k] = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
                }
                lpend = -1;
            };
            for (int l = L0; l < L1; ++l, ++it) {
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                [[maybe_unused]] const bool trace_on = ti == 0 && (threadIdx.x == 0 || threadIdx.x == 128);
                [[maybe_unused]] const int tb16 = isA ? 0 : 16;
                const double lw = isA ? a.lnk[l] : 0.0; // loss weight, fetched early
                TRACE(0 + tb16, l);
                // ---- prep: A_dyn = [v | x | gx] hi/lo. v (B) and x (A) first, then
                // G x_hat (rows 0-5 on A, rows 6-19 on B, 14-float exchange) ----
                if (isA) {
                    {
                        float hi[16], lo[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) split(x[k], hi[k], lo[k]);
                        st_cols<16>(trow + C_DYN + 40, hi);
                        st_cols<16>(trow + C_DYNLO + 40, lo);
                    }
                    tc::wait_st();
                    tc::fence_before();
                    mbar_arrive(&bars[B_VX]);
                    TRACE(1 + tb16, l);
                    if (lpend >= 0) settle();
                    float gx[KX];
#pragma unroll
                    for (int k = 0; k < KX; ++k) gx[k] = 0.f;
                    int e = 0;
#pragma unroll
                    for (int r = 0; r < 6; ++r)
#pragma unroll
                        for (int c = r; c < KX; ++c, ++e) {
                            gx[r] = fmaf(g[e], x[c], gx[r]);
                            if (c != r) gx[c] = fmaf(g[e], x[r], gx[c]);
                        }
                    tc::named_bar(bar_g, 64);
#pragma unroll
                    for (int k = 6; k < KX; ++k) gx[k] += sGX[k * 128 + col];
                    if constexpr (TR) {
                        float *ti = p.tr_in + static_cast<long>(l) * IN * p.ts + s;
#pragma unroll
                        for (int k = 0; k < KX; ++k) {
                            ti[k * p.ts] = __ldg(a.q32 + (gt * KX + k) * TILE + col);
                            ti[(KX + k) * p.ts] = x[k];
                            ti[(2 * KX + k) * p.ts] = gx[k];
                        }
                    }
                    {
                        float hi[24], lo[24];
#pragma unroll
                        for (int k = 0; k < 24; ++k) {
                            const int j = 16 + k;
                            split(j < KX ? x[j < KX ? j : 0] : gx[j >= KX ? j - KX : 0], hi[k], lo[k]);
                        }
                        st_cols<24>(trow + C_DYN + 56, hi);
                        st_cols<24>(trow + C_DYNLO + 56, lo);
                    }
                    tc::wait_st();
                    tc::fence_before();
                    mbar_arrive(&bars[B_G]);
                } else {
                    if constexpr (TR) {
                        float *ti = p.tr_in + (static_cast<long>(l) * IN + 3 * KX) * p.ts + s;
#pragma unroll
                        for (int k = 0; k < VV; ++k) ti[k * p.ts] = v[k];
                    }
#pragma unroll
                    for (int c = 0; c < VV; c += 16) {
                        float hi[16], lo[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) split(v[c + k < VV ? c + k : 0], hi[k], lo[k]);
                        if (c + 16 <= VV) {
                            st_cols<16>(trow + C_DYN + c, hi);
                            st_cols<16>(trow + C_DYNLO + c, lo);
                        } else {
                            st_cols<8>(trow + C_DYN + c, hi);
                            st_cols<8>(trow + C_DYNLO + c, lo);
                        }
                    }
                    tc::wait_st();
                    tc::fence_before();
                    mbar_arrive(&bars[B_VX]);
                    TRACE(1 + tb16, l);
                    float part[KX];
#pragma unroll
                    for (int k = 6; k < KX; ++k) part[k] = 0.f;
                    int e = 0;
#pragma unroll
                    for (int r = 6; r < KX; ++r)
#pragma unroll
                        for (int c = r; c < KX; ++c, ++e) {
                            part[r] = fmaf(g[e], x[c], part[r]);
                            if (c != r) part[c] = fmaf(g[e], x[r], part[c]);
                        }
#pragma unroll
                    for (int k = 6; k < KX; ++k) sGX[k * 128 + col] = part[k];
                    tc::named_arrive(bar_g, 64);
                }
                TRACE(2 + tb16, l);

                // this layer's bias row came with W23; its barrier cannot re-arm before
                // this thread's Z arrivals, so waiting here is race-free
                mbar_wait_guard(&bars[B_W23F], ph);
                // ---- epilogue 1: z = relu(U1) -> z_hi (in place), z_lo. Each W1 group
                // (GW hidden units) is shared by A (first EW) and B (last EW).
#pragma unroll 1
                for (int h = 0; h < NH; ++h) {
                    mbar_wait_guard(&bars[h == 0 ? B_U1A : B_U1B], ph);
                    if (h == 0) TRACE(3 + tb16, l);
                    tc::fence_after();
                    const int c0 = GW * h + (isA ? 0 : EW);
                    uint32_t r[EW];
                    tc::ld_cols_nw<EW>(trow + C_U1 + c0, r);
                    tc::wait_ld();
                    if (h == 0) TRACE(23 + (isA ? 0 : 3), l);
                    float zh[EW], zl[EW];
#pragma unroll
                    for (int k = 0; k < EW; ++k) {
                        const float u = __uint_as_float(r[k]);
                        split(u > 0.f ? u : 0.f, zh[k], zl[k]);
                        if constexpr (TR)
                            p.tr_z[(static_cast<long>(l) * ZH + c0 + k) * p.ts + s] = u > 0.f ? u : 0.f;
                    }
                    st_cols<EW>(trow + C_U1 + c0, zh);
                    st_cols<EW>(trow + C::zlo_col(c0), zl);
                    tc::wait_st();
                    if (h == 0) TRACE(24 + (isA ? 0 : 3), l);
                    tc::fence_before();
                    mbar_arrive(&bars[h == 0 ? B_ZA : B_ZB]);
                }
                TRACE(4 + tb16, l);

                // ---- epilogue 2: x_hat = psi_t(u2 + b2) on both halves; A: loss ----
                mbar_wait_guard(&bars[B_U2], ph);
                TRACE(5 + tb16, l);
                tc::fence_after();
                TRACE(30 + (isA ? 0 : 1), l);
                // bias row: landed with W23 (the MMA warp waited B_W23F before U2)
                const float *bt = reinterpret_cast<const float *>(sm + SM_BT + (it & 1) * BT * 4);
                long long *tr2 = (TRACE_ON && p.trace && blockIdx.x == 0 && l - L0 < 8 && trace_on && isA)
                                     ? p.trace + (l - L0) * 32 + 25
                                     : nullptr;
                if (isA) {
                    epi2_layer<true, C_U2>(trow, bt, x, v, &bars[B_E2L], tr2,
                                           TR ? p.tr_u2 + static_cast<long>(l) * KX * p.ts + s
                                              : nullptr,
                                           p.ts);
#pragma unroll
                    for (int k = 0; k < KX; ++k) sGX[k * 128 + col] = x[k];
                    tc::named_arrive(bar_x, 64);
                } else {
                    epi2_layer<false, C_U2>(trow, bt, x, v, &bars[B_E2L], tr2);
                    tc::named_bar(bar_x, 64);
#pragma unroll
                    for (int k = 0; k < KX; ++k) x[k] = sGX[k * 128 + col];
                }
                // the loss term and x_hat output of this layer are deferred until
                // the next layer's x columns are out (they are off the critical path)
                lpend = l;
                lw_pend = lw;
                TRACE(6 + tb16, l);
            }
            if (isA && lpend >= 0) settle();
            if constexpr (TR) {
                if (isA) {
#pragma unroll
                    for (int k = 0; k < KX; ++k) p.tr_xf[k * p.ts + s] = x[k];
                }
            }
            // ---- tile end: state out, per-tile partials (A warps) ----
            if (p.x_state && live) {
                if (isA) {
#pragma unroll
                    for (int k = 0; k < KX; ++k) p.x_state[s * KX + k] = x[k];
                } else {
#pragma unroll
                    for (int k = 0; k < VV; ++k) p.v_state[s * VV + k] = v[k];
                }
            }
            if (isA) {
                long long errs = 0;
#pragma unroll
                for (int k = 0; k < KX; ++k) errs += (x[k] >= 0.f) != (((xm >> k) & 1u) != 0);
                double loss = live ? wsum / a.denom[gt * TILE + col] : 0.0;
                if (!live) errs = 0;
                loss = warp_sum(loss);
                errs = warp_sum(errs);
                if (lane == 0) { // per lane-quadrant partials, summed in a fixed order later
                    a.tile_loss[gt * 4 + quad] = loss;
                    a.tile_err[gt * 4 + quad] = errs;
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 8) tc::tmem_dealloc(tbase, TMEM_COLS);
}

// ---- device packer (dense images) ---------------------------------------------
// The same images tc_pack builds on the host (ZH = 160, unit r = row r), from
// the device FP64 master weights after a training step: one thread per image
// element. rna_tf32 as integer rounding (== rna_tf32_host for finite values).
__device__ __forceinline__ float rna_dev(float v) {
    const uint32_t b = __float_as_uint(v);
    if ((b & 0x7f800000u) == 0x7f800000u) return v;
    return __uint_as_float((b + 0x1000u) & 0xffffe000u);
}

__global__ void k_pack_tc160(const double *__restrict__ params, const double *__restrict__ masks,
                             long P, int L, float *__restrict__ img, float *__restrict__ bt) {
    using C = TcCfg<160>;
    constexpr int ZH = 160, IN = 3 * KX + VV;
    constexpr long W1E = ZH * W1_K, W23E = W23_ROWS * ZH, PER = W1E + W23E + BT;
    const long gid = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= PER * L) return;
    const int l = static_cast<int>(gid / PER);
    const long e = gid % PER;
    const double *pr = params + l * P;
    const double *mk = masks ? masks + l * P : nullptr;
    auto w = [&](long off) { return static_cast<float>(pr[off] * (mk ? mk[off] : 1.0)); };
    const long oW1 = 0, ob1 = static_cast<long>(ZH) * IN, oW2 = ob1 + ZH, ob2 = oW2 + KX * ZH,
               oW3 = ob2 + KX, ob3 = oW3 + static_cast<long>(VV) * ZH, ot = ob3 + VV;
    float *L1hi = img + static_cast<size_t>(l) * C::LAYER_BYTES / 4;
    if (e < W1E) {
        const int i = static_cast<int>(e / W1_K), k = static_cast<int>(e % W1_K);
        float val = 0.f;
        if (k < KX) val = w(oW1 + i * IN + k);
        else if (k == KX) val = w(ob1 + i);
        else if (k >= 24 && k < 64) val = w(oW1 + i * IN + (k + 36));
        else if (k >= 64) val = w(oW1 + i * IN + (k - 44));
        const float hi = rna_dev(val);
        const size_t off = static_cast<size_t>(k / 4) * ZH * 4 + (i / 8) * 32 + (i % 8) * 4 + (k % 4);
        L1hi[off] = hi;
        L1hi[C::W1_HALF / 4 + off] = rna_dev(val - hi);
    } else if (e < W1E + W23E) {
        const long e2 = e - W1E;
        const int o = static_cast<int>(e2 / ZH), i = static_cast<int>(e2 % ZH);
        float val = 0.f;
        if (o < VV) val = w(oW3 + o * ZH + i);
        else if (o < VV + KX) val = w(oW2 + (o - VV) * ZH + i);
        const float hi = rna_dev(val);
        float *L2hi = L1hi + C::W1_BYTES / 4;
        const size_t off = static_cast<size_t>(i / 4) * W23_ROWS * 4 + (o / 8) * 32 + (o % 8) * 4 + (i % 4);
        L2hi[off] = hi;
        L2hi[C::W23_HALF / 4 + off] = rna_dev(val - hi);
    } else {
        const int k = static_cast<int>(e - W1E - W23E);
        float val = 0.f;
        if (k < VV) val = w(ob3 + k);
        else if (k < VV + KX) val = w(ob2 + (k - VV));
        else if (k == 60) val = static_cast<float>(pr[ot]);
        else if (k == 61) val = static_cast<float>(1.0 / pr[ot]);
        bt[static_cast<size_t>(l) * BT + k] = val;
    }
}

// ---- host: packing into the smem images -------------------------------------
float rna_tf32_host(float v) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    if ((b & 0x7f800000u) == 0x7f800000u) return v;
    b = (b + 0x1000u) & 0xffffe000u;
    float r;
    std::memcpy(&r, &b, 4);
    return r;
}

// offset (floats) of element (n, k) in a no-swizzle K-major B image with NR rows
inline size_t img_off(int n, int k, int NR) {
    return static_cast<size_t>(k / 4) * NR * 4 + (n / 8) * 32 + (n % 8) * 4 + (k % 4);
}

} // namespace

int tc_prepare() {
    cudaError_t e = cudaFuncSetAttribute(k_stack_tc<160, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(TcCfg<160>::SM_TOTAL));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_stack_tc<160, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(TcCfg<160>::SM_TOTAL));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_stack_tc<48, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(TcCfg<48>::SM_TOTAL));
    if (e != cudaSuccess)
        return fail(DETNET_ERR_CUDA, "tcgen05 kernel smem attribute: %s", cudaGetErrorString(e));
    return h16_prepare();
}

namespace {
// Pack every layer into the ZH-row smem images of TcCfg<ZH>. units[l] lists
// the hidden units kept for layer l (row r of the W1 image and column r of
// the [W3; W2] image hold unit units[l][r]; rows past the list stay zero, so
// their z = relu(0) = 0 contributes nothing).
template <int ZH>
void pack_images(std::vector<float> &img, std::vector<float> &bt, int K, int Z, int V, int L,
                 const double *params, const double *masks,
                 const std::vector<std::vector<int>> &units) {
    using C = TcCfg<ZH>;
    const int IN = 3 * K + V;
    const long P = Z * IN + Z + static_cast<long>(K) * Z + K + static_cast<long>(V) * Z + V + 1;
    img.assign(static_cast<size_t>(L) * C::LAYER_BYTES / 4, 0.f);
    bt.assign(static_cast<size_t>(L) * BT, 0.f);
    for (int l = 0; l < L; ++l) {
        const double *pr = params + l * P;
        const double *mk = masks ? masks + l * P : nullptr;
        auto w = [&](long off) { return static_cast<float>(pr[off] * (mk ? mk[off] : 1.0)); };
        const long oW1 = 0, ob1 = static_cast<long>(Z) * IN, oW2 = ob1 + Z,
                   ob2 = oW2 + static_cast<long>(K) * Z, oW3 = ob2 + K,
                   ob3 = oW3 + static_cast<long>(V) * Z, ot = ob3 + V;
        float *L1hi = img.data() + static_cast<size_t>(l) * C::LAYER_BYTES / 4;
        float *L1lo = L1hi + C::W1_HALF / 4;
        float *L2hi = L1hi + C::W1_BYTES / 4;
        float *L2lo = L2hi + C::W23_HALF / 4;
        const std::vector<int> &us = units[l];
        for (size_t r = 0; r < us.size(); ++r) {
            const int i = us[r];
            for (int k = 0; k < W1_K; ++k) {
                // K order [q (20) | 1 | 0 0 0 | v (40) | x (20) | gx (20)];
                // the input vector is [q; x; gx; v] (model.cpp:96-99)
                float val = 0.f;
                if (k < KX) val = w(oW1 + i * IN + k);
                else if (k == KX) val = w(ob1 + i);
                else if (k >= 24 && k < 64) val = w(oW1 + i * IN + (k + 36));
                else if (k >= 64) val = w(oW1 + i * IN + (k - 44));
                const float hi = rna_tf32_host(val);
                L1hi[img_off(static_cast<int>(r), k, ZH)] = hi;
                L1lo[img_off(static_cast<int>(r), k, ZH)] = rna_tf32_host(val - hi);
            }
            for (int o = 0; o < W23_ROWS; ++o) {
                float val = 0.f;
                if (o < VV) val = w(oW3 + o * Z + i);
                else if (o < VV + KX) val = w(oW2 + (o - VV) * Z + i);
                const float hi = rna_tf32_host(val);
                L2hi[img_off(o, static_cast<int>(r), W23_ROWS)] = hi;
                L2lo[img_off(o, static_cast<int>(r), W23_ROWS)] = rna_tf32_host(val - hi);
            }
        }
        float *b = bt.data() + static_cast<size_t>(l) * BT;
        for (int k = 0; k < VV; ++k) b[k] = w(ob3 + k);
        for (int k = 0; k < KX; ++k) b[VV + k] = w(ob2 + k);
        b[60] = static_cast<float>(pr[ot]);
        b[61] = static_cast<float>(1.0 / pr[ot]);
    }
}
} // namespace

int tc_pack(TcModel &tc, int K, int Z, int V, int L, const double *params, const double *masks) {
    tc.K = K; tc.Z = Z; tc.V = V; tc.L = L;
    tc.ready = false;
    tc.zh = 0;
    tc.h16_ready = false;
    tc.zh16 = 0;
    if (K != KX || V != VV) return 0; // other dims use the SIMT path
    const int IN = 3 * K + V;
    const long P = Z * IN + Z + static_cast<long>(K) * Z + K + static_cast<long>(V) * Z + V + 1;
    // Live hidden units per layer: a unit whose masked [W2; W3] column is all
    // zero cannot influence x_hat, v or the loss (model.cpp:114-118), so it is
    // dropped; group-pruned models (config 3/4) keep <= 48 of 160.
    std::vector<std::vector<int>> units(L);
    size_t max_alive = 0;
    for (int l = 0; l < L; ++l) {
        const double *pr = params + l * P;
        const double *mk = masks ? masks + l * P : nullptr;
        const long oW2 = static_cast<long>(Z) * IN + Z, oW3 = oW2 + static_cast<long>(K) * Z + K;
        for (int i = 0; i < Z; ++i) {
            bool alive = false;
            for (int o = 0; o < K && !alive; ++o) {
                const long off = oW2 + static_cast<long>(o) * Z + i;
                alive = static_cast<float>(pr[off] * (mk ? mk[off] : 1.0)) != 0.f;
            }
            for (int o = 0; o < V && !alive; ++o) {
                const long off = oW3 + static_cast<long>(o) * Z + i;
                alive = static_cast<float>(pr[off] * (mk ? mk[off] : 1.0)) != 0.f;
            }
            if (alive) units[l].push_back(i);
        }
        max_alive = std::max(max_alive, units[l].size());
    }
    if (max_alive > 160) return 0; // wider than the dense template: SIMT path
    std::vector<float> img, bt;
    if (max_alive <= 48 && !std::getenv("DETNET_TC_NO_COMPACT")) {
        tc.zh = 48;
        pack_images<48>(img, bt, K, Z, V, L, params, masks, units);
        tc.rec_bytes = TcCfg<48>::LAYER_BYTES;
    } else {
        tc.zh = 160;
        pack_images<160>(img, bt, K, Z, V, L, params, masks, units);
        tc.rec_bytes = TcCfg<160>::LAYER_BYTES;
    }
    const size_t wbytes = img.size() * 4, bbytes = bt.size() * 4;
    if (tc.w.ensure(wbytes + bbytes)) return fail(DETNET_ERR_CUDA, "cudaMalloc tc weights");
    if (cudaMemcpy(tc.w.p, img.data(), wbytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(static_cast<char *>(tc.w.p) + wbytes, bt.data(), bbytes,
                   cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(DETNET_ERR_CUDA, "upload tc weights");
    tc.ready = true;
    return h16_pack(tc, K, Z, V, L, params, masks, units, max_alive);
}

// Rebuild the dense images on the device (training: after each Adam step).
// Returns 1 (nothing done) when the packed model is not the dense ZH = 160 one.
int tc_pack_device(TcModel &tc, const double *params, const double *masks, long P,
                   cudaStream_t st) {
    if (!tc.ready || tc.zh != 160) return 1;
    constexpr long PER = 160L * W1_K + W23_ROWS * 160L + BT;
    const long total = PER * tc.L;
    float *img = static_cast<float *>(tc.w.p);
    float *bt = reinterpret_cast<float *>(static_cast<char *>(tc.w.p) +
                                          static_cast<size_t>(tc.L) * tc.rec_bytes);
    k_pack_tc160<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(params, masks, P, tc.L,
                                                                            img, bt);
    if (cudaGetLastError() != cudaSuccess) return fail(DETNET_ERR_CUDA, "tc device pack");
    // split-FP16 images: 0 = rebuilt, 1 = compacted (stale: host repack), else an error
    if (tc.h16_ready) return h16_pack_device(tc, params, masks, P, st);
    return 0;
}

// Dense models with every hidden unit live (ZH = 160, units in natural
// order): both image sets built on the device from FP64 records already
// there -- the images the host packers make (the training path repacks this
// way after every Adam step), without the host loops (~20 ms per update, paid
// by the drop-in seam on every adam_step).
int tc_pack_dense_device(TcModel &tc, int K, int Z, int V, int L, const double *params,
                         const double *masks, cudaStream_t st) {
    tc.K = K; tc.Z = Z; tc.V = V; tc.L = L;
    tc.ready = false;
    tc.h16_ready = false;
    tc.zh = 160;
    tc.rec_bytes = TcCfg<160>::LAYER_BYTES;
    const size_t wbytes = static_cast<size_t>(L) * tc.rec_bytes, bbytes = static_cast<size_t>(L) * BT * 4;
    if (tc.w.ensure(wbytes + bbytes)) return fail(DETNET_ERR_CUDA, "cudaMalloc tc weights");
    tc.ready = true;
    if (int rc = h16_alloc_dense(tc, L, st)) return rc;
    return tc_pack_device(tc, params, masks, record_size(K, Z, V), st);
}

namespace {
int tc_launch_impl(const TcModel &tc, const TcArgs &a, float *xs, float *vs, cudaStream_t st,
                   const TraceBufs *tr, const uint8_t *redo, const int *redo_count) {
    if (!tc.ready) return fail(DETNET_ERR_UNSUPPORTED, "tcgen05 path not packed for these dims");
    TcKArgs p;
    p.a = a;
    p.w = static_cast<const unsigned char *>(tc.w.p);
    p.bt = reinterpret_cast<const float *>(static_cast<const char *>(tc.w.p) +
                                           static_cast<size_t>(tc.L) * tc.rec_bytes);
    p.x_state = xs;
    p.v_state = vs;
    p.trace = nullptr;
    p.tr_in = p.tr_z = p.tr_u2 = p.tr_xf = nullptr;
    p.ts = 0;
    p.redo = redo;
    p.redo_count = redo_count;
    static long long *trace_buf = nullptr;
    const bool tracing = std::getenv("DETNET_TC_TRACE") != nullptr;
    if (tracing) {
        if (!trace_buf) cudaMalloc(&trace_buf, 8 * 32 * sizeof(long long));
        cudaMemsetAsync(trace_buf, 0, 8 * 32 * sizeof(long long), st);
        p.trace = trace_buf;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = static_cast<int>(std::min<long>(a.n_tiles, sms));
    if (grid <= 0) return 0;
    if (tr) {
        if (tc.zh != 160) return fail(DETNET_ERR_UNSUPPORTED, "tcgen05 training trace needs the dense images");
        p.tr_in = tr->in;
        p.tr_z = tr->z;
        p.tr_u2 = tr->u2;
        p.tr_xf = tr->xf;
        p.ts = tr->ts;
        k_stack_tc<160, true><<<grid, NTHREADS, TcCfg<160>::SM_TOTAL, st>>>(p);
    } else if (tc.zh == 48) {
        k_stack_tc<48, false><<<grid, NTHREADS, TcCfg<48>::SM_TOTAL, st>>>(p);
    } else {
        k_stack_tc<160, false><<<grid, NTHREADS, TcCfg<160>::SM_TOTAL, st>>>(p);
    }
    if (tracing) {
        long long h[8 * 32];
        cudaMemcpyAsync(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        const char *nm[32] = {"A:prep0", "A:vx", "A:g", "A:u1ok", "A:zarr", "A:u2ok", "A:epi2end",
                              "M:vx", "M:w1iss", "M:zready", "M:w23iss", "M:w1f", "M:w23f", "M:g",
                              "P:u1ok", "P:u2ok", "B:prep0", "B:vx", "B:pair", "B:u1ok", "B:zarr",
                              "B:u2ok", "B:epi2end", "A:e1ld", "A:e1st", "A:e2ld", "B:e1ld",
                              "A:e2tr2", "A:e2pre", "A:e2iss", "A:fence", "B:fence"};
        const long long t0 = h[0];
        for (int l = 0; l < 8; ++l) {
            std::fprintf(stderr, "layer %d:", l);
            for (int e = 0; e < 32; ++e)
                if (nm[e]) std::fprintf(stderr, " %s=%lld", nm[e], h[l * 32 + e] - t0);
            std::fprintf(stderr, "\n");
        }
    }
    return 0;
}

} // namespace

int tc_launch_state(const TcModel &tc, const TcArgs &a, float *xs, float *vs, cudaStream_t st,
                    const TraceBufs *tr) {
    return tc_launch_impl(tc, a, xs, vs, st, tr, nullptr, nullptr);
}

int tc_launch_redo(const TcModel &tc, const TcArgs &a, float *xs, float *vs, cudaStream_t st,
                   const TraceBufs *tr, const uint8_t *redo, const int *redo_count) {
    return tc_launch_impl(tc, a, xs, vs, st, tr, redo, redo_count);
}

int tc_launch(const TcModel &tc, const TcArgs &a, cudaStream_t st) {
    return tc_launch_state(tc, a, nullptr, nullptr, st, nullptr);
}

void tc_release(TcModel &tc) {
    tc.w.release();
    tc.w16.release();
    tc.h16_ready = false;
    tc.ready = false;
}

} // namespace detnet
