// stack_h16.cu -- K2-H: the fused DetNet layer stack on tcgen05 tensor cores
// with split-FP16 operands. The default tensor-core path for K=20, v=40;
// stack_tc.cu's 3xTF32 kernel recomputes the (rare) tiles whose activations
// leave the FP16 range.
//
// Same layer algebra as stack_tc.cu -- forward_pre (model.cpp:84-122) +
// loss_plain (loss.cpp:9-31) + the error count (kernels.cpp:63-65) over a
// persistent loop of 128-sample tiles:
//   U1[128 x ZH]  = [q 1 | v x gx][128 x 112] . W1'^T          (b1 folded)
//   U2V[128 x 64] = relu(U1)[128 x ZH] . [W3; W2]^T   (+ [b3; b2] in the epilogue)
// Every operand a is split into two FP16 halves, hi = fp16_rn(a),
// lo = fp16_rn(a - hi) (22 significant bits, as in the 3xTF32 split), and a
// product is hi.hi + hi.lo + lo.hi accumulated in FP32 by kind::f16 MMAs. An
// FP16 MMA takes as many tensor-pipe cycles as a TF32 one of the same N but
// covers K = 16 instead of 8 (tools/micro/mma_rate.cu: N=80, 50 cycles both),
// so a layer needs half the tensor time of the 3xTF32 kernel.
//
// Scaling (all powers of two, so exact): [q 1 | v x gx] enter the MMAs times
// S_IN = 2 and both weight images times WSC = 16, so U1 = S_Z u1 (S_Z = 32),
// z = relu(U1) stays scaled into the second GEMM and U2V = S_U2 [v'; u2]
// (S_U2 = 512); the epilogue folds the unscaling into its bias FMAs. FP16
// range: every converted operand feeds a running max per thread; a tile in
// which any scaled operand reaches the FP16 limit (|z| >~ 2047, |q|, |v|,
// |G x_hat| >~ 32750) is flagged, keeps its input state, and is recomputed by
// the 3xTF32 kernel (FP32 range) on the same stream before anything reads it.
// Below the FP16 normal range a lo half keeps an absolute error <= 2^-25 of
// its scaled value (<= 2^-26 of an activation, 2^-29 of a weight), far under
// the FP32 rounding of the sums it enters.
//
// On-chip residency (one CTA per SM, 384 threads; cf. stack_tc.cu):
//  * TMEM (lane = sample): [0, ZH) U1 accumulator, overwritten in place by
//    the FP16 pairs of z (each thread packs its own columns: hi half then lo
//    half); [ZH, ZH+40) A_dyn hi = pairs of [v (40) | x (20) | gx (20)],
//    [ZH+40, ZH+80) A_dyn lo; [ZH+80, ZH+144) U2V = [v' | u2 | pad];
//    [ZH+144, ZH+160) / [ZH+160, ZH+176) [q | 1 | 0...] hi / lo.
//  * SMEM: the layer's W1 (hi+lo, 70 KB) and [W3; W2] (hi+lo, 40 KB) FP16
//    images, no-swizzle K-major, streamed by the bulk-copy engine.
//  * Registers: the sample's Gram matrix split over two threads, as in
//    stack_tc.cu.
// Hidden units per W1 N-group (ZH = 160): group 0 = units [0, 96) (A threads
// take [0, 48), B [48, 96)), group 1 = [96, 160) (A [96, 128), B [128, 160)):
// the group whose epilogue is on the critical path (1) is the smaller one.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "engine.hpp"
#include "gram.cuh"
#include "tc_ptx.cuh"

namespace detnet {
namespace {

using gram::fma2;
using gram::gram_mv;
using gram::sub2;
constexpr int KX = 20, VV = 40, NG = 210;
constexpr int NA = 105; // Gram entries held by thread A (rows 0..5)
constexpr int W1_K = 112, W23_ROWS = 64;
constexpr uint32_t W23_LBO = W23_ROWS * 16;
constexpr int BT = 64; // per-layer [S_IN b3 (40) | b2 (20) | t | 1/t | pad]
constexpr int NTHREADS = 384;
constexpr float S_IN = 2.f, WSC = 16.f, S_Z = S_IN * WSC, S_U2 = S_Z * WSC;
constexpr float F16_SAFE = 65000.f; // fp16 max finite is 65504 (>= 65520 rounds to inf)

template <int ZH> struct HCfg {
    static_assert(ZH == 160 || ZH == 64, "hidden width");
    static constexpr int NH = ZH == 160 ? 2 : 1;
    __host__ __device__ static constexpr int gw(int h) { return ZH == 160 ? (h == 0 ? 96 : 64) : ZH; }
    __host__ __device__ static constexpr int g0(int h) { return h == 0 ? 0 : gw(0); }
    __host__ __device__ static constexpr int ew(int h) { return gw(h) / 2; }
    // z units of (group h, side s): [seg0, seg0 + ew(h)); FP16 pairs hi at
    // columns [seg0, seg0 + ew/2), lo at [seg0 + ew/2, seg0 + ew)
    __host__ __device__ static constexpr int seg0(int h, int s) { return g0(h) + s * ew(h); }
    // TMEM columns of K-step i (z units [16 i, 16 i + 16)) of the second GEMM
    __host__ __device__ static constexpr int zgrp(int i) { return (NH == 2 && 16 * i >= g0(1)) ? 1 : 0; }
    __host__ __device__ static constexpr int zseg(int i) {
        return seg0(zgrp(i), (16 * i - g0(zgrp(i))) >= ew(zgrp(i)) ? 1 : 0);
    }
    __host__ __device__ static constexpr int zhi(int i) { return zseg(i) + (16 * i - zseg(i)) / 2; }
    __host__ __device__ static constexpr int zlo(int i) { return zhi(i) + ew(zgrp(i)) / 2; }
    static constexpr int C_U1 = 0, C_DYN = ZH, C_DYNLO = ZH + 40, C_U2 = ZH + 80, C_QHI = ZH + 144,
                         C_QLO = ZH + 160, COLS = ZH + 176;
    static constexpr uint32_t TMEM_ALLOC = COLS <= 256 ? 256 : 512;
    static constexpr uint32_t W1_HALF = ZH * W1_K * 2, W23_HALF = W23_ROWS * ZH * 2;
    static constexpr uint32_t W1_BYTES = 2 * W1_HALF, W23_BYTES = 2 * W23_HALF;
    static constexpr uint32_t LAYER_BYTES = W1_BYTES + W23_BYTES;
    static constexpr uint32_t W1_LBO = ZH * 16;
    static constexpr uint32_t SM_W1 = 0, SM_W23 = W1_BYTES, SM_GX = W1_BYTES + W23_BYTES,
                              SM_BAR = SM_GX + KX * 128 * 4, SM_TMEM = SM_BAR + 16 * 8,
                              SM_BT = SM_TMEM + 16, SM_TOTAL = SM_BT + 2 * BT * 4;
    static_assert(COLS <= 512, "TMEM budget");
    static_assert(ew(0) % 16 == 0 && ew(NH - 1) % 16 == 0, "z segments are whole K-steps");
};

struct HKArgs {
    TcArgs a;
    const unsigned char *w; // [L][LAYER_BYTES]
    const float *bt;        // [L][BT]
    float *x_state, *v_state;
    uint8_t *redo;          // [global tile] 1 = recompute with the 3xTF32 kernel
    int *redo_count;
    const int *wbad;        // device flag: an image weight is out of FP16 range
    float limit;            // range limit on scaled operands (F16_SAFE; lower in tests)
    // training trace (TR, ZH == 160): the k_stack_simt layout, unscaled
    float *tr_in, *tr_z, *tr_u2, *tr_xf;
    long ts;
    long long *trace; // debug timeline (build with EXTRA=-DDETNET_TC_TRACE)
};

// Debug timeline: clock64 stamps of CTA 0's first 8 layer iterations, 32
// events each (names in h16_launch_state). Compiled out by default.
#ifdef DETNET_TC_TRACE
#define HTRACE(ev, it, cond)                                                                   \
    do {                                                                                       \
        if (p.trace && blockIdx.x == 0 && (it) < 8 && (cond)) p.trace[(it) * 32 + (ev)] = clock64(); \
    } while (0)
#else
#define HTRACE(ev, it, cond)                                                                   \
    do {                                                                                       \
    } while (0)
#endif

enum { B_W1F = 0, B_W23F = 1, B_U1A = 2, B_U1B = 3, B_U2 = 4, B_VX = 5, B_ZA = 6, B_ZB = 7, B_G = 8,
       B_E2L = 9, NBARS = 10 };
constexpr int BAR_RANGE = 12; // named barrier: tile-end range vote of the 256 epilogue threads

// ---- TMEM stores of packed FP16 pairs (32 lanes x 32 bit) -------------------
__device__ __forceinline__ void stu16(uint32_t t, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
                 "%12,%13,%14,%15,%16};" ::"r"(t),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                 "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
                 "r"(v[14]), "r"(v[15])
                 : "memory");
}
__device__ __forceinline__ void stu8(uint32_t t, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                 "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void stu4(uint32_t t, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(t), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3])
                 : "memory");
}
__device__ __forceinline__ void stu2(uint32_t t, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(t), "r"(v[0]),
                 "r"(v[1])
                 : "memory");
}
template <int N> __device__ __forceinline__ void st_u32(uint32_t t, const uint32_t *v) {
    static_assert(N % 2 == 0, "even column count");
#pragma unroll
    for (int c = 0; c + 16 <= N; c += 16) stu16(t + c, v + c);
    constexpr int c8 = N / 16 * 16;
    if constexpr (N - c8 >= 8) stu8(t + c8, v + c8);
    constexpr int c4 = c8 + (N - c8 >= 8 ? 8 : 0);
    if constexpr (N - c4 >= 4) stu4(t + c4, v + c4);
    constexpr int c2 = c4 + (N - c4 >= 4 ? 4 : 0);
    if constexpr (N - c2 >= 2) stu2(t + c2, v + c2);
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }

// (a0, a1) -> FP16 pair of hi halves and pair of lo halves (a0 in the low 16 bits)
__device__ __forceinline__ __half2 split2(float a0, float a1, uint32_t &hi, uint32_t &lo) {
    const __half2 h = __floats2half2_rn(a0, a1);
    const float2 f = __half22float2(h);
    float l0, l1;
    sub2(a0, a1, f.x, f.y, l0, l1);
    hi = h2u(h);
    lo = h2u(__floats2half2_rn(l0, l1));
    return h;
}

// Split N scaled values into N/2 hi and N/2 lo pair columns; running |max|.
template <int N>
__device__ __forceinline__ void split_row(const float *a, float sc, uint32_t *hi, uint32_t *lo,
                                          float &amax) {
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
        const float a0 = a[2 * k] * sc, a1 = a[2 * k + 1] * sc;
        amax = fmaxf(amax, fmaxf(fabsf(a0), fabsf(a1)));
        split2(a0, a1, hi[k], lo[k]);
    }
}

template <int ZH, bool TR>
__global__ void __launch_bounds__(NTHREADS, 1) k_stack_h16(HKArgs p) {
    static_assert(!TR || ZH == 160, "the training trace is written in the dense unit layout");
    constexpr int IN = 3 * KX + VV;
    using C = HCfg<ZH>;
    constexpr int NH = C::NH;
    constexpr int C_U1 = C::C_U1, C_DYN = C::C_DYN, C_DYNLO = C::C_DYNLO, C_U2 = C::C_U2,
                  C_QHI = C::C_QHI, C_QLO = C::C_QLO;
    constexpr uint32_t SM_W1 = C::SM_W1, SM_W23 = C::SM_W23, SM_GX = C::SM_GX, SM_BAR = C::SM_BAR,
                       SM_TMEM = C::SM_TMEM, SM_BT = C::SM_BT;
    constexpr uint32_t W1_HALF = C::W1_HALF, W23_HALF = C::W23_HALF, W1_BYTES = C::W1_BYTES,
                       W23_BYTES = C::W23_BYTES, LAYER_BYTES = C::LAYER_BYTES, W1_LBO = C::W1_LBO;
    constexpr int U1_LAST = NH == 2 ? B_U1B : B_U1A;
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + SM_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + SM_TMEM);
    float *sGX = reinterpret_cast<float *>(sm + SM_GX);
    const TcArgs &a = p.a;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L0 = a.l_begin, L1 = a.l_end, NL = L1 - L0;
    const long my_tiles = a.n_tiles > blockIdx.x ? (a.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (*p.wbad) { // an FP16 weight image overflowed (device repack): 3xTF32 does everything
        if (threadIdx.x == 0) {
            for (long ti = 0; ti < my_tiles; ++ti) p.redo[a.tile0 + blockIdx.x + ti * gridDim.x] = 1;
            if (my_tiles) atomicAdd(p.redo_count, static_cast<int>(my_tiles));
        }
        return;
    }

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
        tc::tmem_alloc(tmem_slot, C::TMEM_ALLOC);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tmem_slot;
    const long total_it = my_tiles * NL;

    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
        if (warp == 8) {
            // ============ MMA issuer (warp-uniform loop, one elected lane) ============
            const uint32_t sw1 = smem_u32(sm + SM_W1), sw23 = smem_u32(sm + SM_W23);
            const uint32_t id2 = tc::idesc_f16(128, W23_ROWS);
            const uint64_t d1 = tc::smem_desc(sw1, W1_LBO, 128);
            const uint64_t d23 = tc::smem_desc(sw23, W23_LBO, 128);
            constexpr uint64_t S1 = (2 * W1_LBO) >> 4, S23 = (2 * W23_LBO) >> 4;
            constexpr uint64_t H1 = W1_HALF >> 4, H23 = W23_HALF >> 4;
            for (long it = 0; it < total_it; ++it) {
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                const int l = L0 + static_cast<int>(it % NL);
                // K steps of W1 (16 features): 0-1 [q 1 0..], 2-3 v, 4 [v x], 5 [x gx], 6 gx
                auto w1_steps = [&](auto hc, int k0, int k1, bool commit) {
                    constexpr int h = decltype(hc)::value;
                    if (tc::elect_one()) {
                        const uint32_t tb = tc::opaque32(tbase);
                        const uint64_t d1h = tc::opaque64(d1 + C::g0(h)); // (g0/8) * 128 B
                        const uint32_t dcol = tb + C_U1 + C::g0(h);
                        constexpr uint32_t id1 = tc::idesc_f16(128, C::gw(h));
#pragma unroll 1
                        for (int kk = k0; kk < k1; ++kk) {
                            const uint32_t ahi = kk < 2 ? C_QHI + 8 * kk : C_DYN + 8 * (kk - 2);
                            const uint32_t alo = kk < 2 ? C_QLO + 8 * kk : C_DYNLO + 8 * (kk - 2);
                            const uint64_t bhi = d1h + kk * S1;
                            tc::mma_f16_ts(dcol, tb + ahi, bhi, id1, kk > 0);
                            tc::mma_f16_ts(dcol, tb + ahi, bhi + H1, id1, 1);
                            tc::mma_f16_ts(dcol, tb + alo, bhi, id1, 1);
                        }
                        if (commit) tc::commit(&bars[h == 0 ? B_U1A : B_U1B]);
                    }
                    __syncwarp();
                };
                [[maybe_unused]] const bool t0n = lane == 0;
                mbar_wait_guard(&bars[B_W1F], ph);
                HTRACE(0, it, t0n);
                // U1 is overwritten by the [q 1] steps. The previous layer's W23 MMAs
                // (reading z there) precede them in the tensor pipe's issue order;
                // waiting for the epilogue's U2V reads (E2L) keeps these MMAs from
                // competing with those TMEM loads (measured ~1.5% faster). A tile's
                // first layer waits for its q columns instead.
                if (l == L0) mbar_wait_guard(&bars[B_VX], ph);
                else mbar_wait_guard(&bars[B_E2L], ph ^ 1);
                HTRACE(1, it, t0n);
                tc::fence_after();
                w1_steps(std::integral_constant<int, 0>{}, 0, 2, false);
                if constexpr (NH == 2) w1_steps(std::integral_constant<int, 1>{}, 0, 2, false);
                if (l != L0) mbar_wait_guard(&bars[B_VX], ph);
                HTRACE(2, it, t0n);
                tc::fence_after();
                w1_steps(std::integral_constant<int, 0>{}, 2, 5, false);
                mbar_wait_guard(&bars[B_G], ph);
                HTRACE(3, it, t0n);
                tc::fence_after();
                w1_steps(std::integral_constant<int, 0>{}, 5, 7, true);
                if constexpr (NH == 2) w1_steps(std::integral_constant<int, 1>{}, 2, 7, true);
                HTRACE(4, it, t0n);
                mbar_wait_guard(&bars[B_W23F], ph);
                HTRACE(5, it, t0n);
                // U2V = z . [W3; W2]^T, K split by the z groups
                auto w23_group = [&](auto hc) {
                    constexpr int h = decltype(hc)::value;
                    mbar_wait_guard(&bars[h == 0 ? B_ZA : B_ZB], ph);
                    HTRACE(6 + h, it, t0n);
                    tc::fence_after();
                    if (tc::elect_one()) {
                        const uint32_t tb = tc::opaque32(tbase);
                        const uint64_t d23b = tc::opaque64(d23);
                        constexpr int i0 = C::g0(h) / 16, i1 = (C::g0(h) + C::gw(h)) / 16;
                        sfor<i0, i1>([&](auto ic) {
                            constexpr int i = decltype(ic)::value;
                            const uint64_t bhi = d23b + i * S23;
                            tc::mma_f16_ts(tb + C_U2, tb + C::zhi(i), bhi, id2, i > 0);
                            tc::mma_f16_ts(tb + C_U2, tb + C::zhi(i), bhi + H23, id2, 1);
                            tc::mma_f16_ts(tb + C_U2, tb + C::zlo(i), bhi, id2, 1);
                        });
                        if (h == NH - 1) tc::commit(&bars[B_U2]);
                    }
                    __syncwarp();
                };
                w23_group(std::integral_constant<int, 0>{});
                if constexpr (NH == 2) w23_group(std::integral_constant<int, 1>{});
                HTRACE(8, it, t0n);
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
                const int lnext = L0 + static_cast<int>((it + 1) % NL);
                mbar_wait_guard(&bars[U1_LAST], ph); // every W1 group consumed
                HTRACE(28, it, lane == 0);
                load_w1(lnext);
                mbar_wait_guard(&bars[B_E2L], ph);   // W23 consumed, U2V + bias row read
                HTRACE(29, it, lane == 0);
                load_w23(lnext, it + 1);
            }
        }
    } else {
        // ========================= epilogue warps ==========================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 240;" ::: "memory");
        const bool isA = warp >= 4;
        const int side = isA ? 0 : 1;
        const int quad = warp & 3;
        const int col = quad * 32 + lane;
        const uint32_t trow = tbase + (static_cast<uint32_t>(quad * 32) << 16);
        const int bar_x = 1 + quad, bar_g = 6 + quad;
        const float lim = p.limit;
        long it = 0;
        for (long ti = 0; ti < my_tiles; ++ti) {
            const long tile = blockIdx.x + ti * gridDim.x;
            const long gt = a.tile0 + tile;
            const long s = tile * TILE + col;
            DETNET_DASSERT(tile < a.n_tiles && gt >= 0 && L0 >= 0 && L1 > L0);
            const bool live = s < a.n;
            float g[NA];
            const float *gps = a.gp + gt * NG * TILE + col;
            const int e0 = isA ? 0 : NA;
#pragma unroll
            for (int e = 0; e < NA; ++e) g[e] = __ldg(gps + (e0 + e) * TILE);
            float x[KX], v[VV]; // x_hat unscaled; v scaled by S_IN (B side)
#pragma unroll
            for (int k = 0; k < KX; ++k) x[k] = (p.x_state && live) ? p.x_state[s * KX + k] : 0.f;
            float amax = 0.f;             // running max |scaled operand| (signed values)
            __half2 zmax = __float2half2_rn(0.f); // running max of the z pairs (>= 0)
            if (!isA) {
#pragma unroll
                for (int k = 0; k < VV; ++k)
                    v[k] = (p.v_state && live) ? S_IN * p.v_state[s * VV + k] : 0.f;
                float qv[32];
#pragma unroll
                for (int k = 0; k < KX; ++k) qv[k] = a.q32[(gt * KX + k) * TILE + col];
                qv[KX] = 1.f;
#pragma unroll
                for (int k = KX + 1; k < 32; ++k) qv[k] = 0.f;
                uint32_t qh[16], ql[16];
                split_row<32>(qv, S_IN, qh, ql, amax);
                st_u32<16>(trow + C_QHI, qh);
                st_u32<16>(trow + C_QLO, ql);
            }
            double wsum = 0.0;
            uint32_t xm = 0;
            if (isA) xm = a.xmask[gt * TILE + col];
            int lpend = -1;
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
            auto store_v = [&]() { // B: v pairs -> A_dyn (scaled by S_IN)
                uint32_t hi[VV / 2], lo[VV / 2];
                split_row<VV>(v, 1.f, hi, lo, amax);
                st_u32<VV / 2>(trow + C_DYN, hi);
                st_u32<VV / 2>(trow + C_DYNLO, lo);
            };
            for (int l = L0; l < L1; ++l, ++it) {
                const uint32_t ph = static_cast<uint32_t>(it & 1);
                const double lw = isA ? a.lnk[l] : 0.0;
                [[maybe_unused]] const bool tA = threadIdx.x == 128, tB = threadIdx.x == 0;
                [[maybe_unused]] const int tb9 = isA ? 9 : 19; // A events 9-18, B events 19-27
                HTRACE(tb9, it, tA || tB);
                // ---- prep: A_dyn pairs = [v | x | gx]: v (B) and x (A), then G x_hat
                if (isA) {
                    {
                        uint32_t hi[KX / 2], lo[KX / 2];
                        float xa = 0.f; // |S_IN x_hat| <= 2: no range check needed
                        split_row<KX>(x, S_IN, hi, lo, xa);
                        st_u32<KX / 2>(trow + C_DYN + VV / 2, hi);
                        st_u32<KX / 2>(trow + C_DYNLO + VV / 2, lo);
                    }
                    tc::wait_st();
                    tc::fence_before();
                    mbar_arrive(&bars[B_VX]);
                    HTRACE(10, it, tA);
                    float gx[KX];
#pragma unroll
                    for (int k = 0; k < KX; ++k) gx[k] = 0.f;
                    gram_mv<0, 6>(g, x, gx);
                    tc::named_bar(bar_g, 64);
                    HTRACE(11, it, tA);
#pragma unroll
                    for (int k = 6; k < KX; ++k) gx[k] += sGX[k * 128 + col];
                    if constexpr (TR) {
                        float *tin = p.tr_in + static_cast<long>(l) * IN * p.ts + s;
#pragma unroll
                        for (int k = 0; k < KX; ++k) {
                            tin[k * p.ts] = __ldg(a.q32 + (gt * KX + k) * TILE + col);
                            tin[(KX + k) * p.ts] = x[k];
                            tin[(2 * KX + k) * p.ts] = gx[k];
                        }
                    }
                    {
                        uint32_t hi[KX / 2], lo[KX / 2];
                        split_row<KX>(gx, S_IN, hi, lo, amax);
                        st_u32<KX / 2>(trow + C_DYN + (VV + KX) / 2, hi);
                        st_u32<KX / 2>(trow + C_DYNLO + (VV + KX) / 2, lo);
                    }
                    tc::wait_st();
                    tc::fence_before();
                    mbar_arrive(&bars[B_G]);
                    HTRACE(12, it, tA);
                    if (lpend >= 0) settle(); // previous layer's loss / x_hat, off the critical path
                } else {
                    if constexpr (TR) {
                        float *tin = p.tr_in + (static_cast<long>(l) * IN + 3 * KX) * p.ts + s;
#pragma unroll
                        for (int k = 0; k < VV; ++k) tin[k * p.ts] = v[k] * (1.f / S_IN);
                    }
                    if (l == L0) store_v(); // later layers: stored in the previous epilogue 2
                    tc::wait_st();
                    tc::fence_before();
                    mbar_arrive(&bars[B_VX]);
                    HTRACE(20, it, tB);
                    float part[KX];
#pragma unroll
                    for (int k = 0; k < KX; ++k) part[k] = 0.f;
                    gram_mv<6, KX>(g, x, part);
#pragma unroll
                    for (int k = 6; k < KX; ++k) sGX[k * 128 + col] = part[k];
                    tc::named_arrive(bar_g, 64);
                    HTRACE(21, it, tB);
                }

                mbar_wait_guard(&bars[B_W23F], ph);
                // ---- epilogue 1: z = relu(U1) -> FP16 pairs in place (hi, then lo) ----
                auto epi1 = [&](auto hc) {
                    constexpr int h = decltype(hc)::value;
                    constexpr int E = C::ew(h);
                    mbar_wait_guard(&bars[h == 0 ? B_U1A : B_U1B], ph);
                    HTRACE((isA ? 13 : 22) + 2 * h, it, tA || tB);
                    tc::fence_after();
                    const int c0 = C::seg0(h, side);
                    uint32_t r[E];
                    tc::ld_cols_nw<E>(trow + C_U1 + c0, r);
                    tc::wait_ld();
                    uint32_t hp[E / 2], lp[E / 2];
#pragma unroll
                    for (int k = 0; k < E / 2; ++k) {
                        const float u0 = __uint_as_float(r[2 * k]), u1 = __uint_as_float(r[2 * k + 1]);
                        const float z0 = u0 > 0.f ? u0 : 0.f, z1 = u1 > 0.f ? u1 : 0.f;
                        zmax = __hmax2(zmax, split2(z0, z1, hp[k], lp[k]));
                        if constexpr (TR) {
                            float *tz = p.tr_z + (static_cast<long>(l) * ZH + c0 + 2 * k) * p.ts + s;
                            tz[0] = z0 * (1.f / S_Z);
                            tz[p.ts] = z1 * (1.f / S_Z);
                        }
                    }
                    st_u32<E / 2>(trow + C_U1 + c0, hp);
                    st_u32<E / 2>(trow + C_U1 + c0 + E / 2, lp);
                    tc::wait_st();
                    tc::fence_before();
                    mbar_arrive(&bars[h == 0 ? B_ZA : B_ZB]);
                    HTRACE((isA ? 14 : 23) + 2 * h, it, tA || tB);
                };
                epi1(std::integral_constant<int, 0>{});
                if constexpr (NH == 2) epi1(std::integral_constant<int, 1>{});

                // ---- epilogue 2: x_hat = psi_t(u2 + b2) (A), v = v' + b3 (B) ----
                mbar_wait_guard(&bars[B_U2], ph);
                HTRACE(isA ? 17 : 26, it, tA || tB);
                tc::fence_after();
                const float *bt = reinterpret_cast<const float *>(sm + SM_BT + (it & 1) * BT * 4);
                if (isA) {
                    uint32_t r[KX];
                    tc::ld_cols_nw<KX>(trow + C_U2 + VV, r);
                    float b[KX];
#pragma unroll
                    for (int k = 0; k < KX / 4; ++k) {
                        const float4 q = reinterpret_cast<const float4 *>(bt + VV)[k];
                        b[4 * k] = q.x; b[4 * k + 1] = q.y; b[4 * k + 2] = q.z; b[4 * k + 3] = q.w;
                    }
                    const float2 tt = *reinterpret_cast<const float2 *>(bt + 60); // (t, 1/t)
                    tc::wait_ld();
                    mbar_arrive(&bars[B_E2L]);
#pragma unroll
                    for (int k = 0; k < KX; ++k) {
                        const float uu = fmaf(__uint_as_float(r[k]), 1.f / S_U2, b[k]);
                        if constexpr (TR) p.tr_u2[(static_cast<long>(l) * KX + k) * p.ts + s] = uu;
                        // psi_t (model.cpp:32-51) as a clamp of u / t: 3 instructions
                        x[k] = fminf(fmaxf(uu * tt.y, -1.f), 1.f);
                    }
#pragma unroll
                    for (int k = 0; k < KX; ++k) sGX[k * 128 + col] = x[k];
                    tc::named_arrive(bar_x, 64);
                    HTRACE(18, it, tA);
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
                    mbar_arrive(&bars[B_E2L]);
#pragma unroll
                    for (int k = 0; k < VV; ++k) v[k] = fmaf(__uint_as_float(r[k]), S_IN / S_U2, b[k]);
                    // next layer's v columns now (U2V is read, this layer's W1 long done)
                    if (l + 1 < L1) store_v();
                    tc::named_bar(bar_x, 64);
#pragma unroll
                    for (int k = 0; k < KX; ++k) x[k] = sGX[k * 128 + col];
                    HTRACE(27, it, tB);
                }
                lpend = l;
                lw_pend = lw;
            }
            if (isA && lpend >= 0) settle();
            // ---- tile end: range vote, state out, per-tile partials ----
            const float2 zm = __half22float2(zmax);
            const bool bad_mine = !(fmaxf(amax, fmaxf(zm.x, zm.y)) <= lim); // NaN counts as bad
            uint32_t bad_u;
            asm volatile("{\n\t.reg .pred pi, po;\n\tsetp.ne.u32 pi, %1, 0;\n\t"
                         "bar.red.or.pred po, %2, 256, pi;\n\tselp.u32 %0, 1, 0, po;\n\t}"
                         : "=r"(bad_u)
                         : "r"(static_cast<uint32_t>(bad_mine)), "n"(BAR_RANGE)
                         : "memory");
            const bool bad = bad_u != 0;
            if (threadIdx.x == 0) {
                p.redo[gt] = bad ? 1 : 0;
                if (bad) atomicAdd(p.redo_count, 1);
            }
            if constexpr (TR) {
                if (isA) {
#pragma unroll
                    for (int k = 0; k < KX; ++k) p.tr_xf[k * p.ts + s] = x[k];
                }
            }
            if (p.x_state && live && !bad) { // a redone tile restarts from its input state
                if (isA) {
#pragma unroll
                    for (int k = 0; k < KX; ++k) p.x_state[s * KX + k] = x[k];
                } else {
#pragma unroll
                    for (int k = 0; k < VV; ++k) p.v_state[s * VV + k] = v[k] * (1.f / S_IN);
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
                if (lane == 0) {
                    a.tile_loss[gt * 4 + quad] = loss;
                    a.tile_err[gt * 4 + quad] = errs;
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 8) tc::tmem_dealloc(tbase, C::TMEM_ALLOC);
}

// ---- images ------------------------------------------------------------------
// byte offset of element (n, k) in a no-swizzle K-major FP16 image with NR rows
__host__ __device__ inline size_t img16_off(int n, int k, int NR) {
    return static_cast<size_t>(k / 8) * NR * 16 + (n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
}

// W1 image column k -> index into the layer input [q; x; gx; v] (model.cpp:96-99),
// -1 = the bias b1 (multiplied by the constant input 1), -2 = zero padding.
// K order: [q (20) | 1 | 0 x 11 | v (40) | x (20) | gx (20)].
__host__ __device__ inline int w1_src(int k) {
    if (k < KX) return k;
    if (k == KX) return -1;
    if (k < 32) return -2;
    if (k < 72) return 3 * KX + (k - 32);
    if (k < 92) return KX + (k - 72);
    return 2 * KX + (k - 92);
}

// The dense (ZH = 160, unit r = row r) images from the device FP64 master
// weights after a training step; one thread per element. Sets *bad when a
// scaled weight leaves the FP16 range (the kernel then defers to 3xTF32).
__global__ void k_pack_h16_160(const double *__restrict__ params, const double *__restrict__ masks,
                               long P, int L, unsigned char *__restrict__ img,
                               float *__restrict__ bt, int *__restrict__ bad) {
    using C = HCfg<160>;
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
    unsigned char *lay = img + static_cast<size_t>(l) * C::LAYER_BYTES;
    auto put = [&](unsigned char *base, uint32_t half_bytes, size_t off, float val) {
        const float sv = val * WSC;
        if (!(fabsf(sv) <= F16_SAFE)) atomicExch(bad, 1);
        const __half hi = __float2half_rn(sv);
        const __half lo = __float2half_rn(sv - __half2float(hi));
        *reinterpret_cast<__half *>(base + off) = hi;
        *reinterpret_cast<__half *>(base + half_bytes + off) = lo;
    };
    if (e < W1E) {
        const int i = static_cast<int>(e / W1_K), k = static_cast<int>(e % W1_K);
        const int src = w1_src(k);
        const float val = src >= 0 ? w(oW1 + i * IN + src) : (src == -1 ? w(ob1 + i) : 0.f);
        put(lay, C::W1_HALF, img16_off(i, k, ZH), val);
    } else if (e < W1E + W23E) {
        const long e2 = e - W1E;
        const int o = static_cast<int>(e2 / ZH), i = static_cast<int>(e2 % ZH);
        float val = 0.f;
        if (o < VV) val = w(oW3 + o * ZH + i);
        else if (o < VV + KX) val = w(oW2 + (o - VV) * ZH + i);
        put(lay + C::W1_BYTES, C::W23_HALF, img16_off(o, i, W23_ROWS), val);
    } else {
        const int k = static_cast<int>(e - W1E - W23E);
        float val = 0.f;
        if (k < VV) val = S_IN * w(ob3 + k);
        else if (k < VV + KX) val = w(ob2 + (k - VV));
        else if (k == 60) val = static_cast<float>(pr[ot]);
        else if (k == 61) val = static_cast<float>(1.0 / pr[ot]);
        bt[static_cast<size_t>(l) * BT + k] = val;
    }
}

// Host packing of the ZH-row images; units[l] lists the hidden units kept for
// layer l (row r of W1 / column r of [W3; W2] = unit units[l][r]). Returns
// false when a scaled weight is outside the FP16 range.
template <int ZH>
bool pack_images16(std::vector<unsigned char> &img, std::vector<float> &bt, int K, int Z, int V,
                   int L, const double *params, const double *masks,
                   const std::vector<std::vector<int>> &units) {
    using C = HCfg<ZH>;
    const int IN = 3 * K + V;
    const long P = Z * IN + Z + static_cast<long>(K) * Z + K + static_cast<long>(V) * Z + V + 1;
    img.assign(static_cast<size_t>(L) * C::LAYER_BYTES, 0);
    bt.assign(static_cast<size_t>(L) * BT, 0.f);
    bool ok = true;
    auto put = [&](unsigned char *base, uint32_t half_bytes, size_t off, float val) {
        const float sv = val * WSC;
        if (!(std::fabs(sv) <= F16_SAFE)) ok = false;
        const __half hi = __float2half_rn(sv);
        const __half lo = __float2half_rn(sv - __half2float(hi));
        std::memcpy(base + off, &hi, 2);
        std::memcpy(base + half_bytes + off, &lo, 2);
    };
    for (int l = 0; l < L; ++l) {
        const double *pr = params + l * P;
        const double *mk = masks ? masks + l * P : nullptr;
        auto w = [&](long off) { return static_cast<float>(pr[off] * (mk ? mk[off] : 1.0)); };
        const long oW1 = 0, ob1 = static_cast<long>(Z) * IN, oW2 = ob1 + Z,
                   ob2 = oW2 + static_cast<long>(K) * Z, oW3 = ob2 + K,
                   ob3 = oW3 + static_cast<long>(V) * Z, ot = ob3 + V;
        unsigned char *lay = img.data() + static_cast<size_t>(l) * C::LAYER_BYTES;
        const std::vector<int> &us = units[l];
        for (size_t r = 0; r < us.size(); ++r) {
            const int i = us[r];
            for (int k = 0; k < W1_K; ++k) {
                const int src = w1_src(k);
                const float val = src >= 0 ? w(oW1 + i * IN + src) : (src == -1 ? w(ob1 + i) : 0.f);
                put(lay, C::W1_HALF, img16_off(static_cast<int>(r), k, ZH), val);
            }
            for (int o = 0; o < W23_ROWS; ++o) {
                float val = 0.f;
                if (o < VV) val = w(oW3 + o * Z + i);
                else if (o < VV + KX) val = w(oW2 + (o - VV) * Z + i);
                put(lay + C::W1_BYTES, C::W23_HALF, img16_off(o, static_cast<int>(r), W23_ROWS), val);
            }
        }
        float *b = bt.data() + static_cast<size_t>(l) * BT;
        for (int k = 0; k < VV; ++k) b[k] = S_IN * w(ob3 + k);
        for (int k = 0; k < KX; ++k) b[VV + k] = w(ob2 + k);
        b[60] = static_cast<float>(pr[ot]);
        b[61] = static_cast<float>(1.0 / pr[ot]);
    }
    return ok;
}

} // namespace

int h16_prepare() {
    cudaError_t e = cudaFuncSetAttribute(k_stack_h16<160, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(HCfg<160>::SM_TOTAL));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_stack_h16<160, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(HCfg<160>::SM_TOTAL));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_stack_h16<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(HCfg<64>::SM_TOTAL));

    if (e != cudaSuccess)
        return fail(DETNET_ERR_CUDA, "split-fp16 kernel smem attribute: %s", cudaGetErrorString(e));
    return 0;
}

// Pack the split-FP16 images (called by tc_pack with the same live-unit lists).
int h16_pack(TcModel &tc, int K, int Z, int V, int L, const double *params, const double *masks,
             const std::vector<std::vector<int>> &units, size_t max_alive) {
    tc.h16_ready = false;
    tc.zh16 = 0;
    std::vector<unsigned char> img;
    std::vector<float> bt;
    bool ok;
    if (max_alive <= 64 && !std::getenv("DETNET_TC_NO_COMPACT")) {
        tc.zh16 = 64;
        ok = pack_images16<64>(img, bt, K, Z, V, L, params, masks, units);
        tc.rec16 = HCfg<64>::LAYER_BYTES;
    } else {
        tc.zh16 = 160;
        ok = pack_images16<160>(img, bt, K, Z, V, L, params, masks, units);
        tc.rec16 = HCfg<160>::LAYER_BYTES;
    }
    if (!ok) { tc.zh16 = 0; return 0; } // weights outside FP16 range: 3xTF32 only
    const size_t wbytes = img.size(), bbytes = bt.size() * 4;
    if (tc.w16.ensure(wbytes + bbytes + 16)) return fail(DETNET_ERR_CUDA, "cudaMalloc fp16 images");
    char *base = static_cast<char *>(tc.w16.p);
    if (cudaMemcpy(base, img.data(), wbytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(base + wbytes, bt.data(), bbytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(base + wbytes + bbytes, 0, 16) != cudaSuccess)
        return fail(DETNET_ERR_CUDA, "upload fp16 images");
    tc.h16_ready = true;
    return 0;
}

// Buffers of the dense (ZH = 160) images for tc_pack_dense_device; the
// device packer fills them (and raises the range flag cleared here).
int h16_alloc_dense(TcModel &tc, int L, cudaStream_t st) {
    tc.zh16 = 160;
    tc.rec16 = HCfg<160>::LAYER_BYTES;
    const size_t wbytes = static_cast<size_t>(L) * tc.rec16, bbytes = static_cast<size_t>(L) * BT * 4;
    if (tc.w16.ensure(wbytes + bbytes + 16)) return fail(DETNET_ERR_CUDA, "cudaMalloc fp16 images");
    CK(cudaMemsetAsync(static_cast<char *>(tc.w16.p) + wbytes + bbytes, 0, 16, st));
    tc.h16_ready = true;
    return 0;
}

int h16_pack_device(TcModel &tc, const double *params, const double *masks, long P,
                    cudaStream_t st) {
    if (!tc.h16_ready || tc.zh16 != 160) return 1;
    constexpr long PER = 160L * W1_K + W23_ROWS * 160L + BT;
    const long total = PER * tc.L;
    unsigned char *img = static_cast<unsigned char *>(tc.w16.p);
    const size_t wbytes = static_cast<size_t>(tc.L) * tc.rec16;
    float *bt = reinterpret_cast<float *>(img + wbytes);
    int *bad = reinterpret_cast<int *>(img + wbytes + static_cast<size_t>(tc.L) * BT * 4);
    k_pack_h16_160<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(params, masks, P,
                                                                              tc.L, img, bt, bad);
    return cudaGetLastError() == cudaSuccess ? 0 : fail(DETNET_ERR_CUDA, "fp16 device pack");
}

int h16_launch_state(const TcModel &tc, const TcArgs &a, float *xs, float *vs, cudaStream_t st,
                     const TraceBufs *tr, uint8_t *redo, int *redo_count, int sms) {
    if (!tc.h16_ready) return fail(DETNET_ERR_UNSUPPORTED, "split-fp16 images not packed");
    HKArgs p;
    p.a = a;
    p.w = static_cast<const unsigned char *>(tc.w16.p);
    const size_t wbytes = static_cast<size_t>(tc.L) * tc.rec16;
    p.bt = reinterpret_cast<const float *>(static_cast<const char *>(tc.w16.p) + wbytes);
    p.wbad = reinterpret_cast<const int *>(static_cast<const char *>(tc.w16.p) + wbytes +
                                           static_cast<size_t>(tc.L) * BT * 4);
    p.x_state = xs;
    p.v_state = vs;
    p.redo = redo;
    p.redo_count = redo_count;
    const char *lim = std::getenv("DETNET_H16_LIMIT"); // tests: force the 3xTF32 recompute
    p.limit = lim ? static_cast<float>(std::atof(lim)) : F16_SAFE;
    p.tr_in = p.tr_z = p.tr_u2 = p.tr_xf = nullptr;
    p.ts = 0;
    p.trace = nullptr;
    const int grid = static_cast<int>(std::min<long>(a.n_tiles, sms));
    if (grid <= 0) return 0;
    static long long *trace_buf = nullptr;
    const bool tracing = std::getenv("DETNET_TC_TRACE") != nullptr;
    if (tracing) {
        if (!trace_buf) cudaMalloc(&trace_buf, 8 * 32 * sizeof(long long));
        cudaMemsetAsync(trace_buf, 0, 8 * 32 * sizeof(long long), st);
        p.trace = trace_buf;
    }
    if (tr) {
        if (tc.zh16 != 160) return fail(DETNET_ERR_UNSUPPORTED, "training trace needs the dense images");
        p.tr_in = tr->in;
        p.tr_z = tr->z;
        p.tr_u2 = tr->u2;
        p.tr_xf = tr->xf;
        p.ts = tr->ts;
        k_stack_h16<160, true><<<grid, NTHREADS, HCfg<160>::SM_TOTAL, st>>>(p);
    } else if (tc.zh16 == 64) {
        k_stack_h16<64, false><<<grid, NTHREADS, HCfg<64>::SM_TOTAL, st>>>(p);
    } else {
        k_stack_h16<160, false><<<grid, NTHREADS, HCfg<160>::SM_TOTAL, st>>>(p);
    }
    if (tracing) {
        long long h[8 * 32];
        cudaMemcpyAsync(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        const char *nm[32] = {"M:w1f", "M:e2l", "M:vx", "M:g", "M:w1iss", "M:w23f", "M:za", "M:zb",
                              "M:w23iss", "A:start", "A:vx", "A:gbar", "A:g", "A:u1a", "A:za",
                              "A:u1b", "A:zb", "A:u2", "A:end", "B:start", "B:vx", "B:gpart",
                              "B:u1a", "B:za", "B:u1b", "B:zb", "B:u2", "B:end", "P:u1last",
                              "P:e2l", nullptr, nullptr};
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

} // namespace detnet
