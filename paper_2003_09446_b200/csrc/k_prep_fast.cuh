// k_prep_fast.cuh -- K1 fast path: per-sample preprocessing with a pair of
// threads per sample (64 samples per 128-thread CTA).
//
// Computes what evaluate_one needs before the layer loop (kernels.cpp:55-58):
//   q = H^T y, G = H^T H                      -> FP32 outputs for the layer stack
//   d = x - x_tilde = G^-1 H^T (H x - y)      -> denom = max(||d||^2, 1e-12)
// Instead of the reference's FP64 LU (linalg.cpp:44-79, kept bit-exact in
// k_preprocess.cuh), d starts from an FP32 Cholesky solve of G d0 = G x - q
// (Cholesky in shared memory) and is refined (up to two steps) with the
// residual H^T (H (x - d) - y) formed in FP64 straight from the FP32 inputs,
// so d (hence the loss denominator) is FP64-accurate (~1e-10 relative) for
// well-conditioned samples. Samples whose Cholesky pivots collapse or whose
// refinement correction is not small are queued for the exact reference LU
// (k_preprocess on an index list), which also owns SingularMatrixError.
//
// Work split inside a pair (lanes 2i, 2i+1 = one sample; both stream the same
// H rows, so each 80-byte row is fetched once per pair):
//   half 0: Gram rows 0..R0-1 (upper-triangle entries [0, NA)) and q;
//   half 1: Gram rows R0..K-1. The solve runs in a second kernel (k_prep_solve),
//   one thread per sample.
#pragma once

#include "common.cuh"

namespace detnet {

template <int K> struct PrepSplit {
    static constexpr int NG = K * (K + 1) / 2;
    // first row index whose entries belong to half 1 (about half the entries)
    static constexpr int r0() {
        int acc = 0;
        for (int r = 0; r < K; ++r) {
            if (2 * (acc + (K - r)) > NG) return r == 0 ? 1 : r;
            acc += K - r;
        }
        return K;
    }
    static constexpr int R0 = r0();
    static constexpr int NA = [] {
        int a = 0;
        for (int r = 0; r < R0; ++r) a += K - r;
        return a;
    }();
    static constexpr int NB = NG - NA;
};

__host__ __device__ constexpr int tri_idx(int K, int a, int b) { // a <= b
    return a * K - a * (a - 1) / 2 + (b - a);
}

constexpr int PREP_FAST_SAMPLES = 64; // per CTA

// Shared-memory load that ptxas may not hoist or CSE: keeps the unrolled
// factor/solve loops from parking all 210 factor entries in registers.
__device__ __forceinline__ float lds_v(const float *p) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return v;
}

// K1a: Gram and q (FP32 accumulation) with two threads per sample.
template <int K>
__global__ void __launch_bounds__(128)
    k_prep_gram(long n, int N, const float *__restrict__ H, const float *__restrict__ y,
                const int8_t *__restrict__ x, float *__restrict__ gp, float *__restrict__ q32,
                uint32_t *__restrict__ xmask) {
    using S = PrepSplit<K>;
    constexpr int NG = S::NG, NA = S::NA, NB = S::NB, R0 = S::R0;
    constexpr int NMAX = NA > NB ? NA : NB;
    static_assert(K % 4 == 0, "rows are read as float4");
    const int half = threadIdx.x & 1;
    const int ls = threadIdx.x >> 1; // local sample
    const long s = static_cast<long>(blockIdx.x) * PREP_FAST_SAMPLES + ls;
    const bool live = s < n;
    const long sc = live ? s : n - 1;
    const long tile = sc / TILE;
    const int col = static_cast<int>(sc % TILE);
    const float4 *Hs = reinterpret_cast<const float4 *>(H + sc * static_cast<long>(N) * K);
    const float *ys = y + sc * N;
    const int8_t *xs = x + sc * K;

    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (xs[j] > 0) mask |= 1u << j;

    // ---- pass 1 over H: Gram halves and q (half 0), FP32 ----
    float acc[NMAX];
#pragma unroll
    for (int e = 0; e < NMAX; ++e) acc[e] = 0.f;
    float q[K];
#pragma unroll
    for (int j = 0; j < K; ++j) q[j] = 0.f;
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float h[K];
#pragma unroll
        for (int c = 0; c < K / 4; ++c) {
            const float4 v = __ldg(Hs + i * (K / 4) + c);
            h[4 * c] = v.x; h[4 * c + 1] = v.y; h[4 * c + 2] = v.z; h[4 * c + 3] = v.w;
        }
        if (half == 0) {
            const float yi = __ldg(ys + i);
            int e = 0;
#pragma unroll
            for (int a = 0; a < R0; ++a)
#pragma unroll
                for (int b = a; b < K; ++b, ++e) acc[e] = fmaf(h[a], h[b], acc[e]);
#pragma unroll
            for (int j = 0; j < K; ++j) q[j] = fmaf(h[j], yi, q[j]);
        } else {
            int e = 0;
#pragma unroll
            for (int a = R0; a < K; ++a)
#pragma unroll
                for (int b = a; b < K; ++b, ++e) acc[e] = fmaf(h[a], h[b], acc[e]);
        }
    }
    if (!live) return;
    {
        const int e0 = half == 0 ? 0 : NA;
        const int ne = half == 0 ? NA : NB;
#pragma unroll
        for (int e = 0; e < NMAX; ++e)
            if (e < ne) gp[(tile * NG + e0 + e) * TILE + col] = acc[e];
    }
    if (half == 0) {
#pragma unroll
        for (int j = 0; j < K; ++j) q32[(tile * K + j) * TILE + col] = q[j];
        xmask[s] = mask;
    }
}

// K1b: x_tilde via FP32 Cholesky in shared memory + FP64 refinement, one
// thread per sample; flags ill-conditioned samples for the exact LU.
template <int K>
__global__ void __launch_bounds__(PREP_FAST_SAMPLES)
    k_prep_solve(long n, int N, const float *__restrict__ H, const float *__restrict__ y,
                 const float *__restrict__ gp, const float *__restrict__ q32,
                 const uint32_t *__restrict__ xmask, double *__restrict__ denom,
                 uint8_t *__restrict__ flag, int *__restrict__ fb_count,
                 long *__restrict__ fb_list) {
    constexpr int NG = K * (K + 1) / 2;
    static_assert(K % 4 == 0, "rows are read as float4");
    extern __shared__ float gs_raw[]; // [NG][PREP_FAST_SAMPLES]
    float(*Gs)[PREP_FAST_SAMPLES] = reinterpret_cast<float(*)[PREP_FAST_SAMPLES]>(gs_raw);
    const int ls = threadIdx.x;
    const long s = static_cast<long>(blockIdx.x) * PREP_FAST_SAMPLES + ls;
    const bool live = s < n;
    const long sc = live ? s : n - 1;
    const long tile = sc / TILE;
    const int col = static_cast<int>(sc % TILE);
    const float4 *Hs = reinterpret_cast<const float4 *>(H + sc * static_cast<long>(N) * K);
    const float *ys = y + sc * N;
    const uint32_t mask = xmask[sc];
#pragma unroll 4
    for (int e = 0; e < NG; ++e) Gs[e][ls] = gp[(tile * NG + e) * TILE + col];
    __syncwarp();
    float r32[K]; // initial residual G x - q in FP32 (only a starting guess)
#pragma unroll
    for (int j = 0; j < K; ++j) r32[j] = -q32[(tile * K + j) * TILE + col];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = a; b < K; ++b) {
            const float g = lds_v(&Gs[tri_idx(K, a, b)][ls]);
            r32[a] = fmaf(g, (mask >> b) & 1u ? 1.f : -1.f, r32[a]);
            if (b != a) r32[b] = fmaf(g, (mask >> a) & 1u ? 1.f : -1.f, r32[b]);
        }

    // ---- FP32 Cholesky in place: L[i][j] (i > j) stored at Gs[tri(j, i)],
    // the diagonal holds 1 / L[j][j] ----
    bool bad = false;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        float sjj = lds_v(&Gs[tri_idx(K, j, j)][ls]);
        const float gjj = sjj;
#pragma unroll
        for (int k = 0; k < j; ++k) {
            const float l = lds_v(&Gs[tri_idx(K, k, j)][ls]);
            sjj = fmaf(-l, l, sjj);
        }
        if (!(sjj > 1e-5f * gjj)) bad = true;
        const float dinv = rsqrtf(fmaxf(sjj, 1e-30f));
        Gs[tri_idx(K, j, j)][ls] = dinv;
#pragma unroll 1
        for (int i = j + 1; i < K; ++i) {
            float sij = lds_v(&Gs[tri_idx(K, j, i)][ls]);
#pragma unroll
            for (int k = 0; k < j; ++k)
                sij = fmaf(-lds_v(&Gs[tri_idx(K, k, i)][ls]), lds_v(&Gs[tri_idx(K, k, j)][ls]), sij);
            Gs[tri_idx(K, j, i)][ls] = sij * dinv;
        }
    }
    // solve L L^T d = b (FP32)
    auto solve = [&](float (&b)[K]) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            float t = b[i];
#pragma unroll
            for (int k = 0; k < i; ++k) t = fmaf(-lds_v(&Gs[tri_idx(K, k, i)][ls]), b[k], t);
            b[i] = t * lds_v(&Gs[tri_idx(K, i, i)][ls]);
        }
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            float t = b[i];
#pragma unroll
            for (int k = i + 1; k < K; ++k) t = fmaf(-lds_v(&Gs[tri_idx(K, i, k)][ls]), b[k], t);
            b[i] = t * lds_v(&Gs[tri_idx(K, i, i)][ls]);
        }
    };
    solve(r32); // d0 = G^-1 (G x - q) = x - x_tilde (FP32 estimate)
    double xd[K]; // x - d = current x_tilde estimate
#pragma unroll
    for (int j = 0; j < K; ++j) xd[j] = ((mask >> j) & 1u ? 1.0 : -1.0) - static_cast<double>(r32[j]);
    // ---- refinement: res = H^T (H (x - d) - y) in FP64 from the FP32 inputs,
    // d <- d + G^-1 res; at most two steps ----
    double dn = 0.0;
    bool conv = false;
#pragma unroll 1
    for (int step = 0; step < 2 && !conv; ++step) {
        double res[K];
#pragma unroll
        for (int j = 0; j < K; ++j) res[j] = 0.0;
#pragma unroll 1
        for (int i = 0; i < N; ++i) {
            float h[K];
#pragma unroll
            for (int c = 0; c < K / 4; ++c) {
                const float4 v = __ldg(Hs + i * (K / 4) + c);
                h[4 * c] = v.x; h[4 * c + 1] = v.y; h[4 * c + 2] = v.z; h[4 * c + 3] = v.w;
            }
            double t = -static_cast<double>(__ldg(ys + i));
#pragma unroll
            for (int j = 0; j < K; ++j) t = fma(static_cast<double>(h[j]), xd[j], t);
#pragma unroll
            for (int j = 0; j < K; ++j) res[j] = fma(static_cast<double>(h[j]), t, res[j]);
        }
        float c32[K];
#pragma unroll
        for (int j = 0; j < K; ++j) c32[j] = static_cast<float>(res[j]);
        solve(c32);
        double cmax = 0.0, dmax = 0.0;
        dn = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            xd[j] -= static_cast<double>(c32[j]);
            const double dj = ((mask >> j) & 1u ? 1.0 : -1.0) - xd[j];
            dn = fma(dj, dj, dn);
            cmax = fmax(cmax, fabs(static_cast<double>(c32[j])));
            dmax = fmax(dmax, fabs(dj));
        }
        conv = cmax <= 1e-5 * dmax;
    }
    if (!conv || !(dn == dn)) bad = true;
    if (!live) return;
    if (bad) {
        // exact reference LU (and the singular test) for this sample
        const int slot = atomicAdd(fb_count, 1);
        fb_list[slot] = s;
        flag[s] = 0;
        denom[s] = 1.0;
    } else {
        flag[s] = dn < 1e-12 ? 1 : 0;
        denom[s] = dn < 1e-12 ? 1e-12 : dn;
    }
}

} // namespace detnet
