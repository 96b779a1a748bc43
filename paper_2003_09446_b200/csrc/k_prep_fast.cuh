// k_prep_fast.cuh -- K1 fast path: per-sample preprocessing with a pair of
// threads per sample (64 samples per 128-thread CTA).
//
// Computes what evaluate_one needs before the layer loop (kernels.cpp:55-58):
//   q = H^T y, G = H^T H                      -> FP32 outputs for the layer stack
//   d = x - x_tilde = G^-1 H^T (H x - y)      -> denom = max(||d||^2, 1e-12)
// Instead of the reference's FP64 LU (linalg.cpp:44-79, kept bit-exact in
// k_preprocess.cuh), the solve is an FP32 Cholesky in shared memory plus one
// step of iterative refinement whose residual H^T (H x - y) - H^T H d0 is
// formed in FP64 straight from the FP32 inputs (products exact in FP64), so
// d (hence the loss denominator) is FP64-accurate (~1e-10 relative) for
// well-conditioned samples. Samples whose Cholesky pivots collapse or whose
// refinement correction is not small are queued for the exact reference LU
// (k_preprocess on an index list), which also owns SingularMatrixError.
//
// Work split inside a pair (lanes 2i, 2i+1 = one sample; both stream the same
// H rows, so each 80-byte row is fetched once per pair):
//   half 0: Gram rows 0..R0-1 (upper-triangle entries [0, NA)), q (FP64), Cholesky,
//           solves, refinement;  half 1: Gram rows R0..K-1, r = H^T (H x - y).
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

template <int K>
__global__ void __launch_bounds__(128)
    k_prep_fast(long n, int N, const float *__restrict__ H, const float *__restrict__ y,
                const int8_t *__restrict__ x, float *__restrict__ gp, float *__restrict__ q32,
                double *__restrict__ denom, uint32_t *__restrict__ xmask,
                uint8_t *__restrict__ flag, int *__restrict__ fb_count,
                long *__restrict__ fb_list) {
    using S = PrepSplit<K>;
    constexpr int NG = S::NG, NA = S::NA, NB = S::NB, R0 = S::R0;
    constexpr int NMAX = NA > NB ? NA : NB;
    static_assert(K % 4 == 0, "rows are read as float4");
    extern __shared__ float gs_raw[]; // [NG][PREP_FAST_SAMPLES]
    float(*Gs)[PREP_FAST_SAMPLES] = reinterpret_cast<float(*)[PREP_FAST_SAMPLES]>(gs_raw);
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

    // ---- pass 1: Gram halves, q (half 0), r = H^T (H x - y) in FP64 (half 1)
    float acc[NMAX];
#pragma unroll
    for (int e = 0; e < NMAX; ++e) acc[e] = 0.f;
    // w: q (half 0) or r = H^T (H x - y) (half 1), both FP64 accumulators
    double w[K];
#pragma unroll
    for (int j = 0; j < K; ++j) w[j] = 0.0;
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float h[K];
#pragma unroll
        for (int c = 0; c < K / 4; ++c) {
            const float4 v = __ldg(Hs + i * (K / 4) + c);
            h[4 * c] = v.x; h[4 * c + 1] = v.y; h[4 * c + 2] = v.z; h[4 * c + 3] = v.w;
        }
        const float yi = __ldg(ys + i);
        if (half == 0) {
            int e = 0;
#pragma unroll
            for (int a = 0; a < R0; ++a)
#pragma unroll
                for (int b = a; b < K; ++b, ++e) acc[e] = fmaf(h[a], h[b], acc[e]);
#pragma unroll
            for (int j = 0; j < K; ++j) w[j] = fma(static_cast<double>(h[j]), static_cast<double>(yi), w[j]);
        } else {
            int e = 0;
#pragma unroll
            for (int a = R0; a < K; ++a)
#pragma unroll
                for (int b = a; b < K; ++b, ++e) acc[e] = fmaf(h[a], h[b], acc[e]);
            double ei = -static_cast<double>(yi);
#pragma unroll
            for (int j = 0; j < K; ++j) ei += (mask >> j) & 1u ? static_cast<double>(h[j]) : -static_cast<double>(h[j]);
#pragma unroll
            for (int j = 0; j < K; ++j) w[j] = fma(static_cast<double>(h[j]), ei, w[j]);
        }
    }
    // Gram entries -> shared (for the factorization) and global (layer stack)
    {
        const int e0 = half == 0 ? 0 : NA;
        const int ne = half == 0 ? NA : NB;
#pragma unroll
        for (int e = 0; e < NMAX; ++e)
            if (e < ne) {
                Gs[e0 + e][ls] = acc[e];
                if (live) gp[(tile * NG + e0 + e) * TILE + col] = acc[e];
            }
    }
    if (half == 0 && live) {
#pragma unroll
        for (int j = 0; j < K; ++j) q32[(tile * K + j) * TILE + col] = __double2float_rn(w[j]);
    }
    // r from the odd lane to the even lane of the pair
    double r[K];
#pragma unroll
    for (int j = 0; j < K; ++j) r[j] = __shfl_down_sync(0xffffffffu, w[j], 1);
    __syncthreads();
    if (half == 1) return;

    // ---- FP32 Cholesky in place: L[i][j] (i > j) stored at Gs[tri(j, i)],
    // the diagonal holds 1 / L[j][j] ----
    bool bad = false;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        float sjj = Gs[tri_idx(K, j, j)][ls];
        const float gjj = sjj;
#pragma unroll
        for (int k = 0; k < j; ++k) {
            const float l = Gs[tri_idx(K, k, j)][ls];
            sjj = fmaf(-l, l, sjj);
        }
        if (!(sjj > 1e-5f * gjj)) bad = true;
        const float dinv = rsqrtf(fmaxf(sjj, 1e-30f));
        Gs[tri_idx(K, j, j)][ls] = dinv;
#pragma unroll 1
        for (int i = j + 1; i < K; ++i) {
            float sij = Gs[tri_idx(K, j, i)][ls];
#pragma unroll
            for (int k = 0; k < j; ++k)
                sij = fmaf(-Gs[tri_idx(K, k, i)][ls], Gs[tri_idx(K, k, j)][ls], sij);
            Gs[tri_idx(K, j, i)][ls] = sij * dinv;
        }
    }
    // solve L L^T d = b (FP32)
    auto solve = [&](const float (&b)[K], float (&d)[K]) {
        float z[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            float t = b[i];
#pragma unroll
            for (int k = 0; k < i; ++k) t = fmaf(-Gs[tri_idx(K, k, i)][ls], z[k], t);
            z[i] = t * Gs[tri_idx(K, i, i)][ls];
        }
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            float t = z[i];
#pragma unroll
            for (int k = i + 1; k < K; ++k) t = fmaf(-Gs[tri_idx(K, i, k)][ls], d[k], t);
            d[i] = t * Gs[tri_idx(K, i, i)][ls];
        }
    };
    float b[K], d0[K];
#pragma unroll
    for (int j = 0; j < K; ++j) b[j] = static_cast<float>(r[j]);
    solve(b, d0);
    // ---- refinement: r <- r - H^T (H d0) in FP64 (the residual) ----
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float h[K];
#pragma unroll
        for (int c = 0; c < K / 4; ++c) {
            const float4 v = __ldg(Hs + i * (K / 4) + c);
            h[4 * c] = v.x; h[4 * c + 1] = v.y; h[4 * c + 2] = v.z; h[4 * c + 3] = v.w;
        }
        double f = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) f = fma(static_cast<double>(h[j]), static_cast<double>(d0[j]), f);
#pragma unroll
        for (int j = 0; j < K; ++j) r[j] = fma(-static_cast<double>(h[j]), f, r[j]);
    }
    float corr[K];
#pragma unroll
    for (int j = 0; j < K; ++j) b[j] = static_cast<float>(r[j]);
    solve(b, corr);
    double dn = 0.0, cmax = 0.0, dmax = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const double dj = static_cast<double>(d0[j]) + static_cast<double>(corr[j]);
        dn = fma(dj, dj, dn);
        cmax = fmax(cmax, fabs(static_cast<double>(corr[j])));
        dmax = fmax(dmax, fabs(dj));
    }
    if (!(cmax <= 1e-5 * dmax) || !(dn == dn)) bad = true;
    if (!live) return;
    xmask[s] = mask;
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
