// k_preprocess.cuh -- K1 exact path: per-sample preprocessing, one warp per
// sample, bit-identical to the reference. Used for all samples when exact
// preprocessing is requested (and for dims without a fast path), and for the
// samples the fast path (k_prep_fast.cuh) flags as ill-conditioned.
//
// Restates the part of evaluate_one before the layer loop (kernels.cpp:55-58):
//   q = H^T y            matvec_transpose, linalg.cpp:20-29 (i outer)
//   G = H^T H            gram, linalg.cpp:31-42 (upper triangle, i ascending)
//   x_tilde = G^-1 q     solve_normal_equations, linalg.cpp:44-79
//   denom = max(||x - x_tilde||^2, 1e-12), flagged    loss.cpp:16-19
// in FP64 with the reference's operation order, so on FP32-representable
// inputs q, G, x_tilde and denom are bit-identical to the reference. (A
// product of two FP32 values is exact in FP64, so acc + a*b may use DFMA.)
// The layer stack consumes FP32 roundings of q and G.
//
// LU: warp_solve_normal below (one row per lane, parallel elimination).
//
// Optional FP64 outputs (the FP64 training mode, k_train64.cuh): g64 [s][K*K]
// and q64 [s][K], the reference's own G and q.
//
// Outputs (tile SoA, TILE samples per tile):
//   gp  [tile][K(K+1)/2][TILE]  packed upper triangle of G (row-major a<=b)
//   q32 [tile][K][TILE]
//   denom[s] (f64), xmask[s] (bit j set <=> x_j = +1), flag[s] (u8)
//   *singular = min sample index whose ZF pivot test failed (or unchanged)
#pragma once

#include "common.cuh"

namespace detnet {

// solve_normal_equations (linalg.cpp:44-79) on one warp: LU with partial
// pivoting of [G | q] in FP64 with the reference's operation order. Lane
// r < K owns row r in registers; row swaps are tracked as a position
// permutation (pos), reproducing the reference's first-strict-maximum pivot
// choice over positions. Returns true if the pivot test (<= 1e-12 max|G|)
// fails; otherwise xs (replicated on every lane) = G^-1 q.
template <int K>
__device__ __forceinline__ bool warp_solve_normal(const double *sG, const double *sq, int lane,
                                                  double (&xs)[K]) {
    constexpr unsigned FULL = 0xffffffffu;
    const bool rl = lane < K;
    double row[K + 1];
#pragma unroll
    for (int j = 0; j < K; ++j) row[j] = rl ? sG[lane * K + j] : 0.0;
    row[K] = rl ? sq[lane] : 0.0;
    double gmax = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) gmax = fmax(gmax, fabs(row[j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(FULL, gmax, o));
    const double tol = dmul(1e-12, gmax);

    int pos = rl ? lane : 1000 + lane;
#pragma unroll
    for (int cc = 0; cc < K; ++cc) {
        // pivot: max |A(p, cc)| over positions p >= cc, lowest position on ties
        double bv = (rl && pos >= cc) ? fabs(row[cc]) : -1.0;
        int bp = (rl && pos >= cc) ? pos : 1 << 20;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, bv, o);
            const int op = __shfl_xor_sync(FULL, bp, o);
            if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; }
        }
        if (bv <= tol) return true;
        const int pl = __ffs(__ballot_sync(FULL, pos == bp)) - 1;
        const int cl = __ffs(__ballot_sync(FULL, pos == cc)) - 1;
        if (lane == cl) pos = bp;
        if (lane == pl) pos = cc;
        double pr[K + 1];
#pragma unroll
        for (int j = cc; j <= K; ++j) pr[j] = __shfl_sync(FULL, row[j], pl);
        if (rl && pos > cc) {
            const double f = ddiv(row[cc], pr[cc]);
            if (f != 0.0) {
#pragma unroll
                for (int j = cc; j <= K; ++j) row[j] = dsub(row[j], dmul(f, pr[j]));
            }
        }
    }
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
        double acc = row[K];
#pragma unroll
        for (int j = i + 1; j < K; ++j) acc = dsub(acc, dmul(row[j], xs[j]));
        const double xi = ddiv(acc, row[i]);
        const int li = __ffs(__ballot_sync(FULL, pos == i)) - 1;
        xs[i] = __shfl_sync(FULL, xi, li);
    }
    return false;
}

template <int K>
__global__ void __launch_bounds__(256)
    k_preprocess(long n, int N, const float *__restrict__ H, const float *__restrict__ y,
                 const int8_t *__restrict__ x, float *__restrict__ gp, float *__restrict__ q32,
                 double *__restrict__ denom, uint32_t *__restrict__ xmask,
                 uint8_t *__restrict__ flag, unsigned long long *__restrict__ singular,
                 const long *__restrict__ list, const int *__restrict__ list_count,
                 double *__restrict__ g64 = nullptr, double *__restrict__ q64 = nullptr) {
    static_assert(K <= 32, "one lane per row");
    constexpr int NG = gram_entries(K);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    // per-warp scratch (doubles): H [N*K], y [N], G [K*K], q [K]
    const int per = N * K + N + K * K + K;
    double *sH = reinterpret_cast<double *>(smem_raw) + static_cast<size_t>(warp) * per;
    double *sy = sH + N * K;
    double *sG = sy + N;
    double *sq = sG + K * K;

    // optional index list: only the listed samples (the fast path's fallbacks)
    const long n_eff = list ? static_cast<long>(*list_count) : n;
    for (long si = static_cast<long>(blockIdx.x) * warps + warp; si < n_eff;
         si += static_cast<long>(gridDim.x) * warps) {
        const long s = list ? list[si] : si;
        DETNET_DASSERT(s >= 0 && s < n);
        const float *Hs = H + s * static_cast<long>(N) * K;
        for (int i = lane; i < N * K; i += 32) sH[i] = static_cast<double>(__ldg(Hs + i));
        for (int i = lane; i < N; i += 32) sy[i] = static_cast<double>(__ldg(y + s * N + i));
        __syncwarp();
        const long tile = s / TILE;
        const int col = static_cast<int>(s % TILE);

        if (lane < K) {
            double qj = 0.0;
            for (int i = 0; i < N; ++i) qj = fma(sH[i * K + lane], sy[i], qj);
            sq[lane] = qj;
            q32[(tile * K + lane) * TILE + col] = __double2float_rn(qj);
            if (q64) q64[s * K + lane] = qj;
        }
        for (int e = lane; e < NG; e += 32) {
            int a = 0, rem = e;
            while (rem >= K - a) { rem -= K - a; ++a; }
            const int b = a + rem;
            double acc = 0.0;
            for (int i = 0; i < N; ++i) acc = fma(sH[i * K + a], sH[i * K + b], acc);
            sG[a * K + b] = acc;
            sG[b * K + a] = acc;
            gp[(tile * NG + e) * TILE + col] = __double2float_rn(acc);
        }
        __syncwarp();
        if (g64) // FP64 training mode: the full Gram matrix, sample-major
            for (int e = lane; e < K * K; e += 32) g64[s * K * K + e] = sG[e];

        double xs[K];
        const bool sing = warp_solve_normal<K>(sG, sq, lane, xs);
        if (!sing) {
            if (lane == 0) {
                const int8_t *xv = x + s * K;
                uint32_t mask = 0;
                double dn = 0.0;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    const double df = dsub(static_cast<double>(xv[i]), xs[i]);
                    dn = dadd(dn, dmul(df, df));
                    if (xv[i] > 0) mask |= 1u << i;
                }
                flag[s] = dn < 1e-12 ? 1 : 0;
                denom[s] = dn < 1e-12 ? 1e-12 : dn;
                xmask[s] = mask;
            }
        } else if (lane == 0) {
            atomicMin(singular, static_cast<unsigned long long>(s));
            flag[s] = 0;
            denom[s] = 1.0;
            xmask[s] = 0;
        }
        __syncwarp();
    }
}

// Padding samples of the last tile: neutral values so the stack kernels can
// run full tiles without bounds checks on loads.
__global__ void k_pad_tail(long n, long n_pad, int K, float *gp, float *q32, double *denom,
                           uint32_t *xmask, uint8_t *flag) {
    const long s = n + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n_pad) return;
    const int NG = gram_entries(K);
    const long tile = s / TILE;
    const int col = static_cast<int>(s % TILE);
    for (int e = 0; e < NG; ++e) gp[(tile * NG + e) * TILE + col] = 0.f;
    for (int k = 0; k < K; ++k) q32[(tile * K + k) * TILE + col] = 0.f;
    denom[s] = 1.0;
    xmask[s] = 0;
    flag[s] = 0;
}

} // namespace detnet
