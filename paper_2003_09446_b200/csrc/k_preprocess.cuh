// k_preprocess.cuh -- K1: per-sample preprocessing, one warp per sample.
//
// Restates the part of evaluate_one before the layer loop (kernels.cpp:55-58):
//   q = H^T y            matvec_transpose, linalg.cpp:20-29 (i outer)
//   G = H^T H            gram, linalg.cpp:31-42 (upper triangle, i ascending)
//   x_tilde = G^-1 q     solve_normal_equations, linalg.cpp:44-79
//   denom = max(||x - x_tilde||^2, 1e-12), flagged    loss.cpp:16-19
// all in FP64 with the reference's operation order and no FMA contraction,
// so on FP32-representable inputs q, G, x_tilde and denom are bit-identical
// to the reference. The layer stack consumes FP32 roundings of q and G.
//
// Outputs (tile SoA, TILE samples per tile):
//   gp  [tile][K(K+1)/2][TILE]  packed upper triangle of G (row-major a<=b)
//   q32 [tile][K][TILE]
//   denom[s] (f64), xmask[s] (bit j set <=> x_j = +1), flag[s] (u8)
//   *singular = min sample index whose ZF pivot test failed (or unchanged)
#pragma once

#include "common.cuh"

namespace detnet {

template <int K>
__global__ void __launch_bounds__(256)
    k_preprocess(long n, int N, const float *__restrict__ H, const float *__restrict__ y,
                 const int8_t *__restrict__ x, float *__restrict__ gp, float *__restrict__ q32,
                 double *__restrict__ denom, uint32_t *__restrict__ xmask,
                 uint8_t *__restrict__ flag, unsigned long long *__restrict__ singular) {
    static_assert(K + 1 <= 32, "one lane per column plus the right-hand side");
    constexpr int NG = gram_entries(K);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    // per-warp scratch: H (N*K floats), y (N floats), G (K*K doubles)
    const int hfl = round_up(N * K + N, 2);
    float *sH = reinterpret_cast<float *>(smem_raw) +
                static_cast<size_t>(warp) * (hfl + 2 * K * K);
    float *sy = sH + N * K;
    double *sG = reinterpret_cast<double *>(sH + hfl);

    for (long s = static_cast<long>(blockIdx.x) * warps + warp; s < n;
         s += static_cast<long>(gridDim.x) * warps) {
        const float *Hs = H + s * static_cast<long>(N) * K;
        for (int i = lane; i < N * K; i += 32) sH[i] = Hs[i];
        for (int i = lane; i < N; i += 32) sy[i] = y[s * N + i];
        __syncwarp();
        const long tile = s / TILE;
        const int col = static_cast<int>(s % TILE);

        // q_j (lane j), i ascending, from 0.0
        double qj = 0.0;
        if (lane < K) {
            for (int i = 0; i < N; ++i)
                qj = dadd(qj, dmul(static_cast<double>(sH[i * K + lane]),
                                   static_cast<double>(sy[i])));
            q32[(tile * K + lane) * TILE + col] = __double2float_rn(qj);
        }
        // G upper triangle, entries spread over lanes
        for (int e = lane; e < NG; e += 32) {
            int a = 0, rem = e;
            while (rem >= K - a) { rem -= K - a; ++a; }
            const int b = a + rem;
            double acc = 0.0;
            for (int i = 0; i < N; ++i)
                acc = dadd(acc, dmul(static_cast<double>(sH[i * K + a]),
                                     static_cast<double>(sH[i * K + b])));
            sG[a * K + b] = acc;
            sG[b * K + a] = acc;
            gp[(tile * NG + e) * TILE + col] = __double2float_rn(acc);
        }
        __syncwarp();

        // LU with partial pivoting: lane j < K owns column j, lane K the rhs.
        double c[K];
#pragma unroll
        for (int r = 0; r < K; ++r) {
            const double qr = __shfl_sync(0xffffffffu, qj, r);
            c[r] = lane < K ? sG[r * K + lane] : (lane == K ? qr : 0.0);
        }
        double gmax = 0.0;
        if (lane < K) {
#pragma unroll
            for (int r = 0; r < K; ++r) gmax = fmax(gmax, fabs(c[r]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
        const double tol = dmul(1e-12, gmax);
        bool sing = false;
#pragma unroll
        for (int cc = 0; cc < K; ++cc) {
            // pivot search in column cc (lane cc), first strict maximum
            int piv = cc;
            double best = fabs(c[cc]);
#pragma unroll
            for (int r = cc + 1; r < K; ++r) {
                const double v = fabs(c[r]);
                if (v > best) { best = v; piv = r; }
            }
            piv = __shfl_sync(0xffffffffu, piv, cc);
            best = __shfl_sync(0xffffffffu, best, cc);
            if (best <= tol) { sing = true; break; }
            if (piv != cc) {
#pragma unroll
                for (int r = cc + 1; r < K; ++r)
                    if (r == piv) { const double t = c[cc]; c[cc] = c[r]; c[r] = t; }
            }
            const double d = __shfl_sync(0xffffffffu, c[cc], cc);
#pragma unroll
            for (int r = cc + 1; r < K; ++r) {
                const double f = __shfl_sync(0xffffffffu, ddiv(c[r], d), cc);
                if (f == 0.0) continue;
                if (lane >= cc && lane <= K) c[r] = dsub(c[r], dmul(f, c[cc]));
            }
        }
        double dn = 0.0;
        if (!sing) {
            // back substitution on the rhs lane
#pragma unroll
            for (int i = K - 1; i >= 0; --i) {
                double acc = c[i];
#pragma unroll
                for (int j = i + 1; j < K; ++j) {
                    const double a = __shfl_sync(0xffffffffu, c[i], j);
                    acc = dsub(acc, dmul(a, c[j]));
                }
                const double aii = __shfl_sync(0xffffffffu, c[i], i);
                if (lane == K) c[i] = ddiv(acc, aii);
            }
            if (lane == K) {
                const int8_t *xs = x + s * K;
                uint32_t mask = 0;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    const double xv = static_cast<double>(xs[i]);
                    const double df = dsub(xv, c[i]);
                    dn = dadd(dn, dmul(df, df));
                    if (xs[i] > 0) mask |= 1u << i;
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

// Padding samples of the last tile: neutral values so the stack kernel can
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
