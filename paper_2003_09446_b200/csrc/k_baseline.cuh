// k_baseline.cuh -- SURVEY 8f row 4: the reference's detector baselines on the
// GPU, batch_baseline_errors (kernels.cpp:105-112, 202-223) with
//   ZF: sign_slice(solve_normal_equations(gram(H), matvec_transpose(H, y)))
//       (channel.cpp:34-36, 67-71; linalg.cpp:20-79)
//   ML: exhaustive search over {-1,+1}^K, first strict minimum of ||y - H s||^2
//       in ascending candidate order (channel.cpp:38-65), K <= 16.
// Inputs are the reference's own FP64 samples and every operation keeps the
// reference's order with separate multiply / add (the reference is compiled
// without FMA contraction), so decisions -- and the error counts -- are
// bit-identical to the reference, including near-zero ZF components and ML
// ties. One warp per sample; per-sample error counts, summed in sample order
// by the host.
#pragma once

#include "common.cuh"
#include "k_preprocess.cuh"

namespace detnet {

template <int K>
__global__ void __launch_bounds__(256)
    k_zf_errors(long n, int N, const double *__restrict__ H, const double *__restrict__ y,
                const double *__restrict__ x, int *__restrict__ errs,
                unsigned long long *__restrict__ singular) {
    static_assert(K <= 32, "one lane per row");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    const int per = N * K + N + K * K + K;
    double *sH = reinterpret_cast<double *>(smem_raw) + static_cast<size_t>(warp) * per;
    double *sy = sH + N * K;
    double *sG = sy + N;
    double *sq = sG + K * K;
    for (long s = static_cast<long>(blockIdx.x) * warps + warp; s < n;
         s += static_cast<long>(gridDim.x) * warps) {
        for (int i = lane; i < N * K; i += 32) sH[i] = H[s * N * K + i];
        for (int i = lane; i < N; i += 32) sy[i] = y[s * N + i];
        __syncwarp();
        if (lane < K) { // matvec_transpose: out[j] += row[j] * v[i], i ascending
            double qj = 0.0;
            for (int i = 0; i < N; ++i) qj = dadd(qj, dmul(sH[i * K + lane], sy[i]));
            sq[lane] = qj;
        }
        for (int e = lane; e < K * K; e += 32) { // gram: i ascending, mirrored
            const int a = e / K, b = e % K;
            if (b >= a) {
                double acc = 0.0;
                for (int i = 0; i < N; ++i) acc = dadd(acc, dmul(sH[i * K + a], sH[i * K + b]));
                sG[a * K + b] = acc;
                sG[b * K + a] = acc;
            }
        }
        __syncwarp();
        double xs[K];
        const bool sing = warp_solve_normal<K>(sG, sq, lane, xs);
        if (lane == 0) {
            if (sing) {
                atomicMin(singular, static_cast<unsigned long long>(s));
                errs[s] = 0;
            } else {
                int e = 0;
#pragma unroll
                for (int j = 0; j < K; ++j) e += (xs[j] >= 0.0 ? 1.0 : -1.0) != x[s * K + j];
                errs[s] = e;
            }
        }
        __syncwarp();
    }
}

template <int K>
__global__ void __launch_bounds__(256)
    k_ml_errors(long n, int N, const double *__restrict__ H, const double *__restrict__ y,
                const double *__restrict__ x, int *__restrict__ errs) {
    static_assert(K <= 16, "exhaustive search limited to K <= 16 (channel.cpp:41)");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    const int per = N * K + N;
    double *sH = reinterpret_cast<double *>(smem_raw) + static_cast<size_t>(warp) * per;
    double *sy = sH + N * K;
    constexpr uint32_t total = 1u << K;
    for (long s = static_cast<long>(blockIdx.x) * warps + warp; s < n;
         s += static_cast<long>(gridDim.x) * warps) {
        for (int i = lane; i < N * K; i += 32) sH[i] = H[s * N * K + i];
        for (int i = lane; i < N; i += 32) sy[i] = y[s * N + i];
        __syncwarp();
        // each lane scans m = lane, lane + 32, ... ascending and keeps its first
        // strict minimum; the warp then keeps the smallest metric, lowest m on
        // ties -- the reference's "first strict minimum" over ascending m.
        double best = 0.0;
        uint32_t bm = 0xffffffffu;
        for (uint32_t m = lane; m < total; m += 32) {
            double metric = 0.0;
            for (int i = 0; i < N; ++i) {
                double r = sy[i];
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const double c = ((m >> (K - 1 - j)) & 1u) ? 1.0 : -1.0;
                    r = dsub(r, dmul(sH[i * K + j], c));
                }
                metric = dadd(metric, dmul(r, r));
            }
            if (bm == 0xffffffffu || metric < best) { best = metric; bm = m; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t om = __shfl_xor_sync(0xffffffffu, bm, o);
            if (om != 0xffffffffu && (bm == 0xffffffffu || ob < best || (ob == best && om < bm))) {
                best = ob;
                bm = om;
            }
        }
        if (lane == 0) {
            int e = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) e += (((bm >> (K - 1 - j)) & 1u) ? 1.0 : -1.0) != x[s * K + j];
            errs[s] = e;
        }
        __syncwarp();
    }
}

} // namespace detnet
