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

// ZF for any K (the register-resident k_zf_errors above is instantiated for
// K <= 20): one warp per sample, the elimination matrix [A | x] in the warp's
// shared-memory slot, H and y read from global memory. Same operation order
// as the reference: matvec_transpose and gram accumulate over i ascending;
// the pivot is the first strict maximum of |A(r, col)| for r >= col (lanes
// scan strided rows, ties resolved to the lowest row); rows are swapped
// physically; each row r > col is eliminated by one lane in the reference's
// j order (f == 0 rows skipped); back substitution runs on lane 0.
__global__ void __launch_bounds__(128)
    k_zf_errors_any(long n, int N, int K, const double *__restrict__ H,
                    const double *__restrict__ y, const double *__restrict__ x,
                    int *__restrict__ errs, unsigned long long *__restrict__ singular) {
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    const int K1 = K + 1; // row stride: [A(r, 0..K-1) | x_r]
    double *sA = reinterpret_cast<double *>(smem_raw) + static_cast<size_t>(warp) * K * K1;
    for (long s = static_cast<long>(blockIdx.x) * warps + warp; s < n;
         s += static_cast<long>(gridDim.x) * warps) {
        const double *Hs = H + s * static_cast<long>(N) * K;
        const double *ys = y + s * static_cast<long>(N);
        for (int j = lane; j < K; j += 32) { // matvec_transpose (linalg.cpp:20-29)
            double qj = 0.0;
            for (int i = 0; i < N; ++i) qj = dadd(qj, dmul(Hs[i * K + j], ys[i]));
            sA[j * K1 + K] = qj;
        }
        for (int e = lane; e < K * K; e += 32) { // gram (linalg.cpp:31-42), mirrored
            const int a = e / K, b = e % K;
            if (b >= a) {
                double acc = 0.0;
                for (int i = 0; i < N; ++i) acc = dadd(acc, dmul(Hs[i * K + a], Hs[i * K + b]));
                sA[a * K1 + b] = acc;
                sA[b * K1 + a] = acc;
            }
        }
        __syncwarp();
        double gmax = 0.0;
        for (int e = lane; e < K * K; e += 32) gmax = fmax(gmax, fabs(sA[(e / K) * K1 + e % K]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(FULL, gmax, o));
        const double tol = dmul(1e-12, gmax);
        bool sing = false;
        for (int col = 0; col < K && !sing; ++col) { // solve_normal_equations (linalg.cpp:44-79)
            double bv = -1.0;
            int bp = 1 << 30;
            for (int r = col + lane; r < K; r += 32) {
                const double a = fabs(sA[r * K1 + col]);
                if (a > bv) { bv = a; bp = r; } // ascending r: first strict maximum
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(FULL, bv, o);
                const int op = __shfl_xor_sync(FULL, bp, o);
                if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; }
            }
            if (bv <= tol) { sing = true; break; }
            if (bp != col)
                for (int j = lane; j < K1; j += 32) {
                    const double t = sA[col * K1 + j];
                    sA[col * K1 + j] = sA[bp * K1 + j];
                    sA[bp * K1 + j] = t;
                }
            __syncwarp();
            const double d = sA[col * K1 + col];
            for (int r = col + 1 + lane; r < K; r += 32) {
                const double f = ddiv(sA[r * K1 + col], d);
                if (f == 0.0) continue;
                for (int j = col; j < K; ++j) sA[r * K1 + j] = dsub(sA[r * K1 + j], dmul(f, sA[col * K1 + j]));
                sA[r * K1 + K] = dsub(sA[r * K1 + K], dmul(f, sA[col * K1 + K]));
            }
            __syncwarp();
        }
        if (lane == 0) {
            if (sing) {
                atomicMin(singular, static_cast<unsigned long long>(s));
                errs[s] = 0;
            } else {
                int e = 0;
                for (int i = K - 1; i >= 0; --i) { // back substitution, x[i] kept in column K
                    double acc = sA[i * K1 + K];
                    for (int j = i + 1; j < K; ++j) acc = dsub(acc, dmul(sA[i * K1 + j], sA[j * K1 + K]));
                    const double xi = ddiv(acc, sA[i * K1 + i]);
                    sA[i * K1 + K] = xi;
                    e += (xi >= 0.0 ? 1.0 : -1.0) != x[s * K + i];
                }
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
