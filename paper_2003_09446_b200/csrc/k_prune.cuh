// k_prune.cuh -- SURVEY 8f row 3: the reference's pruning planner on the
// device-resident FP64 master weights (compression.cpp:43-94):
//   group:   per matrix W (W1, W2, W3) with bias b, column norms of the RAW W
//            (i ascending) and ||b||; columns (and the bias) whose norm is
//            < eta1 * max norm get their mask zeroed  (prune_group_matrix)
//   element: threshold = eta * max |W| over unmasked entries of W1, W2, W3;
//            unmasked entries with |W| < threshold are masked (prune_element)
//   sparse_group = group(eta1) then element(eta2)
// in the reference's FP64 operation order (separate multiply / add, correctly
// rounded sqrt; maxima are order independent), so masks are bit-identical.
// One CTA per layer over the layer-record layout (W1 b1 W2 b2 W3 b3 t).
#pragma once

#include "common.cuh"

namespace detnet {

struct PruneArgs {
    double *params, *masks; // [L][P]
    long P;
    int K, Z, V;
    int kind; // 0 element, 1 group, 2 sparse_group
    double eta, eta1, eta2;
};

__device__ inline double block_max(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double m = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmax(m, red[i]);
    return m;
}

// prune_group_matrix on one (W rows x cols, b) block of a record
__device__ inline void group_matrix(const double *W, double *M, const double *b, double *mb,
                                    int rows, int cols, double eta1, double *norms, double *red) {
    for (int j = threadIdx.x; j <= cols; j += blockDim.x) {
        double sq = 0.0;
        if (j < cols) {
            for (int i = 0; i < rows; ++i) sq = dadd(sq, dmul(W[i * cols + j], W[i * cols + j]));
        } else {
            for (int i = 0; i < rows; ++i) sq = dadd(sq, dmul(b[i], b[i]));
        }
        norms[j] = __dsqrt_rn(sq);
    }
    __syncthreads();
    double m = 0.0;
    for (int j = threadIdx.x; j <= cols; j += blockDim.x) m = fmax(m, norms[j]);
    const double threshold = dmul(eta1, block_max(m, red));
    for (int e = threadIdx.x; e < rows * cols; e += blockDim.x)
        if (norms[e % cols] < threshold) M[e] = 0.0;
    if (norms[cols] < threshold)
        for (int i = threadIdx.x; i < rows; i += blockDim.x) mb[i] = 0.0;
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_prune(PruneArgs a) {
    __shared__ double norms[1024];
    __shared__ double red[32];
    const int K = a.K, Z = a.Z, V = a.V, IN = 3 * K + V;
    double *p = a.params + blockIdx.x * a.P, *mk = a.masks + blockIdx.x * a.P;
    const long oW1 = 0, ob1 = static_cast<long>(Z) * IN, oW2 = ob1 + Z,
               ob2 = oW2 + static_cast<long>(K) * Z, oW3 = ob2 + K,
               ob3 = oW3 + static_cast<long>(V) * Z;
    if (a.kind != 0) {
        group_matrix(p + oW1, mk + oW1, p + ob1, mk + ob1, Z, IN, a.eta1, norms, red);
        group_matrix(p + oW2, mk + oW2, p + ob2, mk + ob2, K, Z, a.eta1, norms, red);
        group_matrix(p + oW3, mk + oW3, p + ob3, mk + ob3, V, Z, a.eta1, norms, red);
    }
    if (a.kind != 1) {
        const double eta = a.kind == 0 ? a.eta : a.eta2;
        double m = 0.0;
        auto scan = [&](long off, long cnt) {
            for (long e = threadIdx.x; e < cnt; e += blockDim.x)
                if (mk[off + e] != 0.0) m = fmax(m, fabs(p[off + e]));
        };
        scan(oW1, static_cast<long>(Z) * IN);
        scan(oW2, static_cast<long>(K) * Z);
        scan(oW3, static_cast<long>(V) * Z);
        const double threshold = dmul(eta, block_max(m, red));
        auto cut = [&](long off, long cnt) {
            for (long e = threadIdx.x; e < cnt; e += blockDim.x)
                if (mk[off + e] != 0.0 && fabs(p[off + e]) < threshold) mk[off + e] = 0.0;
        };
        cut(oW1, static_cast<long>(Z) * IN);
        cut(oW2, static_cast<long>(K) * Z);
        cut(oW3, static_cast<long>(V) * Z);
    }
}

} // namespace detnet
