// k_train64.cuh -- the FP64 training step in the reference's operation order
// (detnet_ctx_set_train_precision(ctx, 1)): on FP32-representable samples its
// batch_gradient is bit-identical to the reference's (kernels.cpp:160-200),
// so a training run on the GPU follows the reference's own trajectory.
//
// Every floating-point operation below is the reference's, in its order, with
// separate IEEE multiply / add / divide (dmul/dadd/..., no FMA contraction):
//   forward_pre      model.cpp:84-122 (matvec linalg.cpp:8-18, masked_affine
//                    model.cpp:58-80 with W (.) M and b (.) mb formed first,
//                    relu :28-31, soft_sign :33-43)
//   loss_plain       loss.cpp:9-31
//   backward_data    backward.cpp:105-165 (masked_transpose_apply :32-43,
//                    accumulate_outer :21-29, soft_sign_du/dt model.cpp:45-51)
//   batch_gradient   kernels.cpp:160-200: min(16, n) index-contiguous blocks,
//                    each accumulating its samples' gradients in index order,
//                    blocks merged in block order (then x 1/n, regularizer and
//                    Adam in k_train.cuh, already bit-exact).
// Preprocessing (q, G, x_tilde, denom) is k_preprocess's exact LU, which is
// bit-identical to linalg.cpp:20-79 on FP32-representable inputs.
//
// Layout: one warp per sample for the forward and the reverse sweep (lanes
// over the hidden units / outputs of each dot product; every dot product is
// one lane's sequential chain, exactly the reference's loop), traces and
// adjoints sample-major per layer ([l][s][feature], FP64). The weight
// gradients are then batch contractions done per (block, output entry) as a
// sequential sum over the block's samples -- the reference's accumulation
// order -- on 32x32 output tiles staged through shared memory.
#pragma once

#include "common.cuh"

namespace detnet {

// Per-layer FP64 images built from the master params and masks:
//  wb [L][P]  : the record with W (.) M and b (.) mb (t unmasked) -- what the
//               reverse sweep reads row-major (masked_transpose_apply)
//  wf [L][PF] : forward images W1m^T [IN][Z], [W2m; W3m]^T [Z][K+V],
//               b1m [Z], [b2m; b3m] [K+V], t
__host__ __device__ inline long f64_fwd_rec(int K, int Z, int V) {
    const long IN = 3L * K + V;
    return IN * Z + static_cast<long>(Z) * (K + V) + Z + (K + V) + 1;
}

__global__ void k_pack64(const double *params, const double *masks, int K, int Z, int V, int L,
                         double *wb, double *wf) {
    const int IN = 3 * K + V, O = K + V;
    const long P = static_cast<long>(Z) * IN + Z + static_cast<long>(K) * Z + K +
                   static_cast<long>(V) * Z + V + 1;
    const long PF = f64_fwd_rec(K, Z, V);
    const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long>(L) * P) return;
    const int l = static_cast<int>(idx / P);
    const long e = idx % P;
    const long oW1 = 0, ob1 = static_cast<long>(Z) * IN, oW2 = ob1 + Z,
               ob2 = oW2 + static_cast<long>(K) * Z, oW3 = ob2 + K,
               ob3 = oW3 + static_cast<long>(V) * Z, ot = ob3 + V;
    const double p = params[idx];
    const double wm = e == ot ? p : dmul(p, masks ? masks[idx] : 1.0);
    wb[idx] = wm;
    double *f = wf + static_cast<long>(l) * PF;
    const long fW23 = static_cast<long>(IN) * Z, fb1 = fW23 + static_cast<long>(Z) * O,
               fb23 = fb1 + Z, ft = fb23 + O;
    if (e < ob1) {
        const long i = (e - oW1) / IN, j = (e - oW1) % IN;
        f[j * Z + i] = wm;
    } else if (e < oW2) {
        f[fb1 + (e - ob1)] = wm;
    } else if (e < ob2) {
        const long k = (e - oW2) / Z, i = (e - oW2) % Z;
        f[fW23 + i * O + k] = wm;
    } else if (e < oW3) {
        f[fb23 + (e - ob2)] = wm;
    } else if (e < ob3) {
        const long v = (e - oW3) / Z, i = (e - oW3) % Z;
        f[fW23 + i * O + K + v] = wm;
    } else if (e < ot) {
        f[fb23 + K + (e - ob3)] = wm;
    } else {
        f[ft] = p;
    }
}

struct Fwd64Args {
    const double *g64;      // [s][K*K] Gram matrices (exact preprocessing)
    const double *q64;      // [s][K]
    const double *denom;    // [s]
    const uint32_t *xmask;  // [s] bit i <=> x_i = +1
    const double *wf;       // [L][PF]
    const double *lnk;      // [L] ln(l+1) (host std::log, as loss.cpp:28)
    int K, Z, V, L;
    int first_term;         // loss terms k = first_term..L (kernels.cpp:69-71)
    long n;
    double *tr_in, *tr_z, *tr_u2, *tr_xh; // [L][n][IN|Z|K|K]
    double *loss;           // [n]
    long long *err;         // [n]
};

constexpr int F64_WARPS = 8;

// per-warp shared scratch (doubles): G [K][K+1], in [IN], z [Z]
__host__ __device__ inline int f64_fwd_scratch(int K, int Z, int V) {
    return K * (K + 1) + 3 * K + V + Z;
}

// forward_pre + loss_plain + the error count of one sample per warp
__global__ void __launch_bounds__(32 * F64_WARPS) k_fwd64(Fwd64Args a) {
    extern __shared__ double sm64[];
    const int K = a.K, Z = a.Z, V = a.V, IN = 3 * K + V, O = K + V, KP = K + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long s = static_cast<long>(blockIdx.x) * F64_WARPS + warp;
    if (s >= a.n) return;
    DETNET_DASSERT(K <= 32 && Z <= 256 && V <= 64 && a.first_term >= 1);
    double *sG = sm64 + static_cast<long>(warp) * f64_fwd_scratch(K, Z, V);
    double *sin = sG + K * KP;
    double *sz = sin + IN;
    const long PF = f64_fwd_rec(K, Z, V);
    for (int e = lane; e < K * K; e += 32) sG[(e / K) * KP + e % K] = a.g64[s * K * K + e];
    for (int j = lane; j < IN; j += 32) sin[j] = j < K ? a.q64[s * K + j] : 0.0; // x_hat_0 = 0, v_0 = 0
    const uint32_t xm = a.xmask[s];
    const double dn = a.denom[s];
    double loss = 0.0;
    __syncwarp();
    for (int l = 0; l < a.L; ++l) {
        const double *f = a.wf + static_cast<long>(l) * PF;
        const double *W1T = f, *W23T = f + static_cast<long>(IN) * Z, *b1 = W23T + static_cast<long>(Z) * O,
                     *b23 = b1 + Z;
        const double t = f[PF - 1];
        // gx = G x_hat (matvec: acc from 0, j ascending)
        if (lane < K) {
            double acc = 0.0;
            for (int j = 0; j < K; ++j) acc = dadd(acc, dmul(sG[lane * KP + j], sin[K + j]));
            sin[2 * K + lane] = acc;
        }
        __syncwarp();
        double *tin = a.tr_in + (static_cast<long>(l) * a.n + s) * IN;
        for (int j = lane; j < IN; j += 32) tin[j] = sin[j];
        // u1 = (W1 (.) M1) in + b1 (.) mb1; z = relu(u1)
        double *tz = a.tr_z + (static_cast<long>(l) * a.n + s) * Z;
        for (int i0 = 0; i0 < Z; i0 += 128) {
            double acc[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = i0 + lane + 32 * r;
                acc[r] = i < Z ? __ldg(b1 + i) : 0.0;
            }
            for (int j = 0; j < IN; ++j) {
                const double xj = sin[j];
                const double *col = W1T + static_cast<long>(j) * Z;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = i0 + lane + 32 * r;
                    if (i < Z) acc[r] = dadd(acc[r], dmul(__ldg(col + i), xj));
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = i0 + lane + 32 * r;
                if (i < Z) {
                    const double zi = acc[r] > 0.0 ? acc[r] : 0.0;
                    sz[i] = zi;
                    tz[i] = zi;
                }
            }
        }
        __syncwarp();
        // [u2; v] = [W2m; W3m] z + [b2m; b3m]
        double out[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) out[r] = (lane + 32 * r < O) ? __ldg(b23 + lane + 32 * r) : 0.0;
        for (int i = 0; i < Z; ++i) {
            const double zi = sz[i];
            const double *row = W23T + static_cast<long>(i) * O;
#pragma unroll
            for (int r = 0; r < 2; ++r)
                if (lane + 32 * r < O) out[r] = dadd(out[r], dmul(__ldg(row + lane + 32 * r), zi));
        }
        double *tu2 = a.tr_u2 + (static_cast<long>(l) * a.n + s) * K;
        double *txh = a.tr_xh + (static_cast<long>(l) * a.n + s) * K;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int o = lane + 32 * r;
            if (o < K) {
                const double u = out[r];
                tu2[o] = u;
                const double xo = u <= -t ? -1.0 : (u >= t ? 1.0 : ddiv(u, t));
                txh[o] = xo;
                sin[K + o] = xo;
            } else if (o < O) {
                sin[3 * K + (o - K)] = out[r];
            }
        }
        __syncwarp();
        // loss_plain term k = l + 1 (sequential over i, as loss.cpp:23-28)
        if (lane == 0 && l + 1 >= a.first_term) {
            double e2 = 0.0;
            for (int i = 0; i < K; ++i) {
                const double d = dsub((xm >> i) & 1u ? 1.0 : -1.0, sin[K + i]);
                e2 = dadd(e2, dmul(d, d));
            }
            loss = dadd(loss, ddiv(dmul(a.lnk[l], e2), dn));
        }
        __syncwarp();
    }
    // hard decision x_hat_L >= 0 -> +1 (kernels.cpp:63-65)
    const bool wrong = lane < K && ((sin[K + lane] >= 0.0) != (((xm >> lane) & 1u) != 0));
    const unsigned bad = __ballot_sync(0xffffffffu, wrong);
    if (lane == 0) {
        a.loss[s] = loss;
        a.err[s] = __popc(bad);
    }
}

struct Bwd64Args {
    const double *g64, *denom;
    const uint32_t *xmask;
    const double *wb;       // [L][P] masked records
    const double *lnk;      // [L] ln(l+1)
    int K, Z, V, L, lf;
    long n;
    const double *tr_in, *tr_z, *tr_u2, *tr_xh;
    double *u1bar;          // [L][n][Z]
    double *u2bar;          // [L][n][K]
    double *vbar;           // [L][n][V]  (v_bar entering layer l)
    double *tbar;           // [L][n]
};

// per-warp scratch: G [K][K+1], a_bar [K], v_bar [V], u2_bar [K], t terms [K],
// u1_bar [Z], in_bar [IN]
__host__ __device__ inline int f64_bwd_scratch(int K, int Z, int V) {
    return K * (K + 1) + K + V + K + K + Z + 3 * K + V;
}

// backward_data (backward.cpp:105-165), one sample per warp
__global__ void __launch_bounds__(32 * F64_WARPS) k_bwd64(Bwd64Args a) {
    extern __shared__ double sm64[];
    const int K = a.K, Z = a.Z, V = a.V, IN = 3 * K + V, KP = K + 1;
    const long P = static_cast<long>(Z) * IN + Z + static_cast<long>(K) * Z + K +
                   static_cast<long>(V) * Z + V + 1;
    const long oW2 = static_cast<long>(Z) * IN + Z, oW3 = oW2 + static_cast<long>(K) * Z + K;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long s = static_cast<long>(blockIdx.x) * F64_WARPS + warp;
    if (s >= a.n) return;
    double *sG = sm64 + static_cast<long>(warp) * f64_bwd_scratch(K, Z, V);
    double *sa = sG + K * KP, *sv = sa + K, *su2 = sv + V, *sdt = su2 + K, *su1 = sdt + K,
           *sib = su1 + Z;
    for (int e = lane; e < K * K; e += 32) sG[(e / K) * KP + e % K] = a.g64[s * K * K + e];
    for (int k = lane; k < K; k += 32) sa[k] = 0.0;
    for (int k = lane; k < V; k += 32) sv[k] = 0.0;
    const uint32_t xm = a.xmask[s];
    const double dn = a.denom[s];
    __syncwarp();
    for (int l = a.L - 1; l >= a.lf; --l) {
        const double *wl = a.wb + static_cast<long>(l) * P;
        const double *W1 = wl, *W2 = wl + oW2, *W3 = wl + oW3;
        const double t = wl[P - 1];
        const long ls = static_cast<long>(l) * a.n + s;
        // a_bar += w (x_hat_{l+1} - x), w = 2 ln(l+1) / denom
        const double w = ddiv(dmul(2.0, a.lnk[l]), dn);
        for (int i = lane; i < K; i += 32) {
            const double xi = (xm >> i) & 1u ? 1.0 : -1.0;
            const double ab = dadd(sa[i], dmul(w, dsub(a.tr_xh[ls * K + i], xi)));
            sa[i] = ab;
            const double u = a.tr_u2[ls * K + i];
            const bool lin = u >= -t && u < t;
            const double ub = dmul(ab, lin ? ddiv(1.0, t) : 0.0);
            su2[i] = ub;
            a.u2bar[ls * K + i] = ub;
            sdt[i] = dmul(ab, lin ? ddiv(-u, dmul(t, t)) : 0.0);
        }
        for (int k = lane; k < V; k += 32) a.vbar[ls * V + k] = sv[k];
        __syncwarp();
        if (lane == 0) {
            double tb = 0.0;
            for (int i = 0; i < K; ++i) tb = dadd(tb, sdt[i]);
            a.tbar[ls] = tb;
        }
        // z_bar = (W2 (.) M2)^T u2_bar + (W3 (.) M3)^T v_bar; u1_bar = z_bar [u1 > 0]
        const double *zl = a.tr_z + ls * Z;
        for (int i0 = 0; i0 < Z; i0 += 128) {
            double z2[4], z3[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) z2[r] = z3[r] = 0.0;
            for (int k = 0; k < K; ++k) {
                const double u = su2[k];
                if (u == 0.0) continue;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = i0 + lane + 32 * r;
                    if (i < Z) z2[r] = dadd(z2[r], dmul(__ldg(W2 + static_cast<long>(k) * Z + i), u));
                }
            }
            for (int k = 0; k < V; ++k) {
                const double u = sv[k];
                if (u == 0.0) continue;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = i0 + lane + 32 * r;
                    if (i < Z) z3[r] = dadd(z3[r], dmul(__ldg(W3 + static_cast<long>(k) * Z + i), u));
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = i0 + lane + 32 * r;
                if (i < Z) {
                    const double ub = zl[i] > 0.0 ? dadd(z2[r], z3[r]) : 0.0;
                    su1[i] = ub;
                    a.u1bar[ls * Z + i] = ub;
                }
            }
        }
        __syncwarp();
        // in_bar = (W1 (.) M1)^T u1_bar for the x, Gx and v blocks (q is data)
        for (int j0 = K; j0 < IN; j0 += 96) {
            double acc[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) acc[r] = 0.0;
            for (int i = 0; i < Z; ++i) {
                const double u = su1[i];
                if (u == 0.0) continue;
                const double *row = W1 + static_cast<long>(i) * IN;
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const int j = j0 + lane + 32 * r;
                    if (j < IN) acc[r] = dadd(acc[r], dmul(__ldg(row + j), u));
                }
            }
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const int j = j0 + lane + 32 * r;
                if (j < IN) sib[j] = acc[r];
            }
        }
        __syncwarp();
        // a_bar <- G gx_bar + x_bar; v_bar <- v block
        for (int i = lane; i < K; i += 32) {
            double acc = 0.0;
            for (int j = 0; j < K; ++j) acc = dadd(acc, dmul(sG[i * KP + j], sib[2 * K + j]));
            sa[i] = dadd(acc, sib[K + i]);
        }
        for (int k = lane; k < V; k += 32) sv[k] = sib[3 * K + k];
        __syncwarp();
    }
}

// Weight-gradient block partials: part[b][l][e] = the reference's per-block
// accumulation of entry e over block b's samples in index order,
//   W: acc += (A_s[i] * B_s[j]) * M[i][j]   (accumulate_outer)
//   b: acc += A_s[i] * mb[i]
// Jobs: (layer, which) with which 0 = W1/b1 (A = u1_bar, B = in), 1 = W2/b2
// (A = u2_bar, B = z), 2 = W3/b3 (A = v_bar, B = z).
struct Dw64Args {
    const double *u1bar, *u2bar, *vbar, *tr_in, *tr_z;
    const double *masks;   // [L][P] or null (all ones)
    int K, Z, V, L, lf;
    long n;
    int nblocks;           // min(16, n)
    double *part;          // [nblocks][L][P]
};

constexpr int DW64_T = 32;

// grid: (N tiles incl. the bias column, M tiles, (layer - lf) * 3 * nblocks)
__global__ void __launch_bounds__(256) k_dw64(Dw64Args a) {
    __shared__ double sA[DW64_T][DW64_T + 1], sB[DW64_T][DW64_T + 1];
    const int K = a.K, Z = a.Z, V = a.V, IN = 3 * K + V;
    const long P = static_cast<long>(Z) * IN + Z + static_cast<long>(K) * Z + K +
                   static_cast<long>(V) * Z + V + 1;
    const int nb = a.nblocks;
    const int job = blockIdx.z / nb, blk = blockIdx.z % nb;
    const int l = a.lf + job / 3, which = job % 3;
    int M, NN, Astride, Bstride;
    const double *A, *B;
    long oW, ob;
    const long ls0 = static_cast<long>(l) * a.n;
    if (which == 0) {
        M = Z; NN = IN; A = a.u1bar + ls0 * Z; Astride = Z; B = a.tr_in + ls0 * IN; Bstride = IN;
        oW = 0; ob = static_cast<long>(Z) * IN;
    } else if (which == 1) {
        M = K; NN = Z; A = a.u2bar + ls0 * K; Astride = K; B = a.tr_z + ls0 * Z; Bstride = Z;
        oW = static_cast<long>(Z) * IN + Z; ob = oW + static_cast<long>(K) * Z;
    } else {
        M = V; NN = Z; A = a.vbar + ls0 * V; Astride = V; B = a.tr_z + ls0 * Z; Bstride = Z;
        oW = static_cast<long>(Z) * IN + Z + static_cast<long>(K) * Z + K; ob = oW + static_cast<long>(V) * Z;
    }
    const int m0 = blockIdx.y * DW64_T, n0 = blockIdx.x * DW64_T;
    if (m0 >= M || n0 > NN) return;
    const long lo = a.n * blk / nb, hi = a.n * (blk + 1) / nb;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const double *mk = a.masks ? a.masks + static_cast<long>(l) * P : nullptr;
    double c[2][2], mm[2][2];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            c[p][q] = 0.0;
            const int i = m0 + ty * 2 + p, j = n0 + tx * 2 + q;
            double m = 1.0;
            if (mk && i < M && j <= NN) m = j < NN ? mk[oW + static_cast<long>(i) * NN + j] : mk[ob + i];
            mm[p][q] = m;
        }
    for (long c0 = lo; c0 < hi; c0 += DW64_T) {
        __syncthreads();
        for (int e = threadIdx.x; e < DW64_T * DW64_T; e += 256) {
            const int ss = e / DW64_T, col = e % DW64_T;
            const long sidx = c0 + ss;
            const bool in = sidx < hi;
            sA[ss][col] = (in && m0 + col < M) ? A[sidx * Astride + m0 + col] : 0.0;
            const int j = n0 + col;
            sB[ss][col] = (in && j < NN) ? B[sidx * Bstride + j] : 1.0; // bias column: B = 1
        }
        __syncthreads();
        const int cnt = static_cast<int>(hi - c0 < DW64_T ? hi - c0 : DW64_T);
        for (int ss = 0; ss < cnt; ++ss) {
            const double a0 = sA[ss][ty * 2], a1 = sA[ss][ty * 2 + 1];
            const double b0 = sB[ss][tx * 2], b1 = sB[ss][tx * 2 + 1];
            c[0][0] = dadd(c[0][0], dmul(dmul(a0, b0), mm[0][0]));
            c[0][1] = dadd(c[0][1], dmul(dmul(a0, b1), mm[0][1]));
            c[1][0] = dadd(c[1][0], dmul(dmul(a1, b0), mm[1][0]));
            c[1][1] = dadd(c[1][1], dmul(dmul(a1, b1), mm[1][1]));
        }
    }
    double *out = a.part + (static_cast<long>(blk) * a.L + l) * P;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int i = m0 + ty * 2 + p, j = n0 + tx * 2 + q;
            if (i >= M || j > NN) continue;
            // bias: acc += u_bar * mb (the A * 1.0 above is exact)
            out[j < NN ? oW + static_cast<long>(i) * NN + j : ob + i] = c[p][q];
        }
}

// t partials: per (layer, block) the sequential sum of the samples' t_bar
__global__ void k_tsum64(const double *tbar, int L, int lf, long n, int nb, int Z, int K, int V,
                         double *part) {
    const int IN = 3 * K + V;
    const long P = static_cast<long>(Z) * IN + Z + static_cast<long>(K) * Z + K +
                   static_cast<long>(V) * Z + V + 1;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (L - lf) * nb) return;
    const int l = lf + idx / nb, blk = idx % nb;
    const long lo = n * blk / nb, hi = n * (blk + 1) / nb;
    double acc = 0.0;
    for (long s = lo; s < hi; ++s) acc = dadd(acc, tbar[static_cast<long>(l) * n + s]);
    part[(static_cast<long>(blk) * L + l) * P + P - 1] = acc;
}

// raw[l][e] = merged block partials, in block order (Gradients::add_scaled
// with scale 1.0 is exact); frozen layers 0
__global__ void k_merge64(const double *part, int L, int lf, long P, int nb, double *raw) {
    const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long>(L) * P) return;
    const int l = static_cast<int>(idx / P);
    if (l < lf) { raw[idx] = 0.0; return; }
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc = dadd(acc, part[static_cast<long>(b) * L * P + idx]);
    raw[idx] = acc;
}

// finish_eval (kernels.cpp:93-103): per-sample losses summed in sample order
// (one thread: the reference's sequential sum), error / flag counts
__global__ void __launch_bounds__(256) k_reduce64(const double *loss, const long long *err,
                                                  const uint8_t *flag, long n, double *out_loss,
                                                  long long *out_err, long long *out_flag,
                                                  double *loss_copy) {
    __shared__ long long se[256], sf[256];
    long long e = 0, f = 0;
    for (long i = threadIdx.x; i < n; i += 256) { e += err[i]; f += flag[i]; }
    se[threadIdx.x] = e;
    sf[threadIdx.x] = f;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) { se[threadIdx.x] += se[threadIdx.x + w]; sf[threadIdx.x] += sf[threadIdx.x + w]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (long i = 0; i < n; ++i) acc = dadd(acc, loss[i]);
        *out_loss = acc;
        *out_err = se[0];
        *out_flag = sf[0];
        if (loss_copy) *loss_copy = acc;
    }
}

} // namespace detnet
