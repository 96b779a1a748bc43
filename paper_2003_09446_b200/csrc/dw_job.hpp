// dw_job.hpp -- argument structs of the training step's reverse sweep and
// weight-gradient contractions, shared by the CUDA-core kernels (k_train.cuh)
// and the tcgen05 ones (bwd_tc.cu, dw_tc.cu).
#pragma once

#include <cstdint>

namespace detnet {

// C[job][m][n] partial over a split of samples: C = A . B^T with A [M][ts],
// B [N][ts]; column n == N is the bias (sum of A). Jobs = (layer, which).
struct DwJob {
    const float *A;
    const float *B;
    int M, N;       // output M x (N + 1)
    double *out;    // [splits][M][N+1] partials
};

// samples per FP32 split (FP64 across splits); 8 splits = one 8,192-sample
// reduction chunk (k_grad_sum)
constexpr int DW_SPLIT = 1024;

struct BwdArgs {
    const float *gp;        // [tile][NG][TILE]
    const double *denom;    // [s]
    const uint32_t *xmask;  // [s]
    const float *wrec;      // SIMT layer records
    long rec_floats;
    const double *lnk;      // ln(l+1)
    int L, lf;              // layers, frozen prefix (sweep l = L-1 .. lf)
    long n, n_tiles, ts;
    const float *tr_in, *tr_z, *tr_u2, *tr_xf;
    float *u1bar;           // [L][Z][ts]
    float *g23bar;          // [L][K+V][ts]
    double *tbar_part;      // [L][ts / 32]: t gradient per 32-sample warp group
    // k_train_bwd_pair only: sweep iterations [it_begin, it_end) of [0, L - lf)
    // (layer L-1-it); a_bar / v_bar carried between chunks in state [K+V][ts]
    int it_begin = 0, it_end = -1;
    float *state = nullptr;
    uint32_t *gate = nullptr; // tcgen05 sweep: [L][5][ts] relu-gate bit masks (bwd_tc.cu)
};


} // namespace detnet
