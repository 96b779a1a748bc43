// dw_tc.cu -- the training step's weight-gradient contractions on tcgen05
// (accumulate_outer, backward.cpp:21-29, summed over the batch as in
// batch_gradient, kernels.cpp:160-200):
//   dW1|b1   [Z][IN+1]  = u1bar[Z][s] . [in; 1][IN+1][s]^T
//   dW23|b23 [K+V][Z+1] = [u2bar; vbar][K+V][s] . [z; 1][Z+1][s]^T
// per 256-sample split (the K dimension is the batch), one CTA per (layer,
// which, split). Operands are the forward trace / reverse-sweep adjoints,
// feature-major in HBM ([row][ts], contiguous over samples = K-major), staged
// through shared memory in 32-sample chunks (double buffered) as 3xTF32
// splits: hi = rna_tf32(v), lo = v - hi, D += Ahi.Bhi + Ahi.Blo + Alo.Bhi in
// FP32 in TMEM (kind::tf32, M = 128, N = 112 | 176, A and B from shared
// memory). The epilogue writes each split's FP32 result as an FP64 partial,
// exactly like the CUDA-core k_dw_gemm it replaces (k_grad_sum folds the
// partials in fixed order), so the step stays deterministic.
#include "dw_job.hpp"
#include "engine.hpp"
#include "tc_ptx.cuh"

namespace detnet {
namespace {

constexpr int DWT_THREADS = 256, DWT_KC = 32; // samples per staged chunk
constexpr int DWT_LOADS = 9; // float4 loads per thread per chunk: ceil((M + N) / 8) * 64 <= 9 * 256
constexpr uint32_t DWT_SMEM = 2 * (256 + 176) * DWT_KC * 4 * 2 + 64;

__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

// byte offset of (row r, chunk column k) in a no-swizzle K-major TF32 image of R rows
__device__ __forceinline__ uint32_t img_off(int r, int k, int R) {
    return static_cast<uint32_t>((k >> 2) * R * 16 + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__global__ void __launch_bounds__(DWT_THREADS, 1)
    k_dw_tc(const DwJob *jobs, long n, long ts, int splits) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const DwJob jb = jobs[blockIdx.x / splits];
    const int sp = static_cast<int>(blockIdx.x % splits);
    const int M = jb.M, N = jb.N;
    const int mt = (M + 127) / 128;
    const int NP = (N + 1 + 15) / 16 * 16; // + the bias column (B row N = 1)
    const int RA = 128 * mt, RB = NP;
    const uint32_t img_a = static_cast<uint32_t>(RA) * DWT_KC * 4, img_b = static_cast<uint32_t>(RB) * DWT_KC * 4;
    const uint32_t stage = 2 * (img_a + img_b); // Ahi Alo Bhi Blo
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + 2 * stage);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(sm + 2 * stage + 16);
    const uint32_t sbase = smem_u32(sm);
    const int tid = threadIdx.x, warp = tid >> 5;
    const long k0 = static_cast<long>(sp) * DW_SPLIT;
    const long k1 = k0 + DW_SPLIT < n ? k0 + DW_SPLIT : n;
    const int nchunks = static_cast<int>((k1 - k0 + DWT_KC - 1) / DWT_KC);
    DETNET_DASSERT(k0 < n && M <= 256 && NP <= 176 && nchunks >= 1 && 2 * stage + 32 <= DWT_SMEM);

    // constant parts of both stages: zero padding rows, the bias row of B
    for (int s = 0; s < 2; ++s) {
        const uint32_t st = sbase + s * stage;
        for (int e = tid; e < (RA - M) * (DWT_KC / 4); e += DWT_THREADS) {
            const int r = M + e / (DWT_KC / 4), k = 4 * (e % (DWT_KC / 4));
            st_shared_v4(st + img_off(r, k, RA), 0.f, 0.f, 0.f, 0.f);
            st_shared_v4(st + img_a + img_off(r, k, RA), 0.f, 0.f, 0.f, 0.f);
        }
        for (int e = tid; e < (RB - N) * (DWT_KC / 4); e += DWT_THREADS) {
            const int r = N + e / (DWT_KC / 4), k = 4 * (e % (DWT_KC / 4));
            const float one = r == N ? 1.f : 0.f;
            st_shared_v4(st + 2 * img_a + img_off(r, k, RB), one, one, one, one);
            st_shared_v4(st + 2 * img_a + img_b + img_off(r, k, RB), 0.f, 0.f, 0.f, 0.f);
        }
    }
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tc::tmem_alloc(tslot, 256);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tslot;
    const uint32_t idesc = tc::idesc_tf32(128, NP);

    // software pipeline: chunk c + 1's global loads are in flight while chunk
    // c is split into the stage images and its MMAs are issued
    // element e -> (row, 4-sample group q): 8 consecutive lanes take 8
    // consecutive rows of one q, so each quarter-warp stores one full 128-byte
    // core-matrix line (no bank conflicts) and each row's 4 groups are 64
    // contiguous bytes of the global row
    const int nv = (M + N + 7) / 8 * 64;
    auto rowq = [](int e, int &row, int &q) {
        row = (e >> 6) * 8 + (e & 7);
        q = (e >> 3) & 7;
    };
    float4 v[DWT_LOADS], nxt[DWT_LOADS];
    auto load_chunk = [&](int c, float4 (&dst)[DWT_LOADS]) {
        const long kc = k0 + static_cast<long>(c) * DWT_KC;
#pragma unroll
        for (int i = 0; i < DWT_LOADS; ++i) {
            const int e = tid + i * DWT_THREADS;
            dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            int row, q;
            rowq(e, row, q);
            if (e < nv && row < M + N) {
                const bool isA = row < M;
                const int r = isA ? row : row - M;
                const float *src = (isA ? jb.A : jb.B) + static_cast<long>(r) * ts + kc + 4 * q;
                if (kc + 4 * q + 4 <= k1) {
                    dst[i] = __ldg(reinterpret_cast<const float4 *>(src));
                } else {
                    if (kc + 4 * q + 0 < k1) dst[i].x = __ldg(src + 0);
                    if (kc + 4 * q + 1 < k1) dst[i].y = __ldg(src + 1);
                    if (kc + 4 * q + 2 < k1) dst[i].z = __ldg(src + 2);
                }
            }
        }
    };
    load_chunk(0, v);
    for (int c = 0; c < nchunks; ++c) {
        const int s = c & 1;
        if (c + 1 < nchunks) load_chunk(c + 1, nxt);
        if (c >= 2) mbar_wait(&bars[s], ((c - 2) >> 1) & 1); // MMAs of chunk c-2 read this stage
        const uint32_t st = sbase + s * stage;
#pragma unroll
        for (int i = 0; i < DWT_LOADS; ++i) {
            const int e = tid + i * DWT_THREADS;
            int row, q;
            rowq(e, row, q);
            if (e >= nv || row >= M + N) continue;
            const bool isA = row < M;
            const int r = isA ? row : row - M;
            const float f[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
            float h[4], l[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                h[j] = tc::tf32_rna(f[j]);
                l[j] = f[j] - h[j];
            }
            const uint32_t off = isA ? img_off(r, 4 * q, RA) : img_off(r, 4 * q, RB);
            const uint32_t hi = isA ? st + off : st + 2 * img_a + off;
            const uint32_t lo = hi + (isA ? img_a : img_b);
            st_shared_v4(hi, h[0], h[1], h[2], h[3]);
            st_shared_v4(lo, l[0], l[1], l[2], l[3]);
        }
        fence_proxy_async(); // generic-proxy smem writes -> the tensor core's async proxy
        __syncthreads();
        if (warp == 0) {
            tc::fence_after();
            if (tc::elect_one()) {
                const uint32_t ahi = st, alo = st + img_a, bhi = st + 2 * img_a, blo = bhi + img_b;
#pragma unroll 1
                for (int ks = 0; ks < DWT_KC / 8; ++ks) {
                    const uint64_t dbh = tc::smem_desc(bhi + ks * 2 * RB * 16, RB * 16, 128);
                    const uint64_t dbl = tc::smem_desc(blo + ks * 2 * RB * 16, RB * 16, 128);
                    for (int t = 0; t < mt; ++t) {
                        const uint32_t ao = t * 2048 + ks * 2 * RA * 16;
                        const uint64_t dah = tc::smem_desc(ahi + ao, RA * 16, 128);
                        const uint64_t dal = tc::smem_desc(alo + ao, RA * 16, 128);
                        const uint32_t d = tbase + t * NP;
                        mma_tf32_ss(d, dah, dbh, idesc, (c > 0 || ks > 0) ? 1u : 0u);
                        mma_tf32_ss(d, dah, dbl, idesc, 1u);
                        mma_tf32_ss(d, dal, dbh, idesc, 1u);
                    }
                }
                tc::commit(&bars[s]);
            }
            __syncwarp();
        }
#pragma unroll
        for (int i = 0; i < DWT_LOADS; ++i) v[i] = nxt[i];
    }
    const int cl = nchunks - 1;
    mbar_wait(&bars[cl & 1], (cl >> 1) & 1);
    tc::fence_after();
    // epilogue: lane = output row, columns = [0, N]; warp w and w + 4 share the
    // lane quadrant w % 4 and split the columns
    const int wq = warp & 3, half = warp >> 2;
    for (int t = 0; t < mt; ++t) {
        const int m = t * 128 + wq * 32 + (tid & 31);
        const uint32_t trow = tbase + t * NP + (static_cast<uint32_t>(wq * 32) << 16);
        double *orow = jb.out + (static_cast<long>(sp) * M + m) * (N + 1);
        for (int c0 = 16 * half; c0 < NP; c0 += 32) {
            uint32_t r[16];
            tc::ld16_nw(trow + c0, r);
            tc::wait_ld();
            if (m < M) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j <= N) orow[c0 + j] = static_cast<double>(__uint_as_float(r[j]));
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 256);
}

} // namespace

int dw_tc_prepare() {
    return cudaFuncSetAttribute(k_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(DWT_SMEM)) == cudaSuccess
               ? 0
               : fail(DETNET_ERR_CUDA, "cudaFuncSetAttribute (dW tcgen05 smem) failed");
}

// jobs [j0, j1) of the device job list; every job's M <= 256, N + 1 <= 176
int dw_tc_launch(const DwJob *jobs, int j0, int j1, long n, long ts, int splits, cudaStream_t st) {
    k_dw_tc<<<static_cast<unsigned>((j1 - j0) * splits), DWT_THREADS, DWT_SMEM, st>>>(jobs + j0, n,
                                                                                    ts, splits);
    return check_launch();
}

} // namespace detnet
