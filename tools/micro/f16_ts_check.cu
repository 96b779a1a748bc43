// Probe: kind::f16 tcgen05.mma with A in TMEM (TS form) -- operand layout
// check against the CPU, and issue-rate comparison with kind::tf32 (same
// M=128, N=80, 32 B of K per row per instruction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 -I../../paper_2003_09446_b200/csrc f16_ts_check.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include "tc_ptx.cuh"
using namespace detnet;

constexpr int N = 80, KF = 16;

__global__ void k_check(const __half *A, const __half *B, float *D, long long *cyc, int chain,
                        int tf32) {
    __shared__ __align__(128) unsigned char sB[N * KF * 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int t = threadIdx.x, warp = t >> 5;
    // B (n, k) -> (k/8)*LBO + (n/8)*128 + (n%8)*16 + (k%8)*2, LBO = N*16
    for (int i = t; i < N * KF; i += 128) {
        const int n = i / KF, k = i % KF;
        *reinterpret_cast<__half *>(sB + (k / 8) * (N * 16) + (n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) =
            B[n * KF + k];
    }
    if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) { tc::tmem_alloc(&slot, 128); tc::tmem_relinquish(); }
    fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = slot;
    // A row t: 8 columns at col 96, fp16 pairs (2c low, 2c+1 high)
    {
        float v[8];
        for (int c = 0; c < 8; ++c) {
            const uint32_t lo = __half_as_ushort(A[t * KF + 2 * c]);
            const uint32_t hi = __half_as_ushort(A[t * KF + 2 * c + 1]);
            v[c] = __uint_as_float(lo | (hi << 16));
        }
        tc::st8(tb + ((warp * 32) << 16) + 96, v);
        tc::wait_st();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint64_t d = tc::smem_desc(smem_u32(sB), N * 16, 128);
        const uint32_t id = tf32 ? tc::idesc_tf32(128, N) : tc::idesc_f16(128, N);
        t0 = clock64();
        if (tc::elect_one()) {
            for (int i = 0; i < chain; ++i) {
                if (tf32) tc::mma_tf32_ts(tb, tb + 96, d, id, i > 0);
                else tc::mma_f16_ts(tb, tb + 96, d, id, i > 0);
            }
            tc::commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        t1 = clock64();
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    tc::fence_after();
    float r[16];
    for (int c = 0; c < N; c += 16) {
        tc::ld16(tb + ((warp * 32) << 16) + c, r);
        for (int j = 0; j < 16; ++j) D[(blockIdx.x * 128 + t) * N + c + j] = r[j];
    }
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tb, 128);
}

int main() {
    std::vector<__half> A(128 * KF), B(N * KF);
    std::vector<float> Af(128 * KF), Bf(N * KF);
    srand(1);
    for (int i = 0; i < 128 * KF; ++i) { Af[i] = (rand() % 17 - 8) / 8.0f; A[i] = __float2half(Af[i]); }
    for (int i = 0; i < N * KF; ++i) { Bf[i] = (rand() % 33 - 16) / 16.0f; B[i] = __float2half(Bf[i]); }
    __half *dA, *dB; float *dD; long long *dc;
    const int grid = 148;
    cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dD, (size_t)grid * 128 * N * 4); cudaMalloc(&dc, grid * 8);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    std::vector<float> D(128 * N);
    k_check<<<1, 128>>>(dA, dB, dD, dc, 1, 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    // hypotheses for the TMEM A layout: H1 column c = (k 2c, 2c+1); H2 = (k c, c+8)
    double err1 = 0, err2 = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double s1 = 0, s2 = 0;
            for (int c = 0; c < 8; ++c) {
                s1 += Af[m * KF + 2 * c] * Bf[n * KF + 2 * c] + Af[m * KF + 2 * c + 1] * Bf[n * KF + 2 * c + 1];
                s2 += Af[m * KF + 2 * c] * Bf[n * KF + c] + Af[m * KF + 2 * c + 1] * Bf[n * KF + c + 8];
            }
            err1 = fmax(err1, fabs(s1 - D[m * N + n]));
            err2 = fmax(err2, fabs(s2 - D[m * N + n]));
        }
    printf("layout: max|err| H1 (pairs 2c,2c+1) = %g   H2 (c, c+8) = %g   D[0][0]=%g\n", err1, err2, D[0]);
    for (int tf = 0; tf < 2; ++tf) {
        for (int rep = 0; rep < 2; ++rep) {
            const int chain = 2048;
            k_check<<<grid, 128>>>(dA, dB, dD, dc, chain, tf);
            cudaDeviceSynchronize();
            std::vector<long long> c(grid);
            cudaMemcpy(c.data(), dc, grid * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto x : c) avg += x;
            avg /= grid;
            if (rep) printf("%s N=%d: %.1f cycles per MMA (%s)\n", tf ? "tf32 K=8 " : "f16  K=16", N, avg / chain,
                            cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
