// Probe: tcgen05.mma (TS form) issue rate vs N and accumulator dependency.
#include <cstdio>
#include <vector>
#include "tc_ptx.cuh"
using namespace detnet;

template <int N, int M = 128>
__global__ void k_rate(long long *cyc, int chain, int tf32, int nacc) {
    extern __shared__ __align__(128) unsigned char sB[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < N * 32 / 4; i += 128) reinterpret_cast<uint32_t *>(sB)[i] = 0x3c003c00u;
    if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) { tc::tmem_alloc(&slot, 512); tc::tmem_relinquish(); }
    fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = slot;
    if (warp == 0) {
        const uint64_t d = tc::smem_desc(smem_u32(sB), N * 16, 128);
        const uint32_t id = tf32 ? tc::idesc_tf32(M, N) : tc::idesc_f16(M, N);
        const long long t0 = clock64();
        if (tc::elect_one()) {
            for (int i = 0; i < chain; ++i) {
                const uint32_t dcol = tb + (i % nacc) * N;
                if (tf32) tc::mma_tf32_ts(dcol, tb + 504, d, id, 1);
                else tc::mma_f16_ts(dcol, tb + 504, d, id, 1);
            }
            tc::commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        if (t == 0) cyc[blockIdx.x] = clock64() - t0;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tb, 512);
}

template <int N, int M = 128> void run(long long *dc, int grid) {
    cudaFuncSetAttribute(k_rate<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    for (int tf = 0; tf < 2; ++tf)
        for (int nacc = 1; nacc <= 2; ++nacc) {
            if (nacc * N > 496) continue;
            double avg = 0;
            for (int rep = 0; rep < 2; ++rep) {
                const int chain = 4096;
                k_rate<N, M><<<grid, 128, N * 32>>>(dc, chain, tf, nacc);
                cudaDeviceSynchronize();
                std::vector<long long> c(grid);
                cudaMemcpy(c.data(), dc, grid * 8, cudaMemcpyDeviceToHost);
                avg = 0;
                for (auto x : c) avg += x;
                avg /= grid * (double)chain;
            }
            printf("M=%d %s N=%3d acc=%d: %6.1f cyc/MMA  (N/2 = %d)  %s\n", M, tf ? "tf32" : "f16 ", N, nacc, avg,
                   N / 2, cudaGetErrorString(cudaGetLastError()));
        }
}

int main() {
    long long *dc;
    cudaMalloc(&dc, 148 * 8);
    run<32>(dc, 148); run<48>(dc, 148); run<64>(dc, 148); run<80>(dc, 148); run<128>(dc, 148);
    run<160>(dc, 148); run<240>(dc, 148);
    // M = 64 (cta_group::1): same N, half the rows
    run<32, 64>(dc, 148); run<64, 64>(dc, 148); run<96, 64>(dc, 148); run<160, 64>(dc, 148);
    return 0;
}
