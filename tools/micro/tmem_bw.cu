// Probe: TMEM load/store throughput per SM (tcgen05.ld/st 32x32b) with 4 or 8
// warps, x16 / x32 loads per wait, to see what bounds the stack epilogue.
#include <cstdio>
#include <vector>
#include "tc_ptx.cuh"
using namespace detnet;

__device__ __forceinline__ void ld32(uint32_t t, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(t));
}
// 16x256b: 16 lanes x 256 bit per instruction (x1: 4 regs/thread)
__device__ __forceinline__ void ld16x256_x4(uint32_t t, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(t));
}

__global__ void k_bw(long long *cyc, unsigned *sink, int iters, int mode) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tc::tmem_alloc(&slot, 512); tc::tmem_relinquish(); }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = slot + ((static_cast<uint32_t>((warp & 3) * 32)) << 16);
    const int colbase = (warp >> 2) * 128; // second warpgroup reads other columns
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t c = tb + colbase + (i & 3) * 32;
        if (mode == 0) {        // load 32 cols, wait
            uint32_t r[32];
            ld32(c, r);
            tc::wait_ld();
            for (int k = 0; k < 32; ++k) acc += r[k];
        } else if (mode == 1) { // 4 x 32 cols in flight, one wait
            uint32_t r[32], q[32], u[32], w[32];
            ld32(tb + colbase, r);
            ld32(tb + colbase + 32, q);
            ld32(tb + colbase + 64, u);
            ld32(tb + colbase + 96, w);
            tc::wait_ld();
            for (int k = 0; k < 32; ++k) acc += r[k] ^ q[k] ^ u[k] ^ w[k];
        } else {                // store 32 cols
            float v[16];
            for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(acc + k);
            tc::st16(c, v);
            tc::st16(c + 16, v);
            tc::wait_st();
            acc += 1;
        }
    }
    const long long t1 = clock64();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(slot, 512);
}

int main() {
    long long *dc; unsigned *ds;
    cudaMalloc(&dc, 148 * 8); cudaMalloc(&ds, 148 * 512 * 4);
    const char *nm[3] = {"ld 32x32b.x32 + wait", "ld 4 x 32x32b.x32 + wait", "st 32x32b.x16 x2 + wait"};
    for (int mode = 0; mode < 3; ++mode)
        for (int warps : {4, 8}) {
            const int iters = 4096;
            for (int rep = 0; rep < 2; ++rep) k_bw<<<148, warps * 32>>>(dc, ds, iters, mode);
            cudaDeviceSynchronize();
            std::vector<long long> c(148);
            cudaMemcpy(c.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
            double avg = 0; for (auto x : c) avg += x; avg /= 148;
            const double bytes = (double)iters * warps * 32 * 32 * 4 * (mode == 1 ? 4 : 1); // per SM
            printf("%-26s warps=%d: %.1f cycles/iter, %.1f B/clk/SM  (%s)\n", nm[mode], warps, avg / iters,
                   bytes / avg, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
