// Throughput probe: F2F.F64.F32, DFMA, FFMA, LDS.128 per SM per clock on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_cvt(const float *in, double *out, int iters) {
    float f[8];
    for (int i = 0; i < 8; ++i) f[i] = in[threadIdx.x + i];
    double acc[8] = {0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[i] += (double)f[i];
            f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(const double *in, double *out, int iters) {
    double a[8], b = in[0], c = in[1];
    for (int i = 0; i < 8; ++i) a[i] = in[threadIdx.x + i];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(const float *in, float *out, int iters) {
    float a[8], b = in[0], c = in[1];
    for (int i = 0; i < 8; ++i) a[i] = in[threadIdx.x + i];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *fi; double *di, *dout; float *fout;
    cudaMalloc(&fi, 4096 * 4); cudaMalloc(&di, 4096 * 8);
    cudaMemset(fi, 0, 4096 * 4); cudaMemset(di, 0, 4096 * 8);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaMalloc(&dout, (size_t)blocks * threads * 8); cudaMalloc(&fout, (size_t)blocks * threads * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int which = 0; which < 3; ++which) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (which == 0) k_cvt<<<blocks, threads>>>(fi, dout, iters);
            if (which == 1) k_dfma<<<blocks, threads>>>(di, dout, iters);
            if (which == 2) k_ffma<<<blocks, threads>>>(fi, fout, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters * 8;
            double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
            if (rep) printf("%s: %.1f ops/clk/SM (%.2f Gop/s, clk %d MHz nominal)\n",
                            which == 0 ? "F2F.F64.F32(+DADD)" : which == 1 ? "DFMA" : "FFMA",
                            per_sm_clk, ops / ms / 1e6, clk / 1000);
        }
    }
    return 0;
}
