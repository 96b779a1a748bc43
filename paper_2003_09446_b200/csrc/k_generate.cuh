// k_generate.cuh -- K0: on-device channel generator.
//
// Restates make_sample (channel.cpp:14-32) under generate_batch's keying
// (kernels.cpp:121-127): sample i draws from base.stream(i) in the order
// SNR (ranged only) -> H row-major Gaussians -> x bits -> noise Gaussians.
// The splitmix64 stream is random access (draw d = mix64(s0 + (d+1)*gamma)),
// so each thread reads its x bits first and then streams H once, forming
// y = H x in the reference's matvec order (linalg.cpp:8-18) on the fly.
// FP64 transcendental results (log, cos, pow) may differ from glibc in the
// last ulp; after the FP32 rounding the samples match the host generator
// except on rare rounding ties (tests/test_gpu_generator.py bounds this).
#pragma once

#include "common.cuh"

namespace detnet {

__device__ __forceinline__ double u01_from(uint64_t r) {
    return static_cast<double>(r >> 11) * 0x1.0p-53;
}

// Out = float: H, y scaled and rounded to FP32, x as int8 (the engine's input
// format). Out = double: unscaled FP64 ChannelSample fields (H, y, x = +-1.0),
// what unfold::generate_batch returns.
template <typename Out, typename XOut>
__global__ void __launch_bounds__(128) k_generate(uint64_t base, long first, long count, int N,
                                                  int K, double lo, double hi, double scale,
                                                  Out *__restrict__ H, Out *__restrict__ y,
                                                  XOut *__restrict__ x,
                                                  double *__restrict__ sigma2) {
    const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint64_t s0 =
        mix64(base ^ mix64(static_cast<uint64_t>(first + i) + 0xda3e39cb94b95bdbULL));
    const bool ranged = lo != hi;
    const uint64_t d0 = ranged ? 1 : 0;
    double snr = lo;
    if (ranged) snr = dadd(lo, dmul(hi - lo, u01_from(mix64(s0 + kGamma))));
    const double s2 = static_cast<double>(K) * pow(10.0, -snr / 10.0);
    const double sigma = sqrt(s2);

    // x bits: draws d0 + 2NK + j
    uint32_t xbits = 0;
    const uint64_t dx = d0 + 2ull * N * K;
    for (int j = 0; j < K; ++j) {
        const uint64_t r = mix64(s0 + (dx + j + 1) * kGamma);
        if (r >> 63) xbits |= 1u << j;
        x[i * K + j] = (r >> 63) ? XOut(1) : XOut(-1);
    }
    // H and y = H x (row i: acc over j ascending), then noise
    uint64_t st = s0 + d0 * kGamma;
    const double two_pi = 2.0 * 3.141592653589793;
    for (int r = 0; r < N; ++r) {
        double acc = 0.0;
        for (int j = 0; j < K; ++j) {
            st += kGamma;
            const double u1 = 1.0 - u01_from(mix64(st));
            st += kGamma;
            const double u2 = u01_from(mix64(st));
            const double g = dmul(sqrt(-2.0 * log(u1)), cos(dmul(two_pi, u2)));
            H[(i * N + r) * K + j] = static_cast<Out>(dmul(g, scale));
            acc = dadd(acc, (xbits >> j) & 1u ? g : -g);
        }
        // noise draw for row r: d0 + 2NK + K + 2r (+1)
        uint64_t sn = s0 + (dx + K + 2ull * r) * kGamma;
        sn += kGamma;
        const double n1 = 1.0 - u01_from(mix64(sn));
        sn += kGamma;
        const double n2 = u01_from(mix64(sn));
        const double g = dmul(sqrt(-2.0 * log(n1)), cos(dmul(two_pi, n2)));
        y[i * N + r] = static_cast<Out>(dmul(dadd(acc, dmul(sigma, g)), scale));
    }
    if (sigma2) sigma2[i] = s2;
}

} // namespace detnet
