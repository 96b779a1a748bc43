// gram.cuh -- G x for one sample's packed Gram matrix split over two
// threads (rows [0, 6) and [6, 20) of the upper triangle, 105 entries each),
// shared by the tcgen05 forward (stack_h16.cu) and reverse sweep (bwd_tc.cu).
#pragma once

#include "common.cuh"

namespace detnet {
namespace gram {

constexpr int KX = 20;

// packed FP32x2 arithmetic (FADD2 / FFMA2): two lanes per instruction
__device__ __forceinline__ void sub2(float a0, float a1, float b0, float b1, float &d0, float &d1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// (d0, d1) += (a0, a1) * (b0, b1)
__device__ __forceinline__ void fma2(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rd, {%0, %1};\n\tfma.rn.f32x2 rd, ra, rb, rd;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// Rows [R0, R1) of G x for the packed upper triangle g (row-major, r <= c,
// rows R0.. only): gx[r] += sum_c G_rc x_c and, by symmetry, gx[c] += G_rc x_r.
// Column pairs (c, c+1), c even, go through FFMA2: the row part into an
// (even, odd) accumulator pair, the mirrored part into (gx[c], gx[c+1]).
template <int R0, int R1>
__device__ __forceinline__ void gram_mv(const float *g, const float (&x)[KX], float (&gx)[KX]) {
    sfor<R0, R1>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        constexpr int e0 = r * KX - r * (r - 1) / 2 - (R0 * KX - R0 * (R0 - 1) / 2); // entry (r, r)
        gx[r] = fmaf(g[e0], x[r], gx[r]);
        constexpr int c1 = (r + 1) % 2 == 0 ? r + 1 : r + 2; // first paired (even) column
        if constexpr (c1 == r + 2 && r + 1 < KX) {
            gx[r] = fmaf(g[e0 + 1], x[r + 1], gx[r]);
            gx[r + 1] = fmaf(g[e0 + 1], x[r], gx[r + 1]);
        }
        float re = 0.f, ro = 0.f;
        sfor<0, (KX - c1) / 2>([&](auto pc) {
            constexpr int c = c1 + 2 * decltype(pc)::value;
            constexpr int e = e0 + (c - r);
            fma2(re, ro, g[e], g[e + 1], x[c], x[c + 1]);
            fma2(gx[c], gx[c + 1], g[e], g[e + 1], x[r], x[r]);
        });
        if constexpr (c1 < KX) gx[r] += re + ro;
    });
}


} // namespace gram
} // namespace detnet
