// common.cuh -- shared device helpers for the DetNet layer-stack engine.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

// Debug build (make EXTRA=-DDETNET_DEBUG_ASSERT, built by __graft_entry__.build()
// into build/debug/): device-side bounds checks on the index math of every
// kernel family; a failed check prints its location and traps (a launch error
// instead of silent corruption). The stand-in for compute-sanitizer, which this
// GPU pool does not offer. Compiled out of the product library.
#ifdef DETNET_DEBUG_ASSERT
#include <cstdio>
#define DETNET_DASSERT(c)                                                                      \
    do {                                                                                       \
        if (!(c)) {                                                                            \
            printf("DETNET_DASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);             \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define DETNET_DASSERT(c)                                                                      \
    do {                                                                                       \
    } while (0)
#endif

namespace detnet {

// Samples per tile: one tile = one TMEM lane block (128 rows) in the tcgen05
// path and one 128-thread group in the SIMT path. Per-tile SoA buffers
// (packed Gram matrix, q) are laid out [tile][entry][TILE] so consecutive
// threads (samples) read consecutive words.
constexpr int TILE = 128;

__host__ __device__ constexpr int gram_entries(int K) { return K * (K + 1) / 2; }
__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }

// ---- splitmix64 (rng.cpp:10-16) ------------------------------------------
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ---- IEEE-exact FP64 arithmetic without FMA contraction -------------------
// The reference is compiled for baseline x86-64 (no FMA), so every a*b+c it
// evaluates is two roundings. These wrappers keep nvcc from contracting.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ---- mbarrier + bulk-copy (TMA engine, 1-D) helpers -----------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}

// Same, with a watchdog: traps (kernel error instead of a hung GPU) if the
// phase has not completed after ~4 s of SM clocks.
__device__ __forceinline__ void mbar_wait_guard(uint64_t *bar, uint32_t phase) {
    if (mbar_try_wait(bar, phase)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, phase)) {
        if (clock64() - t0 > 8000000000LL) __trap();
    }
}

// 1-D bulk copy global -> shared, completion counted on an mbarrier
// (SASS: UBLKCP). bytes must be a multiple of 16, addresses 16-B aligned.
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Issue a large copy as chunks (each <= 64 KB) on one mbarrier; the caller
// arms the barrier with the total byte count first.
__device__ __forceinline__ void bulk_g2s_chunked(void *dst_smem, const void *src_gmem,
                                                 uint32_t bytes, uint64_t *bar) {
    constexpr uint32_t kChunk = 32768;
    uint32_t off = 0;
    while (off < bytes) {
        const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
        bulk_g2s(static_cast<char *>(dst_smem) + off, static_cast<const char *>(src_gmem) + off, n,
                 bar);
        off += n;
    }
}

// ---- deterministic block reductions ---------------------------------------
// bar.sync on a named barrier (ids 1..15; 0 is __syncthreads)
// (d0, d1) += (a0, a1) * (b0, b1): one fma.rn.f32x2 (SASS FFMA2); each lane is
// rounded exactly like fmaf, so results are bit-identical to two fmaf calls
__device__ __forceinline__ void fma_x2(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rd, {%0, %1};\n\tfma.rn.f32x2 rd, ra, rb, rd;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Compile-time loops: f(std::integral_constant<int, i>) for i in [I, E) (sfor)
// or E-1 down to I (sfor_rev), so register arrays indexed by i stay in registers.
template <int I, int E, class F> __device__ __forceinline__ void sfor(F &&f) {
    if constexpr (I < E) {
        f(std::integral_constant<int, I>{});
        sfor<I + 1, E>(static_cast<F &&>(f));
    }
}
template <int I, int E, class F> __device__ __forceinline__ void sfor_rev(F &&f) { // E-1 .. I
    if constexpr (I < E) {
        f(std::integral_constant<int, E - 1>{});
        sfor_rev<I, E - 1>(static_cast<F &&>(f));
    }
}
#define SF_IDX(v) decltype(v)::value

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

} // namespace detnet
