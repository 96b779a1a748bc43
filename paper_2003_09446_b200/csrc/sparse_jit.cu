// sparse_jit.cu -- K4J: the layer stack of a sparse-group model (BASELINE
// config 4) as a kernel specialised to that model.
//
// The masked branch of masked_affine (model.cpp:69-78) multiplies by a fixed
// set of surviving weights that every sample shares. At ~5 % density inside
// the surviving groups a layer is ~170 W1 and ~150 [W3; W2] products per
// sample, against ~400 multiply-adds for G x_hat: the dense tcgen05 kernels
// spend their time on zeros and on the x_hat -> G x_hat chain, and a
// table-driven CSR walk (k_stack_sparse.cuh) on decoding entries. Here the
// sparsity pattern is compiled into the instruction stream: at first use the
// engine emits CUDA source in which every surviving weight is an FP32
// immediate of an FFMA and every operand a register (the layer input
// [q; x; G x; v], model.cpp:96-99, the hidden units z, the outputs [v'; u2]),
// compiles it with NVRTC for sm_100a and loads it with cudaLibraryLoadData.
// No index or weight is ever loaded; a layer is ~300 FFMAs + G x_hat.
//
// Kernel organisation: one thread per sample, 128-sample tiles (the K1 tile,
// so the per-tile [entry][128] Gram / q layout is read directly), persistent
// CTAs of 128 threads, two per SM. A sample's packed Gram matrix (210 FP32)
// lives in registers (the first GREG entries) and in shared memory (the rest,
// float4 groups [group][128 samples]: 16-byte loads, conflict free); each
// thread touches only its own column, so there is no barrier anywhere and
// the four warps of a tile run decoupled. Per layer: G x_hat (symmetric,
// both triangles from the packed upper one), the hidden units of the live
// set (units with a surviving outgoing weight, model.cpp:114-118) as
// relu(b1 + sum of immediates x registers), the 60 outputs in gather form,
// psi_t (model.cpp:32-51), the depth-weighted loss term (loss.cpp:9-31) and
// x_l. Tile end: error count vs the x bits (kernels.cpp:63-65) and the
// per-lane-quadrant loss / error partials every stack kernel writes, so the
// canonical reduction (k_reduce) is shared.
//
// Arithmetic: FP32 throughout, products accumulated per output in input
// index order (the reference's loop order) with FMA; the loss sum in FP64.
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include "engine.hpp"

namespace detnet {

namespace {

// The fixed part of the generated kernel. Placeholders: @K@ @KP@ @V@ @NB@
// @GB@ @NS@ @CTAS@, @STAGE@ (a tile's Gram blocks into registers / shared
// memory), @GRAM@ (G x_hat), @LAYERS@ (one switch case per layer).
//
// Gram layout: the symmetric G (K padded to even KP) as 2x2 blocks (i, j),
// j >= i, each one float4 in row-major order (G[2i][2j], G[2i][2j+1],
// G[2i+1][2j], G[2i+1][2j+1]); the first GB blocks stay in registers, the
// rest are in shared memory as [block][128 samples] float4. A block is used
// twice with FFMA2 (two FP32 lanes per instruction): rows 2i, 2i+1 take its
// dot products with (x[2j], x[2j+1]) (pair partials, summed at the end),
// rows 2j, 2j+1 take (G[2i][2j], G[2i][2j+1]) x[2i] + (G[2i+1][2j],
// G[2i+1][2j+1]) x[2i+1] (its transpose, by symmetry). 200 FFMA2 for K=20
// instead of 400 FFMA. The shared loads are volatile: the layer loop never
// writes shared memory, so plain loads would be hoisted out of it and held
// in ~200 registers.
const char *kSkeleton = R"JIT(
typedef unsigned int u32;
struct JArgs {
    const float *gp; const float *q32; const double *denom; const u32 *xmask;
    const double *lnk; int l_end; long n, n_tiles, tile0;
    float *xhat; double *tile_loss; long long *tile_err;
};
#define K_ @K@
#define KP_ @KP@
#define V_ @V@
#define GB_ @GB@
__device__ __forceinline__ float relu(float u) { return fmaxf(u, 0.f); }
__device__ __forceinline__ float4 lds4(u32 a) { // volatile: re-read every layer
    float4 t;
    asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(a));
    return t;
}
// (d0, d1) += (a0, a1) * (b0, b1): one FFMA2
__device__ __forceinline__ void f2(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rd, {%0, %1};\n\tfma.rn.f32x2 rd, ra, rb, rd;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// (d0, d1) += (a0, a1): one FADD2
__device__ __forceinline__ void a2(float &d0, float &d1, float a0, float a1) {
    asm("{\n\t.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rd, {%0, %1};\n\t"
        "add.rn.f32x2 rd, rd, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1) : "f"(a0), "f"(a1));
}
template <typename T> __device__ __forceinline__ T wsum32(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
extern "C" __global__ void __launch_bounds__(128, @CTAS@) detnet_sparse_jit(JArgs a) {
    extern __shared__ float4 sG[]; // [NS][128]
    const int col = threadIdx.x, warp = col >> 5, lane = col & 31;
    const u32 sGa = static_cast<u32>(__cvta_generic_to_shared(sG + col));
    for (long tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const long gt = a.tile0 + tile;
        const long s = tile * 128 + col;
        const bool live = s < a.n;
        const float *gps = a.gp + gt * (K_ * (K_ + 1) / 2) * 128 + col;
        float4 gb[GB_ > 0 ? GB_ : 1];
        {
@STAGE@
        }
        float q[K_], x[KP_], v[V_], gx[KP_], u2[K_], xt[K_];
        const u32 xm = a.xmask[gt * 128 + col];
#pragma unroll
        for (int k = 0; k < K_; ++k) {
            q[k] = __ldg(a.q32 + (gt * K_ + k) * 128 + col);
            xt[k] = (xm >> k) & 1u ? 1.f : -1.f;
        }
#pragma unroll
        for (int k = 0; k < KP_; ++k) x[k] = 0.f;
#pragma unroll
        for (int k = 0; k < V_; ++k) v[k] = 0.f;
        double wsum = 0.0;
        for (int l = 0; l < a.l_end; ++l) {
            // q is constant over the layers, so q x weight products would be
            // loop invariants: hoisted out of the loop for all layers at once
            // (hundreds of registers). Re-defining q each layer keeps them here.
#pragma unroll
            for (int k = 0; k < K_; ++k) asm volatile("mov.b32 %0, %0;" : "+f"(q[k]));
            {
@GRAM@
            }
            switch (l) {
@LAYERS@
            default: __trap();
            }
            // the depth-weighted loss term of layer l (loss.cpp:9-31), x_l
            float err = 0.f;
#pragma unroll
            for (int k = 0; k < K_; ++k) {
                const float d = xt[k] - x[k];
                err = fmaf(d, d, err);
            }
            wsum += __ldg(a.lnk + l) * static_cast<double>(err);
            if (a.xhat && live) {
                float *o = a.xhat + (s * a.l_end + l) * K_;
#pragma unroll
                for (int k = 0; k < K_; ++k) o[k] = x[k];
            }
        }
        long long errs = 0;
#pragma unroll
        for (int k = 0; k < K_; ++k) errs += (x[k] >= 0.f) != (((xm >> k) & 1u) != 0);
        double loss = live ? wsum / a.denom[gt * 128 + col] : 0.0;
        if (!live) errs = 0;
        loss = wsum32(loss);
        errs = wsum32(errs);
        if (lane == 0) {
            a.tile_loss[gt * 4 + warp] = loss;
            a.tile_err[gt * 4 + warp] = errs;
        }
    }
}
)JIT";

void replace_all(std::string &s, const std::string &from, const std::string &to) {
    size_t p = 0;
    while ((p = s.find(from, p)) != std::string::npos) {
        s.replace(p, from.size(), to);
        p += to.size();
    }
}

// FP32 immediate, exact (hex float literal)
std::string fimm(float f) {
    if (f == 0.f) return std::signbit(f) ? "-0.0f" : "0.0f";
    char b[48];
    std::snprintf(b, sizeof b, "%af", static_cast<double>(f));
    return b;
}

// layer input index j of [q; x; gx; v] -> register name
std::string in_name(int j, int K) {
    char b[16];
    if (j < K) std::snprintf(b, sizeof b, "q[%d]", j);
    else if (j < 2 * K) std::snprintf(b, sizeof b, "x[%d]", j - K);
    else if (j < 3 * K) std::snprintf(b, sizeof b, "gx[%d]", j - 2 * K);
    else std::snprintf(b, sizeof b, "v[%d]", j - 3 * K);
    return b;
}

// Gram blocks of a KP x KP symmetric matrix: (i, j), j >= i, in row order.
std::vector<std::pair<int, int>> gram_blocks(int K) {
    const int nb = (K + 1) / 2;
    std::vector<std::pair<int, int>> bl;
    for (int i = 0; i < nb; ++i)
        for (int j = i; j < nb; ++j) bl.push_back({i, j});
    return bl;
}

// Per-tile staging: block b = (G[2i][2j], G[2i][2j+1], G[2i+1][2j],
// G[2i+1][2j+1]) gathered from the packed upper triangle K1 writes
// ([entry][128], entry (r, c), r <= c, row-major), zero outside K x K.
std::string gen_stage(int K, int gb) {
    auto pidx = [&](int r, int c) {
        if (r >= K || c >= K) return -1;
        if (r > c) std::swap(r, c);
        return r * K - r * (r - 1) / 2 + (c - r);
    };
    auto ld = [&](int e) {
        return e < 0 ? std::string("0.f") : "__ldg(gps + " + std::to_string(e * 128) + ")";
    };
    const auto bl = gram_blocks(K);
    std::string o;
    for (size_t b = 0; b < bl.size(); ++b) {
        const int i = bl[b].first, j = bl[b].second;
        const std::string t = "make_float4(" + ld(pidx(2 * i, 2 * j)) + ", " + ld(pidx(2 * i, 2 * j + 1)) +
                              ", " + ld(pidx(2 * i + 1, 2 * j)) + ", " + ld(pidx(2 * i + 1, 2 * j + 1)) + ")";
        if (static_cast<int>(b) < gb) o += "gb[" + std::to_string(b) + "] = " + t + ";\n";
        else o += "sG[" + std::to_string((static_cast<int>(b) - gb) * 128) + " + col] = " + t + ";\n";
    }
    return o;
}

// G x_hat from the blocks (see kSkeleton): gx[r] (transposed and diagonal
// parts) + (gd[r], ge[r]) (dot-product pair partials of the direct part).
std::string gen_gram(int K, int gb) {
    const int nb = (K + 1) / 2;
    const auto bl = gram_blocks(K);
    std::string o = "float gd[KP_], ge[KP_];\n#pragma unroll\nfor (int k = 0; k < KP_; ++k) { gx[k] = 0.f; gd[k] = 0.f; ge[k] = 0.f; }\n";
    char b[256];
    for (size_t n = 0; n < bl.size(); ++n) {
        const int i = bl[n].first, j = bl[n].second;
        if (static_cast<int>(n) < gb) std::snprintf(b, sizeof b, "{ const float4 t = gb[%d];\n", static_cast<int>(n));
        else std::snprintf(b, sizeof b, "{ const float4 t = lds4(sGa + %d);\n", (static_cast<int>(n) - gb) * 128 * 16);
        o += b;
        if (i == j) {
            std::snprintf(b, sizeof b,
                          "f2(gx[%d], gx[%d], t.x, t.y, x[%d], x[%d]); f2(gx[%d], gx[%d], t.z, t.w, x[%d], x[%d]); }\n",
                          2 * i, 2 * i + 1, 2 * i, 2 * i, 2 * i, 2 * i + 1, 2 * i + 1, 2 * i + 1);
        } else {
            std::snprintf(b, sizeof b,
                          "f2(gd[%d], ge[%d], t.x, t.y, x[%d], x[%d]); f2(gd[%d], ge[%d], t.z, t.w, x[%d], x[%d]);\n"
                          "f2(gx[%d], gx[%d], t.x, t.y, x[%d], x[%d]); f2(gx[%d], gx[%d], t.z, t.w, x[%d], x[%d]); }\n",
                          2 * i, 2 * i, 2 * j, 2 * j + 1, 2 * i + 1, 2 * i + 1, 2 * j, 2 * j + 1,
                          2 * j, 2 * j + 1, 2 * i, 2 * i, 2 * j, 2 * j + 1, 2 * i + 1, 2 * i + 1);
        }
        o += b;
    }
    for (int i = 0; i + 1 < nb; ++i) { // rows with a direct part
        std::snprintf(b, sizeof b, "a2(gx[%d], gx[%d], gd[%d], gd[%d]); a2(gx[%d], gx[%d], ge[%d], ge[%d]);\n",
                      2 * i, 2 * i + 1, 2 * i, 2 * i + 1, 2 * i, 2 * i + 1, 2 * i, 2 * i + 1);
        o += b;
    }
    return o;
}

struct Term {
    int idx;
    float w;
};

// One layer: the live hidden units, then [v'; u2] in gather form, psi_t.
// Every product is an FFMA (FMUL for the first) with the weight as an FP32
// immediate; biases are added last as FADD immediates (skipped when zero),
// so no weight constant ever needs a register (a constant-initialised
// accumulator would be a loop-invariant MOV that ptxas hoists out of the
// layer loop and spills). A unit without W1 entries has the constant
// z = relu(b1): dead if b1 <= 0, else folded into the output biases.
std::string gen_layer(int l, int K, int Z, int V, const double *p, const double *mk, long &nnz) {
    const int IN = 3 * K + V;
    const long oW1 = 0, ob1 = static_cast<long>(Z) * IN, oW2 = ob1 + Z,
               ob2 = oW2 + static_cast<long>(K) * Z, oW3 = ob2 + K,
               ob3 = oW3 + static_cast<long>(V) * Z, ot = ob3 + V;
    auto w = [&](long off) { return static_cast<float>(p[off] * (mk ? mk[off] : 1.0)); };
    auto wout = [&](int r, int i) {
        return r < V ? w(oW3 + static_cast<long>(r) * Z + i) : w(oW2 + static_cast<long>(r - V) * Z + i);
    };
    std::string o;
    char b[200];
    std::snprintf(b, sizeof b, "case %d: {\n", l);
    o += b;
    std::vector<float> obias(V + K);
    for (int r = 0; r < V; ++r) obias[r] = w(ob3 + r);
    for (int k = 0; k < K; ++k) obias[V + k] = w(ob2 + k);
    // live units: a surviving outgoing weight (else the unit cannot matter)
    std::vector<int> live;
    for (int i = 0; i < Z; ++i) {
        bool any = false;
        for (int r = 0; r < V + K && !any; ++r) any = wout(r, i) != 0.f;
        if (!any) continue;
        bool has_in = false;
        for (int j = 0; j < IN && !has_in; ++j) has_in = w(oW1 + static_cast<long>(i) * IN + j) != 0.f;
        if (!has_in) { // constant unit
            const float zc = std::max(w(ob1 + i), 0.f);
            if (zc > 0.f)
                for (int r = 0; r < V + K; ++r) obias[r] = std::fmaf(wout(r, i), zc, obias[r]);
            continue;
        }
        live.push_back(i);
    }
    for (size_t u = 0; u < live.size(); ++u) {
        const int i = live[u], zu = static_cast<int>(u);
        bool first = true;
        for (int j = 0; j < IN; ++j) {
            const float wt = w(oW1 + static_cast<long>(i) * IN + j);
            if (wt == 0.f) continue;
            ++nnz;
            if (first) std::snprintf(b, sizeof b, "float z%d = %s * %s;", zu, in_name(j, K).c_str(), fimm(wt).c_str());
            else std::snprintf(b, sizeof b, " z%d = fmaf(%s, %s, z%d);", zu, in_name(j, K).c_str(), fimm(wt).c_str(), zu);
            o += b;
            first = false;
        }
        const float b1 = w(ob1 + i);
        if (b1 != 0.f) {
            std::snprintf(b, sizeof b, " z%d = z%d + %s;", zu, zu, fimm(b1).c_str());
            o += b;
        }
        std::snprintf(b, sizeof b, " z%d = relu(z%d);\n", zu, zu);
        o += b;
    }
    // outputs: v' rows (W3, b3) straight into v (its old values are consumed
    // above); u2 rows (W2, b2) pre-scaled by 1/t (FP64 product, one FP32
    // rounding), so psi_t(u) = clamp(u/t, -1, 1) (model.cpp:32-51; t > 0 is
    // checked at upload) is two FMNMX. (An offset form, 2 sat(u/2t + 1/2) - 1,
    // would quantise x near 0 to 2^-23 and flip the sign of tiny outputs.)
    const double tinv = 1.0 / p[ot];
    for (int r = 0; r < V + K; ++r) {
        const bool isv = r < V;
        const std::string acc = isv ? "v[" + std::to_string(r) + "]" : "u2[" + std::to_string(r - V) + "]";
        auto scaled = [&](float wt) { return isv ? wt : static_cast<float>(wt * tinv); };
        const float bias = isv ? obias[r] : static_cast<float>(obias[r] * tinv);
        bool first = true;
        for (size_t u = 0; u < live.size(); ++u) {
            const float wt = wout(r, live[u]);
            if (wt == 0.f) continue;
            ++nnz;
            if (first) std::snprintf(b, sizeof b, "%s = z%d * %s;", acc.c_str(), static_cast<int>(u), fimm(scaled(wt)).c_str());
            else std::snprintf(b, sizeof b, " %s = fmaf(z%d, %s, %s);", acc.c_str(), static_cast<int>(u), fimm(scaled(wt)).c_str(), acc.c_str());
            o += b;
            first = false;
        }
        if (first) { // no products: the bias alone, anchored to a layer-varying value
            if (bias == 0.f) o += acc + " = 0.f;";
            else o += acc + " = fmaf(x[0], 0.f, " + fimm(bias) + ");";
        } else if (bias != 0.f) {
            o += " " + acc + " = " + acc + " + " + fimm(bias) + ";";
        }
        o += "\n";
    }
    o += "#pragma unroll\nfor (int k = 0; k < K_; ++k) x[k] = fminf(fmaxf(u2[k], -1.f), 1.f);\n";
    o += "} break;\n";
    return o;
}

// Cubin caches keyed by the generated source (its 64-bit FNV-1a hash and
// length): per process (models rebuilt with the same weights, replicas on
// other devices, repeated tests; the 16 most recent) and on
// disk ($DETNET_JIT_CACHE, else $XDG_CACHE_HOME or ~/.cache /detnet_b200_jit;
// "off" disables it), so another process with the same model skips NVRTC
// (~13 s at L=40). A disk entry carries the source length and hash and the
// NVRTC version; anything that does not match is recompiled.
std::mutex g_jit_mu;
// in-memory: keyed by (source hash, length), the 16 most recent cubins
constexpr size_t kMemCacheEntries = 16;
std::map<std::pair<uint64_t, size_t>, std::vector<char>> g_jit_cache;
std::vector<std::pair<uint64_t, size_t>> g_jit_order; // insertion order, oldest first

void mem_store(const std::pair<uint64_t, size_t> &k, const std::vector<char> &cubin) {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    if (g_jit_cache.emplace(k, cubin).second) {
        g_jit_order.push_back(k);
        if (g_jit_order.size() > kMemCacheEntries) {
            g_jit_cache.erase(g_jit_order.front());
            g_jit_order.erase(g_jit_order.begin());
        }
    }
}

uint64_t fnv1a(const std::string &s) {
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
    return h;
}

std::string jit_cache_dir() {
    if (const char *d = std::getenv("DETNET_JIT_CACHE")) return std::strcmp(d, "off") ? d : "";
    if (const char *x = std::getenv("XDG_CACHE_HOME")) return std::string(x) + "/detnet_b200_jit";
    if (const char *h = std::getenv("HOME")) return std::string(h) + "/.cache/detnet_b200_jit";
    return "";
}

struct DiskKey {
    uint64_t len, hash;
    int major, minor;
};

bool disk_load(const std::string &path, const DiskKey &k, std::vector<char> &cubin) {
    FILE *f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    DiskKey h{};
    bool ok = std::fread(&h, sizeof h, 1, f) == 1 && h.len == k.len && h.hash == k.hash &&
              h.major == k.major && h.minor == k.minor;
    if (ok) {
        std::fseek(f, 0, SEEK_END);
        const long n = std::ftell(f) - static_cast<long>(sizeof h);
        std::fseek(f, sizeof h, SEEK_SET);
        ok = n > 0;
        if (ok) {
            cubin.resize(static_cast<size_t>(n));
            ok = std::fread(cubin.data(), 1, cubin.size(), f) == cubin.size();
        }
    }
    std::fclose(f);
    return ok;
}

void disk_store(const std::string &dir, const std::string &path, const DiskKey &k,
                const std::vector<char> &cubin) {
    std::string cmd_dir = dir; // mkdir -p, one level at a time
    for (size_t p = 1; p <= cmd_dir.size(); ++p)
        if (p == cmd_dir.size() || cmd_dir[p] == '/') mkdir(cmd_dir.substr(0, p).c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string(getpid());
    FILE *f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    const bool ok = std::fwrite(&k, sizeof k, 1, f) == 1 &&
                    std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
    std::fclose(f);
    if (ok) std::rename(tmp.c_str(), path.c_str()); // atomic: readers see all or nothing
    else std::remove(tmp.c_str());
}

int nvrtc_compile(const std::string &src, std::vector<char> &cubin, std::string &log) {
    const std::pair<uint64_t, size_t> mkey{fnv1a(src), src.size()};
    {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        auto it = g_jit_cache.find(mkey);
        if (it != g_jit_cache.end()) {
            cubin = it->second;
            return 0;
        }
    }
    DiskKey key{src.size(), mkey.first, 0, 0};
    nvrtcVersion(&key.major, &key.minor);
    const std::string dir = jit_cache_dir();
    char name[64];
    std::snprintf(name, sizeof name, "/%016llx.cubin", static_cast<unsigned long long>(key.hash));
    const std::string path = dir.empty() ? "" : dir + name;
    if (!path.empty() && disk_load(path, key, cubin)) {
        mem_store(mkey, cubin);
        return 0;
    }
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "detnet_sparse_jit.cu", 0, nullptr, nullptr) !=
        NVRTC_SUCCESS)
        return fail(DETNET_ERR_CUDA, "nvrtcCreateProgram failed");
    const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "--ptxas-options=-v"};
    const nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
    size_t ls = 0;
    nvrtcGetProgramLogSize(prog, &ls);
    log.assign(ls, '\0');
    if (ls) nvrtcGetProgramLog(prog, &log[0]);
    if (r != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return fail(DETNET_ERR_CUDA, "sparse JIT compile failed: %s: %.300s", nvrtcGetErrorString(r),
                    log.c_str());
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    cubin.resize(n);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    if (!path.empty()) disk_store(dir, path, key, cubin);
    mem_store(mkey, cubin);
    return 0;
}

} // namespace

// Worst layer's surviving products (W1 entries of live units + [W3; W2]
// entries): the per-sample cost of a layer in the JIT kernel. Returns early
// (with a value > stop) once a layer exceeds `stop`.
long jit_layer_nnz(int K, int Z, int V, int L, const double *params, const double *masks, long stop) {
    const long P = record_size(K, Z, V);
    const int IN = 3 * K + V;
    long worst = 0;
    for (int l = 0; l < L; ++l) {
        const double *p = params + l * P, *mk = masks ? masks + l * P : nullptr;
        auto nz = [&](long off) { return static_cast<float>(p[off] * (mk ? mk[off] : 1.0)) != 0.f; };
        const long ob1 = static_cast<long>(Z) * IN, oW2 = ob1 + Z, ob2 = oW2 + static_cast<long>(K) * Z,
                   oW3 = ob2 + K;
        long nnz = 0;
        for (int i = 0; i < Z; ++i) {
            long out = 0;
            for (int r = 0; r < V; ++r) out += nz(oW3 + static_cast<long>(r) * Z + i);
            for (int k = 0; k < K; ++k) out += nz(oW2 + static_cast<long>(k) * Z + i);
            if (!out) continue;
            nnz += out;
            for (int j = 0; j < IN; ++j) nnz += nz(static_cast<long>(i) * IN + j);
            if (nnz > stop) return nnz; // over the limit: the exact count is not needed
        }
        worst = std::max(worst, nnz);
    }
    return worst;
}

int jit_build(JitModel &jm, int K, int Z, int V, int L, const double *params, const double *masks) {
    jit_release(jm);
    if (K > 32) return fail(DETNET_ERR_UNSUPPORTED, "sparse JIT: n_tx > 32");
    const long P = record_size(K, Z, V);
    const int nb = (K + 1) / 2, nblk = nb * (nb + 1) / 2;
    // Gram blocks kept in registers (DETNET_JIT_GREG entries, 4 per block);
    // the rest in shared memory, two CTAs per SM
    const char *ge = std::getenv("DETNET_JIT_GREG");
    const int gb = std::max(0, std::min(nblk, (ge ? std::atoi(ge) : 64) / 4));
    const int ns = nblk - gb;
    const size_t smem = static_cast<size_t>(std::max(ns, 1)) * 128 * 16;
    const int ctas = smem <= 110 * 1024 ? 2 : 1;
    std::string layers;
    long nnz = 0;
    for (int l = 0; l < L; ++l)
        layers += gen_layer(l, K, Z, V, params + l * P, masks ? masks + l * P : nullptr, nnz);
    std::string src = kSkeleton;
    replace_all(src, "@K@", std::to_string(K));
    replace_all(src, "@KP@", std::to_string(2 * nb));
    replace_all(src, "@V@", std::to_string(V));
    replace_all(src, "@GB@", std::to_string(gb));
    replace_all(src, "@CTAS@", std::to_string(ctas));
    replace_all(src, "@STAGE@", gen_stage(K, gb));
    replace_all(src, "@GRAM@", gen_gram(K, gb));
    replace_all(src, "@LAYERS@", layers);
    if (const char *dump = std::getenv("DETNET_JIT_DUMP")) {
        if (FILE *f = std::fopen(dump, "w")) {
            std::fputs(src.c_str(), f);
            std::fclose(f);
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<char> cubin;
    std::string log;
    if (int rc = nvrtc_compile(src, cubin, log)) return rc;
    jm.compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    jm.log = log;
    cudaLibrary_t lib;
    CK(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    cudaKernel_t k;
    if (cudaLibraryGetKernel(&k, lib, "detnet_sparse_jit") != cudaSuccess) {
        cudaLibraryUnload(lib);
        return fail(DETNET_ERR_CUDA, "sparse JIT: kernel symbol missing");
    }
    jm.lib = lib;
    jm.kernel = k;
    jm.smem = smem;
    jm.ctas_per_sm = ctas;
    jm.L = L;
    jm.K = K;
    jm.nnz = nnz;
    jm.attr_device = -1;
    jm.ready = true;
    return 0;
}

int jit_launch(JitModel &jm, const TcArgs &a, cudaStream_t st, int sms, int device) {
    if (!jm.ready) return fail(DETNET_ERR_UNSUPPORTED, "sparse JIT kernel not built");
    if (a.l_begin != 0 || a.l_end > jm.L) return fail(DETNET_ERR_UNSUPPORTED, "sparse JIT: layer range");
    const void *fn = reinterpret_cast<const void *>(jm.kernel);
    if (jm.attr_device != device) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(jm.smem)));
        jm.attr_device = device;
    }
    struct JArgs {
        const float *gp;
        const float *q32;
        const double *denom;
        const uint32_t *xmask;
        const double *lnk;
        int l_end;
        long n, n_tiles, tile0;
        float *xhat;
        double *tile_loss;
        long long *tile_err;
    } ja{a.gp, a.q32, a.denom, a.xmask, a.lnk, a.l_end, a.n, a.n_tiles, a.tile0, a.xhat,
         a.tile_loss, a.tile_err};
    void *args[] = {&ja};
    const long grid = std::min<long>(a.n_tiles, static_cast<long>(sms) * jm.ctas_per_sm);
    if (grid <= 0) return 0;
    CK(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(128), args, jm.smem, st));
    return 0;
}

void jit_release(JitModel &jm) {
    if (jm.lib) cudaLibraryUnload(jm.lib);
    jm = JitModel{};
}

} // namespace detnet
