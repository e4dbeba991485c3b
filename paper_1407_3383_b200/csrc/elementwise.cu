// elementwise.cu -- C2: vector modadd / modsub / modmul over uint32 residues.
//
// One grid-stride kernel per operation; each thread moves 128-bit vectors
// (4 residues) with UNROLL independent loads in flight (HBM-bound: 12 or 16
// bytes per element against ~10 integer instructions).  The modular kernels
// are the paper's Functions 2/4 (sum), 6 (Barrett), 8 (fixed multiplicand)
// and 13 (Montgomery), with the m = n vs m <= n-1 choice made once per
// modulus on the host (n, m fixed at compile time, p at run time).
#include "common.h"
#include "arith.cuh"
#include <new>

struct mm_mod32 {
    uint32_t p;
    int r;               // 2^(r-1) < p <= 2^r
    int full;            // 1 if m = n = 32 (2p > 2^32 possible): full-range forms
    mm::Barrett32 bar;   // Table 3 profile
    uint32_t pinv;       // p^-1 mod 2^32
    uint32_t r2;         // 2^64 mod p
};

namespace mm {

enum Op { OP_ADD, OP_SUB, OP_MUL_BARRETT, OP_MUL_SHOUP, OP_MUL_MONT, OP_SHOUP_PRE, OP_TO_MONT, OP_FROM_MONT };

struct ModDev {
    uint32_t p, pinv, r2;
    Barrett32 bar;
    uint64_t mu;         // floor(2^64 / p): the Shoup companion without a division
};

template <int OP, bool FULL>
__device__ __forceinline__ uint32_t apply(const ModDev& m, uint32_t x, uint32_t y, uint32_t ys) {
    if (OP == OP_ADD) return FULL ? add_full(x, y, m.p) : add_half(x, y, m.p);
    if (OP == OP_SUB) return FULL ? sub_full(x, y, m.p) : sub_half(x, y, m.p);
    if (OP == OP_MUL_BARRETT) return FULL ? mul_barrett_full(x, y, m.p, m.bar.q) : mul_barrett(x, y, m.bar);
    if (OP == OP_MUL_SHOUP) return FULL ? mul_shoup_full(x, y, ys, m.p) : [&] {
        uint32_t d = mul_shoup_lazy(x, y, ys, m.p);
        return umin32(d, d - m.p);
    }();
    if (OP == OP_MUL_MONT) return mul_mont(x, y, m.p, m.pinv);
    if (OP == OP_SHOUP_PRE) {   // psi = floor(y 2^32 / p) by a reciprocal: q = hi(a mu) <= floor(a / p) <= q + 1
        const uint64_t a = (uint64_t)y << 32;
        uint64_t q = __umul64hi(a, m.mu);
        return (uint32_t)(a - q * m.p >= m.p ? q + 1 : q);
    }
    if (OP == OP_TO_MONT) return mul_mont(x, m.r2, m.p, m.pinv);            // x 2^32 mod p
    return mul_mont(x, 1u, m.p, m.pinv);                                    // OP_FROM_MONT
}

static const char* op_name(int op) {
    static const char* names[] = {"modadd", "modsub", "modmul_barrett", "modmul_shoup", "modmul_montgomery",
                                  "shoup_precompute", "to_mont", "from_mont"};
    return names[op];
}

template <int OP> struct OpUses { enum { X = OP != OP_SHOUP_PRE, Y = OP <= OP_MUL_MONT || OP == OP_SHOUP_PRE, YS = OP == OP_MUL_SHOUP }; };

constexpr int EW_THREADS = 256;
constexpr int EW_UNROLL = 4;

// A thread loads, computes and stores in turn, so HBM stays busy only while
// enough other warps are in their load phase: registers are held to five
// CTAs per SM (48; the Shoup precompute 0.82 -> 0.91 of HBM, the others
// unchanged within noise), except for the full-range Shoup product, whose three operand
// streams keep HBM busy at three CTAs per SM and which spills at 48 (0.65 ->
// 0.80 ms).  Two vectors per round at six CTAs per SM made the full-range
// Barrett and Shoup products slower (0.55 -> 0.60 ms, 0.65 -> 0.68 ms).
template <int OP> struct EwMinBlocks { enum { v = OP == OP_MUL_SHOUP ? 1 : 5 }; };
template <int OP> struct EwUnroll { enum { v = EW_UNROLL }; };

template <int OP, bool FULL>
__global__ void __launch_bounds__(EW_THREADS, EwMinBlocks<OP>::v) k_elementwise_v4(ModDev m, const uint4* __restrict__ x,
                                                               const uint4* __restrict__ y,
                                                               const uint4* __restrict__ ys,
                                                               uint4* __restrict__ z, size_t nv) {
    constexpr int U = EwUnroll<OP>::v;
    size_t stride = (size_t)gridDim.x * EW_THREADS * U;
    for (size_t base = (size_t)blockIdx.x * EW_THREADS * U + threadIdx.x; base < nv; base += stride) {
        uint4 vx[U], vy[U], vs[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            size_t i = base + (size_t)u * EW_THREADS;
            if (i < nv) {
                if (OpUses<OP>::X) vx[u] = __ldcs(x + i);
                if (OpUses<OP>::Y) vy[u] = __ldcs(y + i);
                if (OpUses<OP>::YS) vs[u] = __ldcs(ys + i);
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            size_t i = base + (size_t)u * EW_THREADS;
            if (i < nv) {
                uint4 r;
                r.x = apply<OP, FULL>(m, vx[u].x, vy[u].x, vs[u].x);
                r.y = apply<OP, FULL>(m, vx[u].y, vy[u].y, vs[u].y);
                r.z = apply<OP, FULL>(m, vx[u].z, vy[u].z, vs[u].z);
                r.w = apply<OP, FULL>(m, vx[u].w, vy[u].w, vs[u].w);
                __stcs(z + i, r);
            }
        }
    }
}

template <int OP, bool FULL>
__global__ void k_elementwise_scalar(ModDev m, const uint32_t* __restrict__ x, const uint32_t* __restrict__ y,
                                     const uint32_t* __restrict__ ys, uint32_t* __restrict__ z, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t a = OpUses<OP>::X ? x[i] : 0, b = OpUses<OP>::Y ? y[i] : 0, c = OpUses<OP>::YS ? ys[i] : 0;
        z[i] = apply<OP, FULL>(m, a, b, c);
    }
}

// debug range check (MMNTT_DEBUG=1): count inputs >= p
__global__ void k_range_count(const uint32_t* __restrict__ x, size_t n, uint32_t p, unsigned long long* bad) {
    unsigned long long local = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        local += x[i] >= p;
    if (local) atomicAdd(bad, local);
}

static mm_status range_check(const uint32_t* v, size_t n, uint32_t p, cudaStream_t st) {
    if (!v || !n) return MM_OK;
    unsigned long long* d = nullptr;
    unsigned long long h = 0;
    MM_CUDA_TRY(alloc_async((void**)&d, sizeof(*d), st));
    MM_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(*d), st));
    {
        LaunchScope ls("range_check", st);
        k_range_count<<<num_sms() * 4, 256, 0, st>>>(v, n, p, d);
    }
    MM_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    MM_CUDA_TRY(cudaFreeAsync(d, st));
    MM_CUDA_TRY(cudaStreamSynchronize(st));
    if (h) return set_err(MM_E_RANGE, "%llu input residues >= p", h);
    return MM_OK;
}

template <int OP, bool FULL>
static mm_status launch(const mm_mod32* c, const uint32_t* x, const uint32_t* y, const uint32_t* ys, uint32_t* z,
                        size_t n, cudaStream_t st) {
    ModDev m{c->p, c->pinv, c->r2, c->bar, (uint64_t)(((unsigned __int128)1 << 64) / c->p)};
    bool aligned = ((uintptr_t)x | (uintptr_t)y | (uintptr_t)ys | (uintptr_t)z) % 16 == 0;
    size_t nv = aligned ? n / 4 : 0;
    if (nv) {
        size_t want = (nv + EW_THREADS * EwUnroll<OP>::v - 1) / (EW_THREADS * EwUnroll<OP>::v);
        size_t cap = (size_t)num_sms() * 8;
        int grid = (int)(want < cap ? want : cap);
        LaunchScope ls(op_name(OP), st);
        k_elementwise_v4<OP, FULL><<<grid, EW_THREADS, 0, st>>>(m, (const uint4*)x, (const uint4*)y, (const uint4*)ys,
                                                                (uint4*)z, nv);
        MM_LAUNCH_CHECK();
    }
    size_t done = nv * 4;
    if (done < n) {
        size_t rem = n - done;
        int grid = (int)((rem + 255) / 256 < (size_t)num_sms() * 8 ? (rem + 255) / 256 : num_sms() * 8);
        LaunchScope ls("elementwise_tail", st);
        k_elementwise_scalar<OP, FULL><<<grid, 256, 0, st>>>(m, x ? x + done : x, y ? y + done : y,
                                                             ys ? ys + done : ys, z + done, rem);
        MM_LAUNCH_CHECK();
    }
    return MM_OK;
}

template <int OP>
static mm_status run(const mm_mod32* c, const uint32_t* x, const uint32_t* y, const uint32_t* ys, uint32_t* z,
                     size_t n, void* stream) {
    if (!c) return set_err(MM_E_ARG, "null context");
    if (n == 0) return MM_OK;   // empty vectors: nothing to do (pointers may be null)
    if (!z || (OpUses<OP>::X && !x) || (OpUses<OP>::Y && !y) || (OpUses<OP>::YS && !ys))
        return set_err(MM_E_ARG, "null pointer argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (OpUses<OP>::YS && ys == z) return set_err(MM_E_ALIAS, "y_shoup may not alias z");
    if (debug_checks()) {
        mm_status s;
        if (OpUses<OP>::X && (s = range_check(x, n, c->p, st)) != MM_OK) return s;
        if (OpUses<OP>::Y && (s = range_check(y, n, c->p, st)) != MM_OK) return s;
    }
    return c->full ? launch<OP, true>(c, x, y, ys, z, n, st) : launch<OP, false>(c, x, y, ys, z, n, st);
}

}  // namespace mm

using namespace mm;

extern "C" mm_status mm_mod32_create(uint32_t p, mm_mod32** ctx) {
    if (!ctx) return set_err(MM_E_ARG, "ctx is null");
    *ctx = nullptr;
    if (p < 3 || !(p & 1) || !hprime(p)) return set_err(MM_E_INVALID_MODULUS, "p=%u must be an odd prime >= 3", p);
    mm_mod32* c = new (std::nothrow) mm_mod32;
    if (!c) return set_err(MM_E_ARG, "out of host memory");
    c->p = p;
    int r = 0;
    while (r < 32 && (1ull << r) < p) r++;
    c->r = r;
    c->full = r >= 32 ? 1 : 0;   // m = n: the sum x + y may overflow U (Function 1 line 2)
    // Table 3 with n = 32, choosing the best column p admits.
    int n = 32, s, t, h;
    if (r <= n - 2) { s = r - 2 > 0 ? r - 2 : 0; t = n + 1; h = 1; }
    else if (r <= n - 1) { s = r - 1; t = n; h = 2; }
    else { s = r - 1; t = n; h = 3; }
    c->bar.p = p;
    c->bar.s = s;
    c->bar.t = t;
    c->bar.h = h;
    c->bar.q = (uint32_t)(((u128)1 << (s + t)) / p);          // q = floor(2^(s+t)/p)
    c->pinv = inv_mod_2_32(p);
    c->r2 = (uint32_t)(((u128)1 << 64) % p);
    *ctx = c;
    return MM_OK;
}

extern "C" void mm_mod32_destroy(mm_mod32* ctx) { delete ctx; }

extern "C" mm_status mm_mod32_info(const mm_mod32* c, uint64_t out[8]) {
    if (!c || !out) return set_err(MM_E_ARG, "null argument");
    out[0] = c->p; out[1] = c->r; out[2] = c->bar.s; out[3] = c->bar.t;
    out[4] = c->bar.h; out[5] = c->bar.q; out[6] = c->pinv; out[7] = c->r2;
    return MM_OK;
}

extern "C" mm_status mm_modadd_u32(const mm_mod32* c, const uint32_t* x, const uint32_t* y, uint32_t* z, size_t n,
                                   void* st) {
    return run<OP_ADD>(c, x, y, nullptr, z, n, st);
}
extern "C" mm_status mm_modsub_u32(const mm_mod32* c, const uint32_t* x, const uint32_t* y, uint32_t* z, size_t n,
                                   void* st) {
    return run<OP_SUB>(c, x, y, nullptr, z, n, st);
}
extern "C" mm_status mm_modmul_u32(const mm_mod32* c, mm_mul_variant v, const uint32_t* x, const uint32_t* y,
                                   const uint32_t* ys, uint32_t* z, size_t n, void* st) {
    switch (v) {
        case MM_MUL_BARRETT: return run<OP_MUL_BARRETT>(c, x, y, nullptr, z, n, st);
        case MM_MUL_SHOUP: return run<OP_MUL_SHOUP>(c, x, y, ys, z, n, st);
        case MM_MUL_MONTGOMERY: return run<OP_MUL_MONT>(c, x, y, nullptr, z, n, st);
    }
    return set_err(MM_E_ARG, "bad mm_mul_variant %d", (int)v);
}
extern "C" mm_status mm_shoup_precompute_u32(const mm_mod32* c, const uint32_t* y, uint32_t* ys, size_t n, void* st) {
    return run<OP_SHOUP_PRE>(c, nullptr, y, nullptr, ys, n, st);
}
extern "C" mm_status mm_to_mont_u32(const mm_mod32* c, const uint32_t* x, uint32_t* z, size_t n, void* st) {
    return run<OP_TO_MONT>(c, x, nullptr, nullptr, z, n, st);
}
extern "C" mm_status mm_from_mont_u32(const mm_mod32* c, const uint32_t* x, uint32_t* z, size_t n, void* st) {
    return run<OP_FROM_MONT>(c, x, nullptr, nullptr, z, n, st);
}
