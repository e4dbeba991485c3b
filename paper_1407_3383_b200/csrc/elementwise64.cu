// elementwise64.cu -- vector modadd / modsub / modmul over 64-bit residues of
// p = 2^64 - 2^32 + 1 (SURVEY §8(b) mm_mod64_create, "first build: p =
// 2^64 - 2^32 + 1 only"; the 64-bit modulus of BASELINE C4 / C5).
//
// The reduction is the special one of SURVEY O9 / DESIGN R11 (not in the
// paper, which stops at m = n = 64 with generic Barrett / Montgomery,
// P:244-556): 2^64 = 2^32 - 1 and 2^96 = -1 mod p, so a 128-bit product
// x = r0 + r1 2^32 + r2 2^64 + r3 2^96 reduces to (r1:r0) - r3 + r2 (2^32 - 1)
// with carry / borrow folds (FpG::mul, arith.cuh); sums fold each carry out of
// 2^64 as 2^32 - 1.  Outputs are canonical in [0, p).
#include "common.h"
#include "arith.cuh"
#include <new>

struct mm_mod64 {
    uint64_t p;
};

namespace mm {

enum Op64 { OP64_ADD, OP64_SUB, OP64_MUL };

template <int OP>
__device__ __forceinline__ uint64_t apply64(uint64_t x, uint64_t y) {
    if (OP == OP64_ADD) return FpG::canon(FpG::add(x, y));
    if (OP == OP64_SUB) return FpG::canon(FpG::sub(x, y));
    return FpG::canon(FpG::mul(x, y));
}

constexpr int E64_T = 256;

// two 16-byte vectors (4 residues) per thread per iteration, streaming loads
template <int OP>
__global__ void __launch_bounds__(E64_T) k_ew64(const ulonglong2* __restrict__ x, const ulonglong2* __restrict__ y,
                                                ulonglong2* __restrict__ z, long long nv) {
    for (long long i = (long long)blockIdx.x * E64_T + threadIdx.x; i < nv; i += (long long)gridDim.x * E64_T) {
        const ulonglong2 a = __ldcs(x + i), b = __ldcs(y + i);
        __stcs(z + i, make_ulonglong2(apply64<OP>(a.x, b.x), apply64<OP>(a.y, b.y)));
    }
}
template <int OP>
__global__ void __launch_bounds__(E64_T) k_ew64_tail(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y,
                                                     uint64_t* __restrict__ z, long long i0, long long n) {
    const long long i = i0 + (long long)blockIdx.x * E64_T + threadIdx.x;
    if (i < n) z[i] = apply64<OP>(x[i], y[i]);
}
__global__ void k_range64(const uint64_t* __restrict__ x, long long n, unsigned* bad) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (x[i] >= FpG::P) atomicAdd(bad, 1u);
}

static mm_status range64(const uint64_t* x, size_t n, cudaStream_t st) {
    unsigned* bad = nullptr;
    MM_CUDA_TRY(alloc_async((void**)&bad, sizeof(unsigned), st));
    MM_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned), st));
    {
        LaunchScope ls("debug_range_check", st);
        k_range64<<<num_sms() * 4, 256, 0, st>>>(x, (long long)n, bad);
    }
    unsigned h = 0;
    MM_CUDA_TRY(cudaMemcpyAsync(&h, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    MM_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFreeAsync(bad, st);
    if (h) return set_err(MM_E_RANGE, "%u inputs >= p", h);
    return MM_OK;
}

template <int OP>
static mm_status run64(const mm_mod64* c, const uint64_t* x, const uint64_t* y, uint64_t* z, size_t n, cudaStream_t st) {
    static const char* names[] = {"modadd_u64", "modsub_u64", "modmul_u64"};
    if (!c) return set_err(MM_E_ARG, "null context");
    if (n == 0) return MM_OK;
    if (!x || !y || !z) return set_err(MM_E_ARG, "null vector");
    if (debug_checks()) {
        mm_status s;
        if ((s = range64(x, n, st)) != MM_OK || (s = range64(y, n, st)) != MM_OK) return s;
    }
    const bool vec = (((uintptr_t)x | (uintptr_t)y | (uintptr_t)z) & 15) == 0;
    const long long nv = vec ? (long long)(n / 2) : 0;
    LaunchScope ls(names[OP], st);
    if (nv > 0) {
        const long long blocks = (nv + E64_T - 1) / E64_T, cap = (long long)num_sms() * 16;
        k_ew64<OP><<<(int)(blocks < cap ? blocks : cap), E64_T, 0, st>>>((const ulonglong2*)x, (const ulonglong2*)y,
                                                                         (ulonglong2*)z, nv);
    }
    const long long i0 = 2 * nv, rest = (long long)n - i0;
    if (rest > 0) k_ew64_tail<OP><<<(int)((rest + E64_T - 1) / E64_T), E64_T, 0, st>>>(x, y, z, i0, (long long)n);
    MM_LAUNCH_CHECK();
    return MM_OK;
}

}  // namespace mm

using namespace mm;

extern "C" mm_status mm_mod64_create(uint64_t p, mm_mod64** ctx) {
    if (!ctx) return set_err(MM_E_ARG, "ctx is null");
    *ctx = nullptr;
    if (p != FpG::P) return set_err(MM_E_INVALID_MODULUS, "64-bit contexts support only p = 2^64 - 2^32 + 1");
    mm_mod64* c = new (std::nothrow) mm_mod64;
    if (!c) return set_err(MM_E_ARG, "out of host memory");
    c->p = p;
    *ctx = c;
    return MM_OK;
}
extern "C" void mm_mod64_destroy(mm_mod64* ctx) { delete ctx; }
extern "C" mm_status mm_modadd_u64(const mm_mod64* c, const uint64_t* x, const uint64_t* y, uint64_t* z, size_t n,
                                   void* st) {
    return run64<OP64_ADD>(c, x, y, z, n, (cudaStream_t)st);
}
extern "C" mm_status mm_modsub_u64(const mm_mod64* c, const uint64_t* x, const uint64_t* y, uint64_t* z, size_t n,
                                   void* st) {
    return run64<OP64_SUB>(c, x, y, z, n, (cudaStream_t)st);
}
extern "C" mm_status mm_modmul_u64(const mm_mod64* c, const uint64_t* x, const uint64_t* y, uint64_t* z, size_t n,
                                   void* st) {
    return run64<OP64_MUL>(c, x, y, z, n, (cudaStream_t)st);
}
