// elementwise_f64.cu -- modular vector operations over IEEE doubles (paper §3,
// P:558-762): residues of a prime p < 2^50 stored as
// integral doubles, reduced with the FP64 FMA pipe instead of integer
// multiplies.
//
//   modadd : Function 17: a = x + y, b = a - p, b < 0 ? a : b
//            (the sign test replaces _mm_blendv_pd);
//   modsub : the same with a = x - y, b = a + p, a < 0 ? b : a;
//   modmul : Function 16 / 18 for m <= l - 2 = 50:
//            h = x y, l = fma(x, y, -h) (exact: h + l = x y), b = h u with
//            u = 1.0 / p, c = floor(b), d = fma(-c, p, h), e = d + l, then
//            one correction each way (Proposition 13: c - floor(x y / p) in
//            {-1, 0, 1}).
// Every floating operation uses an explicit round-to-nearest intrinsic so that
// the compiler neither contracts nor reorders the sequence the proof covers.
#include "common.h"
#include <math.h>
#include <new>

struct mm_modf64 {
    uint64_t p;
    double pd, u;   // (double) p, 1.0 / p rounded to nearest ("u")
};

namespace mm {

enum OpF { OPF_ADD, OPF_SUB, OPF_MUL };

struct ModF64 {
    double p, u;
};

template <int OP>
__device__ __forceinline__ double apply_f64(const ModF64& m, double x, double y) {
    if (OP == OPF_ADD) {              // Function 17
        const double a = __dadd_rn(x, y);
        const double b = __dsub_rn(a, m.p);
        return b < 0.0 ? a : b;
    }
    if (OP == OPF_SUB) {
        const double a = __dsub_rn(x, y);
        const double b = __dadd_rn(a, m.p);
        return a < 0.0 ? b : a;
    }
    // Function 16
    const double h = __dmul_rn(x, y);
    const double l = __fma_rn(x, y, -h);
    const double b = __dmul_rn(h, m.u);
    const double c = floor(b);
    const double d = __fma_rn(-c, m.p, h);
    double e = __dadd_rn(d, l);
    if (e >= m.p) e = __dsub_rn(e, m.p);
    if (e < 0.0) e = __dadd_rn(e, m.p);
    return e;
}

constexpr int F64_THREADS = 256;

template <int OP>
__global__ void __launch_bounds__(F64_THREADS) k_ew_f64(ModF64 m, const double2* __restrict__ x,
                                                         const double2* __restrict__ y, double2* __restrict__ z,
                                                         long long nv) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
        const double2 a = x[i], b = y[i];
        z[i] = make_double2(apply_f64<OP>(m, a.x, b.x), apply_f64<OP>(m, a.y, b.y));
    }
}
template <int OP>
__global__ void __launch_bounds__(F64_THREADS) k_ew_f64_tail(ModF64 m, const double* __restrict__ x,
                                                             const double* __restrict__ y, double* __restrict__ z,
                                                             long long i0, long long n) {
    const long long i = i0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) z[i] = apply_f64<OP>(m, x[i], y[i]);
}

static const char* f64_name(int op) {
    static const char* names[] = {"modadd_f64", "modsub_f64", "modmul_f64"};
    return names[op];
}

template <int OP>
static mm_status run_f64(const mm_modf64* c, const double* x, const double* y, double* z, size_t n, cudaStream_t st) {
    if (!c) return set_err(MM_E_ARG, "null context");
    if (n == 0) return MM_OK;
    if (!x || !y || !z) return set_err(MM_E_ARG, "null vector");
    const ModF64 m{c->pd, c->u};
    const bool vec = (((uintptr_t)x | (uintptr_t)y | (uintptr_t)z) & 15) == 0;
    const long long nv = vec ? (long long)(n / 2) : 0;
    {
        LaunchScope ls(f64_name(OP), st);
        if (nv > 0) {
            long long blocks = (nv + F64_THREADS - 1) / F64_THREADS;
            const long long cap = (long long)num_sms() * 16;
            k_ew_f64<OP><<<(int)(blocks < cap ? blocks : cap), F64_THREADS, 0, st>>>(
                m, (const double2*)x, (const double2*)y, (double2*)z, nv);
        }
        const long long i0 = 2 * nv, rest = (long long)n - i0;
        if (rest > 0)
            k_ew_f64_tail<OP><<<(int)((rest + F64_THREADS - 1) / F64_THREADS), F64_THREADS, 0, st>>>(m, x, y, z, i0,
                                                                                                 (long long)n);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

}  // namespace mm

using namespace mm;

extern "C" mm_status mm_modf64_create(uint64_t p, mm_modf64** ctx) {
    if (!ctx) return set_err(MM_E_ARG, "ctx is null");
    *ctx = nullptr;
    if (p < 3 || !(p & 1)) return set_err(MM_E_INVALID_MODULUS, "p=%llu must be an odd integer >= 3", (unsigned long long)p);
    if (p >= (1ull << 50))
        return set_err(MM_E_PROFILE, "FP64 products need m <= l - 2 = 50 bits (Function 16), got p=%llu",
                       (unsigned long long)p);
    mm_modf64* c = new (std::nothrow) mm_modf64;
    if (!c) return set_err(MM_E_ARG, "out of host memory");
    c->p = p;
    c->pd = (double)p;        // exact: p < 2^53
    c->u = 1.0 / c->pd;       // host rounding mode: to nearest
    *ctx = c;
    return MM_OK;
}
extern "C" void mm_modf64_destroy(mm_modf64* ctx) { delete ctx; }

extern "C" mm_status mm_modadd_f64(const mm_modf64* c, const double* x, const double* y, double* z, size_t n, void* st) {
    return run_f64<OPF_ADD>(c, x, y, z, n, (cudaStream_t)st);
}
extern "C" mm_status mm_modsub_f64(const mm_modf64* c, const double* x, const double* y, double* z, size_t n, void* st) {
    return run_f64<OPF_SUB>(c, x, y, z, n, (cudaStream_t)st);
}
extern "C" mm_status mm_modmul_f64(const mm_modf64* c, const double* x, const double* y, double* z, size_t n, void* st) {
    return run_f64<OPF_MUL>(c, x, y, z, n, (cudaStream_t)st);
}
