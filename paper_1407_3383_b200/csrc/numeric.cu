// numeric.cu -- modular reductions in IEEE float / double (paper §3,
// P:558-762): Functions 14, 15 and 16 with the rounding
// variants of Propositions 10, 11, 13 and Remark 12, on the FP32 / FP64 pipes.
//
// l = trailing field size (23 float, 52 double), m = bit size of p (p < 2^m),
// u = 1.0 / p rounded to nearest, u-bar = 1.0 / p rounded toward +inf.
//   F14     (m <= l/2):     b = a u, c = floor(b), d = a - c p,
//                                      d >= p -> d - p, d < 0 -> d + p  (Prop. 10)
//   F14_UP  (Prop. 10, 2nd clause):    u-bar, every op rounded toward +inf,
//                                      line 4 (d >= p) dropped
//   F15_UP  (m <= (l-1)/2): u-bar, toward +inf, no correction (Prop. 11)
//   F15_NEAR (Remark 12):              the same in round-to-nearest; only for
//                                      p prime and a = x y with x, y residues
//   F16     (m <= l - 2):   h = x y, l = fma(x, y, -h), c = floor(h u),
//                                      d = fma(-c, p, h), e = d + l, two corrections
//   F16_UP  (Prop. 13, 2nd clause):    u-bar, toward +inf, line 7 dropped
// Each floating operation is an explicit rounding-mode intrinsic
// (__dmul_rn / __dmul_ru, __fma_ru, ...) -- the GPU has per-instruction
// rounding, so "the current rounding mode" of the paper is a property of the
// instruction, and the compiler cannot contract or reorder what the proofs
// cover.  Products x y for F14 / F15 are exact (2m <= l), so the vector
// product z = (x y) rem p is Function 14 / 15 applied to a = x y.
#include "common.h"
#include <math.h>
#include <new>

struct mm_modnum {
    int fbits;            // 32 or 64
    uint64_t p;
    int m;                // p < 2^m
    double pd, u, ub;     // double: p, u, u-bar
    float pf, uf, ubf;    // float
};

namespace mm {

template <class F> struct NumOps;
template <> struct NumOps<double> {
    static __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double mul_ru(double a, double b) { return __dmul_ru(a, b); }
    static __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double add_ru(double a, double b) { return __dadd_ru(a, b); }
    static __device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double sub_ru(double a, double b) { return __dsub_ru(a, b); }
    static __device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
    static __device__ __forceinline__ double fma_ru(double a, double b, double c) { return __fma_ru(a, b, c); }
    static __device__ __forceinline__ double flr(double a) { return floor(a); }
};
template <> struct NumOps<float> {
    static __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float mul_ru(float a, float b) { return __fmul_ru(a, b); }
    static __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float add_ru(float a, float b) { return __fadd_ru(a, b); }
    static __device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float sub_ru(float a, float b) { return __fsub_ru(a, b); }
    static __device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
    static __device__ __forceinline__ float fma_ru(float a, float b, float c) { return __fmaf_ru(a, b, c); }
    static __device__ __forceinline__ float flr(float a) { return floorf(a); }
};

template <class F> struct NumMod {
    F p, u, ub;
};

// Function 14 (and its Prop. 10 toward-+inf form) on an integral a < alpha p
template <class F, bool UP>
__device__ __forceinline__ F fn14(const NumMod<F>& M, F a) {
    typedef NumOps<F> O;
    if (UP) {
        const F b = O::mul_ru(a, M.ub);               // 1. b = a * u-bar
        const F c = O::flr(b);                        // 2. c = floor(b)
        const F d = O::sub_ru(a, O::mul_ru(c, M.p));  // 3. d = a - c * p
        return d < F(0) ? O::add_ru(d, M.p) : d;      // 5. (line 4 discarded, Prop. 10)
    }
    const F b = O::mul_rn(a, M.u);
    const F c = O::flr(b);
    const F d = O::sub_rn(a, O::mul_rn(c, M.p));
    if (d >= M.p) return O::sub_rn(d, M.p);           // 4.
    if (d < F(0)) return O::add_rn(d, M.p);           // 5.
    return d;                                         // 6.
}
// Function 15: u-bar, no correction.  UP: toward +inf (Prop. 11); else to
// nearest (Remark 12: a a product of residues of a prime p)
template <class F, bool UP>
__device__ __forceinline__ F fn15(const NumMod<F>& M, F a) {
    typedef NumOps<F> O;
    const F b = UP ? O::mul_ru(a, M.ub) : O::mul_rn(a, M.ub);   // 1. b = a * u-bar
    const F c = O::flr(b);                                      // 2. c = floor(b)
    return UP ? O::sub_ru(a, O::mul_ru(c, M.p)) : O::sub_rn(a, O::mul_rn(c, M.p));   // 3.
}
// Function 16 (and its Prop. 13 toward-+inf form, line 7 dropped)
template <class F, bool UP>
__device__ __forceinline__ F fn16(const NumMod<F>& M, F x, F y) {
    typedef NumOps<F> O;
    if (UP) {
        const F h = O::mul_ru(x, y);                 // 1. h = a1 * a2
        const F l = O::fma_ru(x, y, -h);             // 2. l = fma(a1, a2, -h)
        const F b = O::mul_ru(h, M.ub);              // 3. b = h * u-bar
        const F c = O::flr(b);                       // 4. c = floor(b)
        const F d = O::fma_ru(-c, M.p, h);           // 5. d = fma(-c, p, h)
        const F e = O::add_ru(d, l);                 // 6. e = d + l
        return e < F(0) ? O::add_ru(e, M.p) : e;     // 8. (line 7 discarded, Prop. 13)
    }
    const F h = O::mul_rn(x, y);
    const F l = O::fma_rn(x, y, -h);
    const F b = O::mul_rn(h, M.u);
    const F c = O::flr(b);
    const F d = O::fma_rn(-c, M.p, h);
    const F e = O::add_rn(d, l);
    if (e >= M.p) return O::sub_rn(e, M.p);          // 7.
    if (e < F(0)) return O::add_rn(e, M.p);          // 8.
    return e;                                        // 9.
}

// MUL: z = (x y) rem p; else z = a rem p (x = a, y unused)
template <class F, int V, bool MUL>
__device__ __forceinline__ F num_apply(const NumMod<F>& M, F x, F y) {
    typedef NumOps<F> O;
    if (V == MM_NUM_F16) return fn16<F, false>(M, x, y);
    if (V == MM_NUM_F16_UP) return fn16<F, true>(M, x, y);
    // F14 / F15: a = x y is exact (2m <= l)
    const F a = MUL ? ((V == MM_NUM_F14_UP || V == MM_NUM_F15_UP) ? O::mul_ru(x, y) : O::mul_rn(x, y)) : x;
    if (V == MM_NUM_F14) return fn14<F, false>(M, a);
    if (V == MM_NUM_F14_UP) return fn14<F, true>(M, a);
    if (V == MM_NUM_F15_UP) return fn15<F, true>(M, a);
    return fn15<F, false>(M, a);
}

constexpr int NUM_T = 256;
template <class F> struct Vec4;
template <> struct Vec4<float> { typedef float4 T; };
template <> struct Vec4<double> { typedef double2 T; };

// 16-byte vectors (4 floats / 2 doubles) per thread, grid-stride
template <class F, int V, bool MUL>
__global__ void __launch_bounds__(NUM_T) k_num(NumMod<F> M, const F* __restrict__ x, const F* __restrict__ y,
                                               F* __restrict__ z, long long nv) {
    typedef typename Vec4<F>::T VT;
    constexpr int L = sizeof(VT) / sizeof(F);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
        VT a = ((const VT*)x)[i], b = a;
        if (MUL) b = ((const VT*)y)[i];
        F* pa = (F*)&a;
        const F* pb = (const F*)&b;
#pragma unroll
        for (int j = 0; j < L; j++) pa[j] = num_apply<F, V, MUL>(M, pa[j], pb[j]);
        ((VT*)z)[i] = a;
    }
}
template <class F, int V, bool MUL>
__global__ void __launch_bounds__(NUM_T) k_num_tail(NumMod<F> M, const F* __restrict__ x, const F* __restrict__ y,
                                                    F* __restrict__ z, long long i0, long long n) {
    const long long i = i0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) z[i] = num_apply<F, V, MUL>(M, x[i], MUL ? y[i] : x[i]);
}
// MMNTT_DEBUG: count inputs outside the variant's domain (non-integral, < 0,
// >= p for residues, >= bound for reduce inputs)
template <class F>
__global__ void k_num_range(const F* __restrict__ x, long long n, F bound, unsigned* bad) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const F v = x[i];
        if (!(v >= F(0) && v < bound && NumOps<F>::flr(v) == v)) atomicAdd(bad, 1u);
    }
}

template <class F, int V, bool MUL>
static void launch_num(const NumMod<F>& M, const F* x, const F* y, F* z, size_t n, cudaStream_t st) {
    constexpr int L = 16 / sizeof(F);
    const bool vec = ((((uintptr_t)x | (uintptr_t)z | (MUL ? (uintptr_t)y : 0)) & 15) == 0);
    const long long nv = vec ? (long long)(n / L) : 0;
    if (nv > 0) {
        const long long blocks = (nv + NUM_T - 1) / NUM_T, cap = (long long)num_sms() * 16;
        k_num<F, V, MUL><<<(int)(blocks < cap ? blocks : cap), NUM_T, 0, st>>>(M, x, y, z, nv);
    }
    const long long i0 = nv * L, rest = (long long)n - i0;
    if (rest > 0) k_num_tail<F, V, MUL><<<(int)((rest + NUM_T - 1) / NUM_T), NUM_T, 0, st>>>(M, x, y, z, i0, (long long)n);
}

template <class F, bool MUL>
static mm_status dispatch_num(const NumMod<F>& M, int v, const F* x, const F* y, F* z, size_t n, cudaStream_t st) {
    switch (v) {
        case MM_NUM_F14: launch_num<F, MM_NUM_F14, MUL>(M, x, y, z, n, st); break;
        case MM_NUM_F14_UP: launch_num<F, MM_NUM_F14_UP, MUL>(M, x, y, z, n, st); break;
        case MM_NUM_F15_UP: launch_num<F, MM_NUM_F15_UP, MUL>(M, x, y, z, n, st); break;
        case MM_NUM_F15_NEAR: launch_num<F, MM_NUM_F15_NEAR, MUL>(M, x, y, z, n, st); break;
        case MM_NUM_F16: launch_num<F, MM_NUM_F16, MUL>(M, x, y, z, n, st); break;
        case MM_NUM_F16_UP: launch_num<F, MM_NUM_F16_UP, MUL>(M, x, y, z, n, st); break;
        default: return set_err(MM_E_ARG, "bad numeric variant %d", v);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

// largest m each variant admits for a trailing field of l bits
static int max_bits(int v, int l) {
    switch (v) {
        case MM_NUM_F14: case MM_NUM_F14_UP: return l / 2;            // Function 14: m <= l / 2
        case MM_NUM_F15_UP: case MM_NUM_F15_NEAR: return (l - 1) / 2;  // Function 15: m <= (l - 1) / 2
        case MM_NUM_F16: case MM_NUM_F16_UP: return l - 2;             // Function 16: m <= l - 2
    }
    return -1;
}

static const char* num_name(int v, bool mul) {
    static const char* names[2][6] = {
        {"reduce_num_f14", "reduce_num_f14_up", "reduce_num_f15_up", "reduce_num_f15_near", "reduce_num_f16", "reduce_num_f16_up"},
        {"mulmod_num_f14", "mulmod_num_f14_up", "mulmod_num_f15_up", "mulmod_num_f15_near", "mulmod_num_f16", "mulmod_num_f16_up"}};
    return (v >= 0 && v < 6) ? names[mul][v] : "num";
}

template <class F>
static mm_status range_check(const F* x, size_t n, F bound, cudaStream_t st) {
    unsigned* bad = nullptr;
    MM_CUDA_TRY(alloc_async((void**)&bad, sizeof(unsigned), st));
    MM_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned), st));
    {
        LaunchScope ls("debug_range_check", st);
        k_num_range<F><<<num_sms() * 4, 256, 0, st>>>(x, (long long)n, bound, bad);
    }
    unsigned h = 0;
    MM_CUDA_TRY(cudaMemcpyAsync(&h, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    MM_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFreeAsync(bad, st);
    if (h) return set_err(MM_E_RANGE, "%u inputs outside the variant's domain", h);
    return MM_OK;
}

static mm_status run_num(const mm_modnum* c, int v, const void* x, const void* y, void* z, size_t n, bool mul,
                         cudaStream_t st) {
    if (!c) return set_err(MM_E_ARG, "null context");
    const int l = c->fbits == 64 ? 52 : 23;
    const int mb = max_bits(v, l);
    if (mb < 0) return set_err(MM_E_ARG, "bad numeric variant %d", v);
    if (c->m > mb)
        return set_err(MM_E_PROFILE, "variant %d needs p < 2^%d for a %d-bit trailing field (p has %d bits)", v, mb, l,
                       c->m);
    if (v == MM_NUM_F15_NEAR && (!mul || !hprime(c->p)))
        return set_err(MM_E_INVALID_MODULUS, "Remark 12's round-to-nearest Function 15 needs p prime and a = x y");
    if (!mul && (v == MM_NUM_F16 || v == MM_NUM_F16_UP))
        return set_err(MM_E_ARG, "Function 16 takes two factors (mm_mulmod_num)");
    if (n == 0) return MM_OK;
    if (!x || !z || (mul && !y)) return set_err(MM_E_ARG, "null vector");
    if (debug_checks()) {
        // residues in [0, p); reduce inputs below alpha p (alpha = 2^(l/2), 2^((l-1)/2))
        double bound = (double)c->p;
        if (!mul) bound = ldexp((double)c->p, (v == MM_NUM_F14 || v == MM_NUM_F14_UP) ? l / 2 : (l - 1) / 2);
        mm_status s;
        if (c->fbits == 64) {
            if ((s = range_check<double>((const double*)x, n, bound, st)) != MM_OK) return s;
            if (mul && (s = range_check<double>((const double*)y, n, bound, st)) != MM_OK) return s;
        } else {
            if ((s = range_check<float>((const float*)x, n, (float)bound, st)) != MM_OK) return s;
            if (mul && (s = range_check<float>((const float*)y, n, (float)bound, st)) != MM_OK) return s;
        }
    }
    LaunchScope ls(num_name(v, mul), st);
    if (c->fbits == 64) {
        const NumMod<double> M{c->pd, c->u, c->ub};
        return mul ? dispatch_num<double, true>(M, v, (const double*)x, (const double*)y, (double*)z, n, st)
                   : dispatch_num<double, false>(M, v, (const double*)x, (const double*)x, (double*)z, n, st);
    }
    const NumMod<float> M{c->pf, c->uf, c->ubf};
    return mul ? dispatch_num<float, true>(M, v, (const float*)x, (const float*)y, (float*)z, n, st)
               : dispatch_num<float, false>(M, v, (const float*)x, (const float*)x, (float*)z, n, st);
}

}  // namespace mm

using namespace mm;

extern "C" mm_status mm_modnum_create(int fbits, uint64_t p, mm_modnum** ctx) {
    if (!ctx) return set_err(MM_E_ARG, "ctx is null");
    *ctx = nullptr;
    if (fbits != 32 && fbits != 64) return set_err(MM_E_ARG, "fbits must be 32 (float) or 64 (double)");
    if (p < 3 || !(p & 1)) return set_err(MM_E_INVALID_MODULUS, "p=%llu must be an odd integer >= 3", (unsigned long long)p);
    int m = 0;
    while (m < 64 && (p >> m)) m++;
    const int l = fbits == 64 ? 52 : 23;
    if (m > l - 2)
        return set_err(MM_E_PROFILE, "p=%llu has %d bits; numeric products need m <= l - 2 = %d (Function 16)",
                       (unsigned long long)p, m, l - 2);
    mm_modnum* c = new (std::nothrow) mm_modnum;
    if (!c) return set_err(MM_E_ARG, "out of host memory");
    c->fbits = fbits;
    c->p = p;
    c->m = m;
    // u = 1/p to nearest (host default rounding); u-bar = the least F value >= 1/p
    // (P:583): the sign of fma(u, p, -1) is exact, so u < 1/p iff it is negative
    c->pd = (double)p;
    c->u = 1.0 / c->pd;
    c->ub = fma(c->u, c->pd, -1.0) < 0.0 ? nextafter(c->u, INFINITY) : c->u;
    c->pf = (float)p;
    c->uf = 1.0f / c->pf;
    c->ubf = fmaf(c->uf, c->pf, -1.0f) < 0.0f ? nextafterf(c->uf, INFINITY) : c->uf;
    *ctx = c;
    return MM_OK;
}
extern "C" void mm_modnum_destroy(mm_modnum* ctx) { delete ctx; }
extern "C" mm_status mm_modnum_info(const mm_modnum* c, double out[6]) {
    if (!c || !out) return set_err(MM_E_ARG, "null argument");
    out[0] = (double)c->p;
    out[1] = c->fbits == 64 ? c->u : (double)c->uf;
    out[2] = c->fbits == 64 ? c->ub : (double)c->ubf;
    out[3] = c->fbits == 64 ? 52 : 23;
    out[4] = c->m;
    out[5] = c->fbits;
    return MM_OK;
}
extern "C" mm_status mm_mulmod_num(const mm_modnum* c, mm_num_variant v, const void* x, const void* y, void* z, size_t n,
                                   void* stream) {
    return run_num(c, (int)v, x, y, z, n, true, (cudaStream_t)stream);
}
extern "C" mm_status mm_reduce_num(const mm_modnum* c, mm_num_variant v, const void* a, void* z, size_t n, void* stream) {
    return run_num(c, (int)v, a, nullptr, z, n, false, (cudaStream_t)stream);
}
