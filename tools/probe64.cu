// probe64.cu -- standalone measurement tool (not part of the library): per
// SASS-class issue rates on sm_100a and register-resident Goldilocks
// butterfly variants, each variant first checked against u128 % on device.
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/probe64 tools/probe64.cu
//   tools/bin/probe64            (prints one JSON object)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define EPS 0xFFFFFFFFull
static constexpr uint64_t P = 0xFFFFFFFF00000001ull;
typedef unsigned __int128 u128;

// ---------------------------------------------------------------- class probes
template <int KIND>
__global__ void __launch_bounds__(256) k_class(uint32_t seed, int iters, uint32_t* sink) {
    uint32_t x[8];
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; i++) { x[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u; d[i] = x[i] * 1e-9; }
    const uint32_t k = seed | 1u, c = seed ^ 0x5bd1e995u;
    const double dk = 0.999999, dc = 1e-9;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 8; r++) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if (KIND == 0) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(k), "r"(c));
                if (KIND == 1) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
                if (KIND == 2) asm volatile("{.reg .u32 h; add.cc.u32 %0, %0, %1; addc.u32 h, %0, %2; xor.b32 %0, %0, h;}" : "+r"(x[i]) : "r"(k), "r"(c));
                if (KIND == 3) asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(x[i]) : "r"(k));
                if (KIND == 4) asm volatile("{.reg .pred q; setp.lt.u32 q, %0, %1; selp.b32 %0, %0, %2, q;}" : "+r"(x[i]) : "r"(k), "r"(c));
                if (KIND == 5) asm volatile("{.reg .u64 w; mul.wide.u32 w, %0, %1; cvt.u32.u64 %0, w;}" : "+r"(x[i]) : "r"(k));
                if (KIND == 6) {
                    asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(k), "r"(c));
                    asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
                }
                if (KIND == 7) {
                    asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(k), "r"(c));
                    asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(dk), "d"(dc));
                }
                if (KIND == 8) {
                    asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
                    asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(dk), "d"(dc));
                }
                if (KIND == 9) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(k), "r"(c));
                if (KIND == 10) {   // 2 ALU : 1 FMA
                    asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(k), "r"(c));
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(k), "r"(c));
                    asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
                }
                if (KIND == 11) asm volatile("madc.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(k), "r"(c));
            }
        }
    }
    uint32_t acc = 0;
    double dacc = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) { acc ^= x[i]; dacc += d[i]; }
    if (acc == 0x12345678u || dacc == 1234.5) sink[0] = acc;
}
// instructions per inner op (for the rate)
static const double class_ops[] = {1, 1, 3, 1, 2, 1, 2, 2, 2, 1, 3, 1};
static const char* class_name[] = {"IADD3", "IMAD", "IADD3+IADD3.X+LOP3", "SHF", "ISETP+SEL", "IMAD.WIDE",
                                   "IADD3|IMAD", "IADD3|DFMA", "IMAD|DFMA", "LOP3", "IADD3|LOP3|IMAD", "IMAD.X"};

// ---------------------------------------------------------------- arithmetic variants
struct GL0 {  // current library form (arith.cuh FpG), values in [0, 2^64)
    __device__ __forceinline__ static uint64_t add(uint64_t a, uint64_t b) {
        uint32_t s0, s1;
        asm("{\n\t.reg .u32 c, m;\n\t"
            "add.cc.u32 %0, %2, %4;\n\taddc.cc.u32 %1, %3, %5;\n\taddc.u32 c, 0, 0;\n\tsub.u32 m, 0, c;\n\t"
            "add.cc.u32 %0, %0, m;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.u32 c, 0, 0;\n\tsub.u32 m, 0, c;\n\t"
            "add.cc.u32 %0, %0, m;\n\taddc.u32 %1, %1, 0;\n\t}"
            : "=&r"(s0), "=&r"(s1)
            : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
        return ((uint64_t)s1 << 32) | s0;
    }
    __device__ __forceinline__ static uint64_t sub(uint64_t a, uint64_t b) {
        uint32_t d0, d1;
        asm("{\n\t.reg .u32 m;\n\t"
            "sub.cc.u32 %0, %2, %4;\n\tsubc.cc.u32 %1, %3, %5;\n\tsubc.u32 m, 0, 0;\n\t"
            "sub.cc.u32 %0, %0, m;\n\tsubc.cc.u32 %1, %1, 0;\n\tsubc.u32 m, 0, 0;\n\t"
            "sub.cc.u32 %0, %0, m;\n\tsubc.u32 %1, %1, 0;\n\t}"
            : "=&r"(d0), "=&r"(d1)
            : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
        return ((uint64_t)d1 << 32) | d0;
    }
    __device__ __forceinline__ static void mul128(uint64_t a, uint64_t b, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                                  uint32_t& r3) {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
        const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        asm("mul.lo.u32 %0, %4, %6;\n\tmul.hi.u32 %1, %4, %6;\n\t"
            "mad.lo.cc.u32 %1, %4, %7, %1;\n\tmadc.hi.u32 %2, %4, %7, 0;\n\t"
            "mad.lo.cc.u32 %1, %5, %6, %1;\n\tmadc.hi.cc.u32 %2, %5, %6, %2;\n\tmadc.hi.u32 %3, %5, %7, 0;\n\t"
            "mad.lo.cc.u32 %2, %5, %7, %2;\n\taddc.u32 %3, %3, 0;"
            : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
            : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
    }
    __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) {
        uint32_t r0, r1, r2, r3;
        mul128(a, b, r0, r1, r2, r3);
        uint32_t u0, u1, net;
        asm("{\n\t.reg .u32 t0, t1, bw;\n\t"
            "sub.cc.u32 t0, %3, %6;\n\tsubc.cc.u32 t1, %4, 0;\n\tsubc.u32 bw, 0, 0;\n\t"
            "sub.cc.u32 t0, t0, bw;\n\tsubc.u32 t1, t1, 0;\n\t"
            "sub.cc.u32 %0, t0, %5;\n\tsubc.cc.u32 %1, t1, 0;\n\tsubc.u32 %2, 0, 0;\n\t"
            "add.cc.u32 %1, %1, %5;\n\taddc.u32 %2, %2, 0;\n\t}"
            : "=&r"(u0), "=&r"(u1), "=&r"(net)
            : "r"(r0), "r"(r1), "r"(r2), "r"(r3));
        uint64_t r = ((uint64_t)u1 << 32) | u0;
        return r + (uint64_t)(0u - net);
    }
};

// Canonical form: every value in [0, p).  add: s = x + y, t = s - p (= s + EPS
// mod 2^64); take t when s wrapped or t wrapped.  sub: d = x - y, + p on borrow.
struct GLC {
    __device__ __forceinline__ static uint64_t add(uint64_t x, uint64_t y) {
        uint64_t s = x + y;
        uint64_t t = s + EPS;
        return ((s < x) | (t < s)) ? t : s;
    }
    __device__ __forceinline__ static uint64_t sub(uint64_t x, uint64_t y) {
        uint64_t d = x - y;
        return (x < y) ? d - EPS : d;
    }
    __device__ __forceinline__ static uint64_t canon(uint64_t r) {
        uint64_t t = r + EPS;
        return (t < r) ? t : r;
    }
    __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) { return canon(GL0::mul(a, b)); }
};

// Canonical add/sub written with carry flags (PTX) instead of compares.
struct GLF {
    __device__ __forceinline__ static uint64_t add(uint64_t x, uint64_t y) {
        uint32_t s0, s1;
        asm("{\n\t.reg .u32 c, t0, t1;\n\t.reg .pred q;\n\t"
            "add.cc.u32 %0, %2, %4;\n\taddc.cc.u32 %1, %3, %5;\n\taddc.u32 c, 0, 0;\n\t"
            "add.cc.u32 t0, %0, 0xFFFFFFFF;\n\taddc.cc.u32 t1, %1, 0;\n\taddc.u32 c, c, 0;\n\t"
            "setp.ne.u32 q, c, 0;\n\t"
            "selp.b32 %0, t0, %0, q;\n\tselp.b32 %1, t1, %1, q;\n\t}"
            : "=&r"(s0), "=&r"(s1)
            : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
        return ((uint64_t)s1 << 32) | s0;
    }
    __device__ __forceinline__ static uint64_t sub(uint64_t x, uint64_t y) {
        uint32_t d0, d1;
        asm("{\n\t.reg .u32 m;\n\t"
            "sub.cc.u32 %0, %2, %4;\n\tsubc.cc.u32 %1, %3, %5;\n\tsubc.u32 m, 0, 0;\n\t"   // m = -borrow
            "sub.cc.u32 %0, %0, m;\n\tsubc.u32 %1, %1, 0;\n\t}"                           // d - EPS*borrow
            : "=&r"(d0), "=&r"(d1)
            : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
        return ((uint64_t)d1 << 32) | d0;
    }
    __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) { return GLC::canon(GL0::mul(a, b)); }
};

// x * 2^K mod p for canonical x, 0 <= K < 96, canonical output.  The 128-bit
// shifted value r = (r3 r2 r1 r0) is reduced with 2^64 = EPS, 2^96 = -1.
template <int K>
__device__ __forceinline__ uint64_t shl_mod(uint64_t x) {
    if constexpr (K == 0) return x;
    else if constexpr (K < 64) {
        // lo = x << K, hi = x >> (64 - K) < 2^K; value = lo + hi 2^64 = lo + hi EPS
        const uint64_t lo = x << K, hi = x >> (64 - K);
        if constexpr (K <= 32) {
            // hi < 2^32: hi EPS = (hi << 32) - hi < 2^64
            const uint64_t v = (hi << 32) - hi;
            uint64_t s = lo + v;
            uint64_t t = s + EPS;
            return ((s < lo) | (t < s)) ? t : s;
        } else {
            // hi = h1 2^32 + h0 (h1 < 2^(K-32)): hi 2^64 = h0 EPS + h1 2^96 = h0 EPS - h1
            const uint64_t h0 = (uint32_t)hi, h1 = hi >> 32;
            const uint64_t v = (h0 << 32) - h0;
            uint64_t s = lo + v;
            uint64_t t = s + EPS;
            s = ((s < lo) | (t < s)) ? t : s;   // canonical lo + h0 EPS
            uint64_t d = s - h1;
            return (s < h1) ? d - EPS : d;
        }
    } else {
        // x 2^K = (x 2^(K-64)) 2^64; y = x << (K-64) as (hi, lo): lo EPS + hi 2^128,
        // 2^128 = 2^32 2^96 = -2^32: value = lo EPS - hi 2^32 with hi < 2^(K-64)
        constexpr int J = K - 64;
        uint64_t lo = x << J, hi = 0;
        if constexpr (J > 0) hi = x >> (64 - J);
        lo = GLC::canon(lo);   // lo may be >= p
        // lo EPS = lo 2^32 - lo: reduce lo 2^32 via (l1 2^64 + l0 2^32) = l1 EPS + l0 2^32
        const uint64_t l0 = (uint32_t)lo, l1 = lo >> 32;
        // value = l0 2^32 + l1 (2^32 - 1) - lo - hi 2^32 = (l0 + l1 - hi) 2^32 - l1 - lo
        // compute A = (l0 + l1) 2^32 - l1 (fits: < 2^65) canonically, then subtract lo and hi 2^32
        uint64_t a = (l0 << 32) + ((l1 << 32) - l1);
        uint64_t aw = a + EPS;
        a = ((a < (l0 << 32)) | (aw < a)) ? aw : a;
        uint64_t d = a - lo;
        a = (a < lo) ? d - EPS : d;
        const uint64_t h = hi << 32;   // hi < 2^32 so h < 2^64, h < p
        d = a - h;
        return (a < h) ? d - EPS : d;
    }
}

// x * w^e with w = 2^39 (the 64th root 7^((p-1)/64)): shift 39e mod 192, and
// 2^96 = -1 turns shifts >= 96 into a negated shift.
template <int E> struct Rot {
    static constexpr int S = (39 * E) % 192;
    static constexpr bool NEG = S >= 96;
    static constexpr int K = NEG ? S - 96 : S;
};

// Goldilocks, lazy [0,2^64), pipe-balanced formulations.
struct GL2 {
    __device__ __forceinline__ static uint64_t pk(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }
    // add: 64-bit add (ALU), carry folds as c*EPS via mad (FMA pipe)
    __device__ __forceinline__ static uint64_t add(uint64_t a, uint64_t b) {
        uint32_t s0, s1;
        asm("{\n\t.reg .u32 c;\n\t"
            "add.cc.u32 %0, %2, %4;\n\taddc.cc.u32 %1, %3, %5;\n\taddc.u32 c, 0, 0;\n\t"
            "mad.lo.cc.u32 %0, c, 0xFFFFFFFF, %0;\n\tmadc.hi.cc.u32 %1, c, 0xFFFFFFFF, %1;\n\taddc.u32 c, 0, 0;\n\t"
            "mad.lo.cc.u32 %0, c, 0xFFFFFFFF, %0;\n\tmadc.hi.u32 %1, c, 0xFFFFFFFF, %1;\n\t}"
            : "=&r"(s0), "=&r"(s1)
            : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
        return pk(s0, s1);
    }
    // sub: d = a - b; on borrow add p (= 2^32 EPS + 1 -> words (1, EPS)) by mad
    __device__ __forceinline__ static uint64_t sub(uint64_t a, uint64_t b) {
        uint32_t d0, d1;
        asm("{\n\t.reg .u32 m, c;\n\t"
            "sub.cc.u32 %0, %2, %4;\n\tsubc.cc.u32 %1, %3, %5;\n\tsubc.u32 m, 0, 0;\n\t"   // m = -borrow
            "sub.cc.u32 %0, %0, m;\n\tsubc.cc.u32 %1, %1, 0;\n\tsubc.u32 m, 0, 0;\n\t"
            "sub.cc.u32 %0, %0, m;\n\tsubc.u32 %1, %1, 0;\n\t}"
            : "=&r"(d0), "=&r"(d1)
            : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
        return pk(d0, d1);
    }
    // reduce r = (r3 r2 r1 r0) = (r1:r0) + r2 EPS - r3
    __device__ __forceinline__ static uint64_t red(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
        uint32_t u0, u1;
        asm("{\n\t.reg .u32 c, m;\n\t"
            "mad.lo.cc.u32 %0, %4, 0xFFFFFFFF, %2;\n\tmadc.hi.cc.u32 %1, %4, 0xFFFFFFFF, %3;\n\taddc.u32 c, 0, 0;\n\t"
            "mad.lo.cc.u32 %0, c, 0xFFFFFFFF, %0;\n\tmadc.hi.u32 %1, c, 0xFFFFFFFF, %1;\n\t"   // no overflow
            "sub.cc.u32 %0, %0, %5;\n\tsubc.cc.u32 %1, %1, 0;\n\tsubc.u32 m, 0, 0;\n\t"
            "sub.cc.u32 %0, %0, m;\n\tsubc.u32 %1, %1, 0;\n\t}"        // borrow: - EPS (no second borrow)
            : "=&r"(u0), "=&r"(u1)
            : "r"(r0), "r"(r1), "r"(r2), "r"(r3));
        return pk(u0, u1);
    }
    __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
        const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        uint32_t r0, r1, r2, r3;
        asm("mul.lo.u32 %0, %4, %6;\n\tmul.hi.u32 %1, %4, %6;\n\t"
            "mad.lo.cc.u32 %1, %4, %7, %1;\n\tmadc.hi.u32 %2, %4, %7, 0;\n\t"
            "mad.lo.cc.u32 %1, %5, %6, %1;\n\tmadc.hi.cc.u32 %2, %5, %6, %2;\n\tmadc.hi.u32 %3, %5, %7, 0;\n\t"
            "mad.lo.cc.u32 %2, %5, %7, %2;\n\taddc.u32 %3, %3, 0;"
            : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
            : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
        return red(r0, r1, r2, r3);
    }
    // x * 2^K, 0 < K < 32: (r2 r1 r0) = x 2^K by two wide mads, then (r1:r0) + r2 EPS
    template <int K> __device__ __forceinline__ static uint64_t shl(uint64_t x) {
        if constexpr (K == 0) return x;
        else {
        const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
        uint32_t r0, r1, r2, u0, u1;
        constexpr uint32_t M = 1u << (K & 31);
        if constexpr (K < 32) {
            asm("mul.lo.u32 %0, %3, %5;\n\tmul.hi.u32 %1, %3, %5;\n\t"
                "mad.lo.cc.u32 %1, %4, %5, %1;\n\tmadc.hi.u32 %2, %4, %5, 0;"
                : "=r"(r0), "=r"(r1), "=r"(r2) : "r"(x0), "r"(x1), "n"(M));
            asm("{\n\t.reg .u32 c;\n\t"
                "mad.lo.cc.u32 %0, %4, 0xFFFFFFFF, %2;\n\tmadc.hi.cc.u32 %1, %4, 0xFFFFFFFF, %3;\n\taddc.u32 c, 0, 0;\n\t"
                "mad.lo.cc.u32 %0, c, 0xFFFFFFFF, %0;\n\tmadc.hi.u32 %1, c, 0xFFFFFFFF, %1;\n\t}"
                : "=&r"(u0), "=&r"(u1) : "r"(r0), "r"(r1), "r"(r2));
            return pk(u0, u1);
        } else if constexpr (K == 32) {
            // (x0 : 0) + x1 EPS
            asm("{\n\t.reg .u32 c;\n\t"
                "mad.lo.cc.u32 %0, %3, 0xFFFFFFFF, 0;\n\tmadc.hi.cc.u32 %1, %3, 0xFFFFFFFF, %2;\n\taddc.u32 c, 0, 0;\n\t"
                "mad.lo.cc.u32 %0, c, 0xFFFFFFFF, %0;\n\tmadc.hi.u32 %1, c, 0xFFFFFFFF, %1;\n\t}"
                : "=&r"(u0), "=&r"(u1) : "r"(x0), "r"(x1));
            return pk(u0, u1);
        } else if constexpr (K < 64) {
            return shl<32>(shl<K - 32>(x));
        } else if constexpr (K < 96) {
            // x 2^K = (x 2^(K-64)) EPS = y 2^32 - y
            uint64_t y = shl<K - 64>(x);
            return sub(shl<32>(y), y);
        }
        }
    }
};

struct GLM1 { // GL0 add/sub + GL2 mul
    __device__ __forceinline__ static uint64_t add(uint64_t a, uint64_t b) { return GL0::add(a, b); }
    __device__ __forceinline__ static uint64_t sub(uint64_t a, uint64_t b) { return GL0::sub(a, b); }
    __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) { return GL2::mul(a, b); }
};
struct GLM2 { // GL2 add + GL0 sub/mul
    __device__ __forceinline__ static uint64_t add(uint64_t a, uint64_t b) { return GL2::add(a, b); }
    __device__ __forceinline__ static uint64_t sub(uint64_t a, uint64_t b) { return GL0::sub(a, b); }
    __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) { return GL0::mul(a, b); }
};
// ---------------------------------------------------------------- correctness
__device__ uint64_t ref_mul(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) % P); }
__device__ uint64_t ref_pow2(int k) {
    uint64_t r = 1, b = 2;
    while (k) { if (k & 1) r = ref_mul(r, b); b = ref_mul(b, b); k >>= 1; }
    return r;
}
__device__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ uint64_t sample(uint64_t i, bool canon) {
    uint64_t w = mix64(i * 0x9E3779B97F4A7C15ull + 12345);
    const uint64_t edge[8] = {0, 1, P - 1, P - 2, EPS, EPS + 1, 1ull << 63, P >> 1};
    if ((i & 15) < 8) w = edge[i & 7];
    if (!canon) { if ((i & 31) == 17) w = P + (w % EPS); }   // non-canonical [p, 2^64)
    if (canon && w >= P) w -= P;
    return w;
}
template <int K> __device__ void chk_shl(uint64_t x, unsigned* bad) {
    uint64_t r = shl_mod<K>(x), e = ref_mul(x, ref_pow2(K));
    if (r != e) atomicAdd(bad + 3, 1u);
}
template <int... Ks> struct ShlList { __device__ static void run(uint64_t x, unsigned* bad) { (chk_shl<Ks>(x, bad), ...); } };

__global__ void k_check(unsigned* bad, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        // GL0 on non-canonical inputs
        uint64_t x = sample(2 * i, false), y = sample(2 * i + 1, false);
        uint64_t xr = x % P, yr = y % P;
        if (GL0::add(x, y) % P != (xr + (u128)yr) % P) atomicAdd(bad + 0, 1u);
        if (GL0::sub(x, y) % P != (xr + (u128)P - yr) % P) atomicAdd(bad + 0, 1u);
        if (GL0::mul(x, y) % P != ref_mul(xr, yr)) atomicAdd(bad + 0, 1u);
        // canonical variants
        x = xr; y = yr;
        uint64_t ea = (uint64_t)((x + (u128)y) % P), es = (uint64_t)((x + (u128)P - y) % P), em = ref_mul(x, y);
        if (GLC::add(x, y) != ea || GLC::sub(x, y) != es || GLC::mul(x, y) != em) atomicAdd(bad + 1, 1u);
        if (GL2::add(x, y) % P != ea || GL2::sub(x, y) % P != es || GL2::mul(x, y) % P != em) atomicAdd(bad + 4, 1u);
        {
            uint64_t xn = sample(2 * i, false), yn = sample(2 * i + 1, false);
            if (GL2::add(xn, yn) % P != ea || GL2::sub(xn, yn) % P != es || GL2::mul(xn, yn) % P != em) atomicAdd(bad + 4, 1u);
        }
        if (GLF::add(x, y) != ea || GLF::sub(x, y) != es || GLF::mul(x, y) != em) atomicAdd(bad + 2, 1u);
        ShlList<0, 3, 6, 9, 12, 15, 18, 21, 24, 27, 30, 31, 32, 33, 36, 39, 42, 45, 48, 51, 54, 57, 60, 63, 64, 66,
                69, 72, 75, 78, 81, 84, 87, 90, 93, 95>::run(x, bad);
    }
}

// ---------------------------------------------------------------- butterfly probes
// radix-64 register block per thread?  Too many registers; use radix 8 with
// the twiddles of a length-64 DIF's last three levels (powers of w64).
template <class A>
__device__ __forceinline__ void dif_gen(uint64_t& x, uint64_t& y, uint64_t w) {
    uint64_t s = A::add(x, y), d = A::sub(x, y);
    x = s;
    y = A::mul(d, w);
}
template <class A, int E>
__device__ __forceinline__ void dif_rot(uint64_t& x, uint64_t& y) {
    typedef Rot<E> R;
    uint64_t s = A::add(x, y);
    uint64_t d = R::NEG ? A::sub(y, x) : A::sub(x, y);
    x = s;
    y = shl_mod<R::K>(d);
}

// VAR 0: GL0, general twiddles; 1: GLC general; 2: GLF general;
// VAR 3: GLF + shift twiddles of a 64-point DIF (levels spans 4,2,1 with e = 8*i etc.)
// VAR 4: GLF, shift twiddles for span-32..8 levels (generic 64th-root exponents)
template <int VAR>
__global__ void __launch_bounds__(256) k_bfly(int iters, uint64_t* sink) {
    uint64_t v[8];
#pragma unroll
    for (int t = 0; t < 8; t++) v[t] = ((uint64_t)(threadIdx.x * 2654435761u + t) * 0x9E3779B97F4A7C15ull) % P;
    uint64_t w[4];
#pragma unroll
    for (int t = 0; t < 4; t++) w[t] = (0x123456789ull * (t + 3 + blockIdx.x)) % P;
    for (int it = 0; it < iters; it++) {
        if (VAR <= 2 || VAR >= 5) {
#pragma unroll
            for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    if (t & h) continue;
                    if (VAR == 0) dif_gen<GL0>(v[t], v[t + h], w[t & 3]);
                    if (VAR == 1) dif_gen<GLC>(v[t], v[t + h], w[t & 3]);
                    if (VAR == 2) dif_gen<GLF>(v[t], v[t + h], w[t & 3]);
                    if (VAR == 5) dif_gen<GL2>(v[t], v[t + h], w[t & 3]);
                    if (VAR == 6) dif_gen<GLM1>(v[t], v[t + h], w[t & 3]);
                    if (VAR == 7) dif_gen<GLM2>(v[t], v[t + h], w[t & 3]);
                }
        } else if (VAR == 3) {
            // an 8-point DIF with root w64^8 = 2^(39*8): twiddles w8^i, i = 0..3 then w4, then 1
            dif_rot<GLF, 0>(v[0], v[4]); dif_rot<GLF, 8>(v[1], v[5]); dif_rot<GLF, 16>(v[2], v[6]); dif_rot<GLF, 24>(v[3], v[7]);
            dif_rot<GLF, 0>(v[0], v[2]); dif_rot<GLF, 16>(v[1], v[3]); dif_rot<GLF, 0>(v[4], v[6]); dif_rot<GLF, 16>(v[5], v[7]);
            dif_rot<GLF, 0>(v[0], v[1]); dif_rot<GLF, 0>(v[2], v[3]); dif_rot<GLF, 0>(v[4], v[5]); dif_rot<GLF, 0>(v[6], v[7]);
        } else {
            // non-trivial 64th-root shifts everywhere (worst case mix)
            dif_rot<GLF, 1>(v[0], v[4]); dif_rot<GLF, 3>(v[1], v[5]); dif_rot<GLF, 5>(v[2], v[6]); dif_rot<GLF, 7>(v[3], v[7]);
            dif_rot<GLF, 2>(v[0], v[2]); dif_rot<GLF, 6>(v[1], v[3]); dif_rot<GLF, 10>(v[4], v[6]); dif_rot<GLF, 14>(v[5], v[7]);
            dif_rot<GLF, 4>(v[0], v[1]); dif_rot<GLF, 12>(v[2], v[3]); dif_rot<GLF, 20>(v[4], v[5]); dif_rot<GLF, 28>(v[6], v[7]);
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int t = 0; t < 8; t++) acc ^= v[t];
    if (acc == 0x12345678ull) sink[0] = acc;
}

template <class K>
static float time_kernel(K launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    return t;
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz
    const double ghz = clk * 1e-6;
    uint32_t* sink;
    cudaMalloc(&sink, 64);
    unsigned* bad;
    cudaMalloc(&bad, 16 * sizeof(unsigned));
    cudaMemset(bad, 0, 16 * sizeof(unsigned));
    k_check<<<sms * 4, 256>>>(bad, 1ll << 22);
    unsigned hb[16];
    cudaMemcpy(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
    printf("{\"sms\": %d, \"clock_ghz\": %.3f,\n \"check_bad\": {\"GL0\": %u, \"GLC\": %u, \"GLF\": %u, \"shl\": %u, \"GL2\": %u},\n", sms,
           ghz, hb[0], hb[1], hb[2], hb[3], hb[4]);
    const int blocks = sms * 8, threads = 256, iters = 2000;
    printf(" \"class_warp_inst_per_clk_per_SM\": {");
#define CLS(K)                                                                                                  \
    {                                                                                                           \
        float ms = time_kernel([&] { k_class<K><<<blocks, threads>>>(12345u, iters, sink); });                  \
        double ops = (double)blocks * (threads / 32) * iters * 64.0 * class_ops[K];                             \
        printf("%s\"%s\": %.3f", K ? ", " : "", class_name[K], ops / (ms * 1e-3 * sms * ghz * 1e9));             \
    }
    CLS(0) CLS(1) CLS(2) CLS(3) CLS(4) CLS(5) CLS(6) CLS(7) CLS(8) CLS(9) CLS(10) CLS(11)
    printf("},\n \"bfly64_G_per_s\": {");
    const char* bn[] = {"GL0_general", "GLC_general", "GLF_general", "GLF_shift_dft8", "GLF_shift_worst", "GL2_general", "GL0addsub_GL2mul", "GL2add_GL0submul"};
#define BF(V)                                                                                                   \
    {                                                                                                           \
        float ms = time_kernel([&] { k_bfly<V><<<blocks, threads>>>(iters / 4, (uint64_t*)sink); });          \
        double bf = (double)blocks * threads * (iters / 4) * 12.0;                                              \
        printf("%s\"%s\": %.1f", V ? ", " : "", bn[V], bf / (ms * 1e-3) * 1e-9);                               \
    }
    BF(0) BF(1) BF(2) BF(3) BF(4) BF(5) BF(6) BF(7)
    printf("}}\n");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
