// arith.cuh -- device modular arithmetic for sm_100a (B200).
//
// 32-bit moduli (U = uint32_t, L = uint64_t in the paper's notation):
//   * modadd / modsub, full range m = n (Function 4) and
//     m <= n-1 (Function 2; P:140 for subtraction);
//   * Barrett's reduction (Function 6) with the Table-3 profile
//      chosen per modulus;
//   * fixed-multiplicand ("Shoup") product (Function 8) with the
//     companion psi = floor(2^32 y / p);
//   * Montgomery's reduction (Function 13) with R = 2^32
//     (m = n = 32 so the mask of line 1 vanishes), in the subtractive
//     form: m = lo * p^-1 mod 2^32, r = hi - umulhi(m, p) (+p if negative).
//     Output x y 2^-32 mod p, canonical -- identical to Function 13.
// 64-bit modulus p = 2^64 - 2^32 + 1 ("Goldilocks", BASELINE C4/C5): products
//   built from 32-bit partial products (IMAD.WIDE.U32) and reduced with
//   2^64 = 2^32 - 1, 2^96 = -1 (mod p).
//
// The lazy-reduction butterflies (Harvey) keep values in [0, 2p) / [0, 4p);
// valid because every NTT prime used with them has p < 2^30 (4p < 2^32).
#pragma once
#include <stdint.h>

namespace mm {

// ----------------------------------------------------------------- 32 bit
__device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

// Function 4, m = n: a = p - y; x >= a ? x - a : x - a + p.
__device__ __forceinline__ uint32_t add_full(uint32_t x, uint32_t y, uint32_t p) {
    uint32_t a = p - y;
    uint32_t d = x - a;
    return x >= a ? d : d + p;
}
// subtraction "in a similar manner": x - y, + p on borrow.
__device__ __forceinline__ uint32_t sub_full(uint32_t x, uint32_t y, uint32_t p) {
    uint32_t d = x - y;
    return x >= y ? d : d + p;
}
// Function 2, m <= n-1: min(a, a - p).
__device__ __forceinline__ uint32_t add_half(uint32_t x, uint32_t y, uint32_t p) {
    uint32_t a = x + y;
    return umin32(a, a - p);
}
__device__ __forceinline__ uint32_t sub_half(uint32_t x, uint32_t y, uint32_t p) {
    uint32_t a = x - y;
    return umin32(a, a + p);
}

// Function 8, d kept in L = 64 bits because for m = n it can
// reach 33 bits.  z = x y mod p, canonical.
__device__ __forceinline__ uint32_t mul_shoup_full(uint32_t x, uint32_t y, uint32_t psi, uint32_t p) {
    uint32_t c = __umulhi(x, psi);                              // 1. (x * psi) >> n
    uint64_t d = (uint64_t)x * y - (uint64_t)c * p;             // 2. d = x y - c p  (in L)
    return (uint32_t)(d >= p ? d - p : d);                      // 3. one correction
}
// Function 8 with the m <= n-1 simplification: d in U; result in
// [0, 2p) before the correction, so the lazy form simply skips line 3.
__device__ __forceinline__ uint32_t mul_shoup_lazy(uint32_t x, uint32_t y, uint32_t psi, uint32_t p) {
    uint32_t c = __umulhi(x, psi);
    return x * y - c * p;
}

// Montgomery REDC of a 64-bit product t = hi:lo < 2^32 p, subtractive form.
// pinv = p^-1 mod 2^32.  Returns t 2^-32 mod p in [0, p).
__device__ __forceinline__ uint32_t redc32(uint32_t lo, uint32_t hi, uint32_t p, uint32_t pinv) {
    uint32_t m = lo * pinv;
    uint32_t mp_hi = __umulhi(m, p);
    uint32_t r = hi - mp_hi;
    return hi >= mp_hi ? r : r + p;
}
__device__ __forceinline__ uint32_t mul_mont(uint32_t x, uint32_t y, uint32_t p, uint32_t pinv) {
    return redc32(x * y, __umulhi(x, y), p, pinv);
}

// Barrett (Function 6) for a = x y < 2^64 with Table 3's profile:
// b = a >> s; c = (b q) >> t; d = a - c p; at most h corrections.
// For C2's p = 3221225473 (m = n = 32): FULL profile s = 31, t = 32, h = 3.
struct Barrett32 {
    uint32_t p, q;
    int s, t, h;
};
__device__ __forceinline__ uint32_t mul_barrett(uint32_t x, uint32_t y, const Barrett32& B) {
    uint64_t a = (uint64_t)x * y;
    uint64_t b = a >> B.s;                                       // < 2^33 for FULL
    // c = (b q) >> t, b q < 2^65: split b = bh 2^32 + bl.
    uint32_t bl = (uint32_t)b, bh = (uint32_t)(b >> 32);
    uint64_t lo = (uint64_t)bl * B.q;
    uint64_t hi = (uint64_t)bh * B.q + (lo >> 32);               // (b q) >> 32
    uint64_t c = hi >> (B.t - 32);                               // t >= 32 here
    uint64_t d = a - c * B.p;
    // Proposition 1: at most h subtractions; predicated, branch-free.
    d = d >= B.p ? d - B.p : d;
    d = d >= B.p ? d - B.p : d;
    d = d >= B.p ? d - B.p : d;
    return (uint32_t)d;
}

// Function 6 with Table 3's FULL profile folded in (m = n = 32: s = 31,
// t = 32, h = 3): b = a >> 31 has 33 bits (bl, bh), c = (b q) >> 32 =
// hi(bl q) + bh q exactly, d = a - c p < 4p (Proposition 1, h = 3), and the
// h corrections become two conditional subtractions (2p, then p).
__device__ __forceinline__ uint32_t mul_barrett_full(uint32_t x, uint32_t y, uint32_t p, uint32_t q) {
    const uint64_t a = (uint64_t)x * y;
    const uint32_t bl = (uint32_t)(a >> 31), bh = (uint32_t)(a >> 63);
    const uint64_t c = (uint64_t)__umulhi(bl, q) + (bh ? (uint64_t)q : 0ull);
    uint64_t d = a - c * p;
    const uint64_t p2 = 2ull * p;
    d = d >= p2 ? d - p2 : d;
    d = d >= p ? d - p : d;
    return (uint32_t)d;
}

// Field used by the 32-bit NTT kernels (p < 2^30; lazy Harvey butterflies).
struct Fp32 {
    typedef uint32_t T;
    typedef uint2 W;         // twiddle (w, floor(w 2^32 / p))
    uint32_t p, p2, pinv;    // pinv = p^-1 mod 2^32 (Montgomery, pointwise)
    uint32_t pr = 0;         // floor(2^32 / p): raw 32-bit words reduced on load (reduce_raw)
    // x w mod p in [0, 2p) for any x < 2^32 (Function 8, lazy).
    __device__ __forceinline__ uint32_t mulw(uint32_t x, W w) const {
        uint32_t c = __umulhi(x, w.y);
        return x * w.x - c * p;
    }
    // Gentleman-Sande (DIF) butterfly, inputs/outputs in [0, 2p):
    // (x, y) -> (x + y, (x - y) w).
    __device__ __forceinline__ void dif(uint32_t& x, uint32_t& y, W w) const {
        uint32_t s = x + y;
        uint32_t d = x - y + p2;
        x = umin32(s, s - p2);
        y = mulw(d, w);
    }
    // Cooley-Tukey (DIT) butterfly, inputs/outputs in [0, 4p):
    // (x, y) -> (x + y w, x - y w).
    __device__ __forceinline__ void dit(uint32_t& x, uint32_t& y, W w) const {
        uint32_t xx = umin32(x, x - p2);
        uint32_t t = mulw(y, w);
        x = xx + t;
        y = xx - t + p2;
    }
    // butterflies with twiddle w^0 = 1 (no product)
    __device__ __forceinline__ void dif1(uint32_t& x, uint32_t& y) const {
        uint32_t s = x + y;
        uint32_t d = x - y + p2;
        x = umin32(s, s - p2);
        y = umin32(d, d - p2);
    }
    __device__ __forceinline__ void dit1(uint32_t& x, uint32_t& y) const {
        uint32_t xx = umin32(x, x - p2);
        uint32_t yy = umin32(y, y - p2);
        x = xx + yy;
        y = xx - yy + p2;
    }
    // any x < 2^32 -> [0, 2p), congruent (the lazy range of the butterflies):
    // q = hi(x floor(2^32/p)) is floor(x/p) or one less (Function 8's argument
    // with the multiplier 1), so x - q p < 2p
    __device__ __forceinline__ uint32_t reduce_raw(uint32_t x) const { return x - __umulhi(x, pr) * p; }
    // [0, 4p) -> [0, p)
    __device__ __forceinline__ uint32_t canon(uint32_t x) const {
        x = umin32(x, x - p2);
        return umin32(x, x - p);
    }
    // general product of two values < 2p (pointwise spectrum product):
    // x y 2^-32 mod p in [0, p) (REDC; the 2^32 factor is folded into the
    // constant that multiplies afterwards).
    __device__ __forceinline__ uint32_t mul_redc(uint32_t x, uint32_t y) const {
        return redc32(x * y, __umulhi(x, y), p, pinv);
    }
};

// ----------------------------------------------------------------- 64 bit
// p = 2^64 - 2^32 + 1; EPS = 2^64 mod p = 2^32 - 1.  Values are kept in
// [0, 2^64) (not necessarily canonical) between operations.
struct FpG {
    typedef uint64_t T;
    typedef uint64_t W;
    static constexpr uint64_t P = 0xFFFFFFFF00000001ull;
    static constexpr uint64_t EPS = 0xFFFFFFFFull;

    // a + b for any a, b < 2^64: each carry out of 2^64 is worth EPS (2^64 = EPS
    // mod p), added as -c in the low word (EPS * c = 2^32 c - c); a second carry
    // leaves s < EPS, so the third fold cannot carry.  Branch-free carry chain.
    __device__ __forceinline__ static uint64_t add(uint64_t a, uint64_t b) {
        uint32_t s0, s1;
        asm("{\n\t.reg .u32 c, m;\n\t"
            "add.cc.u32      %0, %2, %4;\n\t"
            "addc.cc.u32     %1, %3, %5;\n\t"
            "addc.u32        c, 0, 0;\n\t"
            "sub.u32         m, 0, c;\n\t"
            "add.cc.u32      %0, %0, m;\n\t"
            "addc.cc.u32     %1, %1, 0;\n\t"
            "addc.u32        c, 0, 0;\n\t"
            "sub.u32         m, 0, c;\n\t"
            "add.cc.u32      %0, %0, m;\n\t"
            "addc.u32        %1, %1, 0;\n\t}"
            : "=&r"(s0), "=&r"(s1)
            : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
        return ((uint64_t)s1 << 32) | s0;
    }
    // a - b: each borrow is worth -EPS (+p = -EPS mod 2^64); symmetric to add.
    __device__ __forceinline__ static uint64_t sub(uint64_t a, uint64_t b) {
        uint32_t d0, d1;
        asm("{\n\t.reg .u32 m;\n\t"
            "sub.cc.u32      %0, %2, %4;\n\t"
            "subc.cc.u32     %1, %3, %5;\n\t"
            "subc.u32        m, 0, 0;\n\t"
            "sub.cc.u32      %0, %0, m;\n\t"
            "subc.cc.u32     %1, %1, 0;\n\t"
            "subc.u32        m, 0, 0;\n\t"
            "sub.cc.u32      %0, %0, m;\n\t"
            "subc.u32        %1, %1, 0;\n\t}"
            : "=&r"(d0), "=&r"(d1)
            : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
        return ((uint64_t)d1 << 32) | d0;
    }
    // 128-bit product from four 32 x 32 partial products (one mul/mad carry
    // chain: IMAD / IMAD.HI with carry), then with x = r0 + r1 2^32 + r2 2^64
    // + r3 2^96:  x = (r1:r0) - r3 + r2 (2^32 - 1)  (mod p), evaluated with
    // carry/borrow flags instead of compares (Python-checked in DESIGN.md).
    __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
        const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        uint32_t r0, r1, r2, r3;
        asm("mul.lo.u32      %0, %4, %6;\n\t"
            "mul.hi.u32      %1, %4, %6;\n\t"
            "mad.lo.cc.u32   %1, %4, %7, %1;\n\t"
            "madc.hi.u32     %2, %4, %7, 0;\n\t"
            "mad.lo.cc.u32   %1, %5, %6, %1;\n\t"
            "madc.hi.cc.u32  %2, %5, %6, %2;\n\t"
            "madc.hi.u32     %3, %5, %7, 0;\n\t"
            "mad.lo.cc.u32   %2, %5, %7, %2;\n\t"
            "addc.u32        %3, %3, 0;"
            : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
            : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
        uint32_t u0, u1, net;
        asm("{\n\t.reg .u32 t0, t1, bw;\n\t"
            "sub.cc.u32      t0, %3, %6;\n\t"     // t = (r1:r0) - r3, bw = -borrow
            "subc.cc.u32     t1, %4, 0;\n\t"
            "subc.u32        bw, 0, 0;\n\t"
            "sub.cc.u32      t0, t0, bw;\n\t"     // borrow: t -= EPS (no second borrow)
            "subc.u32        t1, t1, 0;\n\t"
            "sub.cc.u32      %0, t0, %5;\n\t"     // u = t - r2, borrow b2
            "subc.cc.u32     %1, t1, 0;\n\t"
            "subc.u32        %2, 0, 0;\n\t"
            "add.cc.u32      %1, %1, %5;\n\t"     // u += r2 2^32, net = carry + b2 in {0,1}
            "addc.u32        %2, %2, 0;\n\t}"
            : "=&r"(u0), "=&r"(u1), "=&r"(net)
            : "r"(r0), "r"(r1), "r"(r2), "r"(r3));
        // net = 1: one 2^64 wrap, add EPS (cannot overflow again)
        uint64_t r = ((uint64_t)u1 << 32) | u0;
        return r + (uint64_t)(0u - net);   // 0u - net = net ? 0xFFFFFFFF : 0
    }
    __device__ __forceinline__ static uint64_t canon(uint64_t x) { return x >= P ? x - P : x; }

    __device__ __forceinline__ uint64_t mulw(uint64_t x, W w) const { return mul(x, w); }
    __device__ __forceinline__ void dif(uint64_t& x, uint64_t& y, W w) const {
        uint64_t s = add(x, y);
        uint64_t d = sub(x, y);
        x = s;
        y = mul(d, w);
    }
    __device__ __forceinline__ void dit(uint64_t& x, uint64_t& y, W w) const {
        uint64_t t = mul(y, w);
        uint64_t s = add(x, t);
        y = sub(x, t);
        x = s;
    }
    __device__ __forceinline__ void dif1(uint64_t& x, uint64_t& y) const {
        uint64_t s = add(x, y);
        y = sub(x, y);
        x = s;
    }
    __device__ __forceinline__ void dit1(uint64_t& x, uint64_t& y) const { dif1(x, y); }
    __device__ __forceinline__ uint64_t mul_redc(uint64_t x, uint64_t y) const { return mul(x, y); }
};

// ----------------------------------------------------------------- FP64
// Residues of an odd prime p < 2^50 held as integral doubles in [0, p) (paper
// §3): products by Function 16 (m <= l - 2 = 50), sums by
// Function 17, every value canonical (2p can exceed 2^50, so no lazy range).
// Round-to-nearest intrinsics keep the compiler from contracting the
// sequences the proofs (Propositions 10-13) cover.
struct FpD {
    typedef double T;
    typedef double W;        // twiddle w (Function 16 with a2 = w)
    double p, u;             // u = 1.0 / p rounded to nearest
    __device__ __forceinline__ double add(double x, double y) const {
        const double a = __dadd_rn(x, y);
        const double b = __dsub_rn(a, p);
        return b < 0.0 ? a : b;
    }
    __device__ __forceinline__ double sub(double x, double y) const {
        const double a = __dsub_rn(x, y);
        return a < 0.0 ? __dadd_rn(a, p) : a;
    }
    __device__ __forceinline__ double mulw(double x, double w) const {   // Function 16
        const double h = __dmul_rn(x, w);
        const double l = __fma_rn(x, w, -h);
        const double c = floor(__dmul_rn(h, u));
        const double d = __fma_rn(-c, p, h);
        double e = __dadd_rn(d, l);
        e = e >= p ? __dsub_rn(e, p) : e;
        return e < 0.0 ? __dadd_rn(e, p) : e;
    }
    __device__ __forceinline__ void dif(double& x, double& y, W w) const {
        const double s = add(x, y), d = sub(x, y);
        x = s;
        y = mulw(d, w);
    }
    __device__ __forceinline__ void dit(double& x, double& y, W w) const {
        const double t = mulw(y, w);
        y = sub(x, t);
        x = add(x, t);
    }
    __device__ __forceinline__ void dif1(double& x, double& y) const {
        const double s = add(x, y), d = sub(x, y);
        x = s;
        y = d;
    }
    __device__ __forceinline__ void dit1(double& x, double& y) const { dif1(x, y); }
    __device__ __forceinline__ double canon(double x) const { return x; }
    __device__ __forceinline__ double mul_redc(double x, double y) const { return mulw(x, y); }
};

}  // namespace mm
