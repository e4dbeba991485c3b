// gold.cuh -- Goldilocks (p = 2^64 - 2^32 + 1) tile transforms of length
// 2^10 .. 2^13 for the 64-bit passes (BASELINE C4 / C5).
//
// Why a separate tile: on sm_100a the Goldilocks butterfly is bound by the
// integer ALU pipe (tools/probe64.cu: ~57 issue cycles per warp-butterfly, of
// which the modular add and sub with their 2^64 -> EPS folds are ~20 and the
// general product ~24).  This tile removes most of both:
//
//  * Structure (Algorithm 1 of the paper, applied inside the
//    tile): L = NA x 64 with j = 64 a + b.  The NA-point DFTs over a and the
//    64-point DFTs over b are themselves 8 x 8 (4 x 8, 2 x 8) splits, so every
//    butterfly twiddle is an 8th root of unity: w_8 = 2^(8S) with w_64 = 2^S
//    (2 has order 192 mod p: w_64 = 2^39 for the root 7^((p-1)/n)),
//    i.e. a shift plus the 2^64 = EPS / 2^96 = -1 reduction.  Only the
//    64-th-root twiddles between the 8-point stages and one w_L^(b k_a)
//    twiddle per element are table products.
//  * Delayed reduction: inside an 8-point DFT the values are 3-word integers
//    (U3, < 2^68); a sum is 3 adds, a difference x - y is x + K p - y with a
//    compile-time multiple K p of p above the bound of y (bounds tracked in
//    the comments).  A value is folded back to one 64-bit word only before a
//    product and at the output.
//
// Output orders are exactly those of the generic radix-2 tiles (ntt_core.cuh):
// forward = DIF natural -> bit-reversed (TFT order), inverse = DIT
// bit-reversed -> natural with the inverse root (unnormalised).  The shifts
// are compiled for w_64 = 2^39 (forward) / 2^153 (inverse), the 64-th root of
// the canonical root 7^((p-1)/n) and of every root whose 64-th root agrees
// with it; the kernel compares full[L/64] with that value at run time and
// runs the generic radix-8 tile for any other root of unity.
#pragma once
#include "arith.cuh"

namespace mm {
namespace gold {

constexpr uint64_t P = 0xFFFFFFFF00000001ull;
constexpr int S_FWD = 39;    // w_64 = 2^39 for w = 7^((p-1)/n)
constexpr int S_INV = 153;   // (2^39)^-1 = 2^(192-39)

// 2^K mod p as (NEG, C): 2^K = (-1)^NEG * C, C = 2^(K mod 96) mod p
template <int K_> struct Pow2 {
    static constexpr int K = ((K_ % 192) + 192) % 192;
    static constexpr bool NEG = K >= 96;
    static constexpr int KR = NEG ? K - 96 : K;
    static constexpr uint64_t C = KR < 64 ? (1ull << KR) : ((1ull << (KR - 32)) - (1ull << (KR - 64)));
};
template <int K> struct Pow2Val {   // 2^K mod p as one word
    static constexpr uint64_t v = Pow2<K>::NEG ? P - Pow2<K>::C : Pow2<K>::C;
};

// ---------------------------------------------------------------- 3-word values
struct U3 {
    uint32_t w0, w1, w2;
};
__device__ __forceinline__ U3 mk(uint64_t x) { return U3{(uint32_t)x, (uint32_t)(x >> 32), 0u}; }

__device__ __forceinline__ U3 add(const U3& a, const U3& b) {
    U3 r;
    asm("add.cc.u32 %0, %3, %6;\n\taddc.cc.u32 %1, %4, %7;\n\taddc.u32 %2, %5, %8;"
        : "=r"(r.w0), "=r"(r.w1), "=r"(r.w2)
        : "r"(a.w0), "r"(a.w1), "r"(a.w2), "r"(b.w0), "r"(b.w1), "r"(b.w2));
    return r;
}
__device__ __forceinline__ U3 add(const U3& a, uint64_t b) {
    U3 r;
    asm("add.cc.u32 %0, %3, %6;\n\taddc.cc.u32 %1, %4, %7;\n\taddc.u32 %2, %5, 0;"
        : "=r"(r.w0), "=r"(r.w1), "=r"(r.w2)
        : "r"(a.w0), "r"(a.w1), "r"(a.w2), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
    return r;
}
__device__ __forceinline__ U3 add(uint64_t a, uint64_t b) {
    U3 r;
    asm("add.cc.u32 %0, %3, %5;\n\taddc.cc.u32 %1, %4, %6;\n\taddc.u32 %2, 0, 0;"
        : "=r"(r.w0), "=r"(r.w1), "=r"(r.w2)
        : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
    return r;
}
// a + K p - b; the caller guarantees b < K p (K a power of two, K p < 2^96).
// K p = K 2^64 - K 2^32 + K has words (K, 2^32 - K, K - 1).
template <uint32_t K> __device__ __forceinline__ U3 subk(const U3& a, const U3& b) {
    U3 t, r;
    asm("add.cc.u32 %0, %3, %6;\n\taddc.cc.u32 %1, %4, %7;\n\taddc.u32 %2, %5, %8;"
        : "=r"(t.w0), "=r"(t.w1), "=r"(t.w2)
        : "r"(a.w0), "r"(a.w1), "r"(a.w2), "n"(K), "n"((uint32_t)(0u - K)), "n"(K - 1));
    asm("sub.cc.u32 %0, %3, %6;\n\tsubc.cc.u32 %1, %4, %7;\n\tsubc.u32 %2, %5, %8;"
        : "=r"(r.w0), "=r"(r.w1), "=r"(r.w2)
        : "r"(t.w0), "r"(t.w1), "r"(t.w2), "r"(b.w0), "r"(b.w1), "r"(b.w2));
    return r;
}
template <uint32_t K> __device__ __forceinline__ U3 subk(const U3& a, uint64_t b) { return subk<K>(a, mk(b)); }
template <uint32_t K> __device__ __forceinline__ U3 subk(uint64_t a, uint64_t b) { return subk<K>(mk(a), mk(b)); }

// U3 (w2 < 2^31) -> one word in [0, 2^64) congruent mod p:
// v = (w1:w0) + w2 2^64 = (w1:w0) + w2 EPS; at most one carry, folded as EPS
// (the fold cannot carry again: the value minus 2^64 is < w2 2^32).
__device__ __forceinline__ uint64_t fold(const U3& a) {
    uint32_t r0, r1;
    asm("{\n\t.reg .u32 c;\n\t"
        "mad.lo.cc.u32 %0, %4, 0xFFFFFFFF, %2;\n\t"
        "madc.hi.cc.u32 %1, %4, 0xFFFFFFFF, %3;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "mad.lo.cc.u32 %0, c, 0xFFFFFFFF, %0;\n\t"
        "madc.hi.u32 %1, c, 0xFFFFFFFF, %1;\n\t}"
        : "=&r"(r0), "=&r"(r1)
        : "r"(a.w0), "r"(a.w1), "r"(a.w2));
    return ((uint64_t)r1 << 32) | r0;
}

// (hi : 0) + m EPS reduced to one word in [0, 2^64): the 65-bit sum's carry
// is folded as EPS (cannot carry again: the sum minus 2^64 is < 2^64 - 2^33)
__device__ __forceinline__ uint64_t add_eps(uint32_t hi, uint32_t m) {
    uint32_t r0, r1;
    asm("{\n\t.reg .u32 c;\n\t"
        "mad.lo.cc.u32 %0, %3, 0xFFFFFFFF, 0;\n\t"
        "madc.hi.cc.u32 %1, %3, 0xFFFFFFFF, %2;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "mad.lo.cc.u32 %0, c, 0xFFFFFFFF, %0;\n\t"
        "madc.hi.u32 %1, c, 0xFFFFFFFF, %1;\n\t}"
        : "=&r"(r0), "=&r"(r1)
        : "r"(hi), "r"(m));
    return ((uint64_t)r1 << 32) | r0;
}
// u - (d1 : d0) mod p for u, (d1 : d0) in [0, 2^64) with (d1 : d0) < p: one
// borrow, repaid by - EPS (= + p mod 2^64; cannot borrow again since the
// subtrahend is below p)
__device__ __forceinline__ uint64_t sub_word(uint64_t u, uint32_t d0, uint32_t d1) {
    uint32_t r0, r1;
    asm("{\n\t.reg .u32 m;\n\t"
        "sub.cc.u32 %0, %2, %4;\n\tsubc.cc.u32 %1, %3, %5;\n\tsubc.u32 m, 0, 0;\n\t"
        "sub.cc.u32 %0, %0, m;\n\tsubc.u32 %1, %1, 0;\n\t}"
        : "=&r"(r0), "=&r"(r1)
        : "r"((uint32_t)u), "r"((uint32_t)(u >> 32)), "r"(d0), "r"(d1));
    return ((uint64_t)r1 << 32) | r0;
}
__device__ __forceinline__ uint64_t sub_small(uint64_t u, uint32_t d) { return sub_word(u, d, 0u); }

// x 2^K (0 <= K < 96) for x in [0, 2^64), result in [0, 2^64)
template <int K> __device__ __forceinline__ uint64_t mul2k(uint64_t x) {
    if constexpr (K == 0) {
        return x;
    } else if constexpr (K < 32) {
        const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
        U3 y;
        y.w0 = x0 << K;
        y.w1 = __funnelshift_l(x0, x1, K);
        y.w2 = x1 >> (32 - K);
        return fold(y);
    } else if constexpr (K < 64) {
        // y = x 2^(K-32) = (y2 y1 y0); x 2^K = y0 2^32 + y1 2^64 + y2 2^96
        //   = (y0 : 0) + y1 EPS - y2   (2^64 = EPS, 2^96 = -1)
        constexpr int R = K - 32;
        const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
        const uint32_t y0 = x0 << R, y1 = R ? __funnelshift_l(x0, x1, R) : x1, y2 = R ? x1 >> (32 - R) : 0u;
        return sub_small(add_eps(y0, y1), y2);
    } else {
        // y = x 2^(K-64) = (y2 y1 y0); x 2^K = y 2^64 = y0 EPS + y1 2^96 + y2 2^128
        //   = y0 EPS - y1 - y2 2^32   (2^128 = 2^32 2^96 = -2^32)
        constexpr int R = K - 64;
        const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
        const uint32_t y0 = x0 << R, y1 = R ? __funnelshift_l(x0, x1, R) : x1, y2 = R ? x1 >> (32 - R) : 0u;
        // y1 + y2 2^32 < 2^64 since y2 < 2^R <= 2^31: one subtrahend word pair
        return sub_word(add_eps(0u, y0), y1, y2);
    }
}

// -x mod p for x in [0, 2^64): p - x, plus p on borrow (p - x + p > 0, and the
// wrapped difference exceeds EPS so the repayment cannot borrow again)
__device__ __forceinline__ uint64_t neg(uint64_t x) { return sub_word(P, (uint32_t)x, (uint32_t)(x >> 32)); }

// x 2^E mod p for a compile-time E (any sign / size)
template <int E> __device__ __forceinline__ uint64_t mulpow(uint64_t x) {
    typedef Pow2<E> W;
    const uint64_t y = mul2k<W::KR>(x);
    return W::NEG ? neg(y) : y;
}

__host__ __device__ constexpr int brev3c(int x) { return ((x & 1) << 2) | (x & 2) | ((x >> 2) & 1); }
__host__ __device__ constexpr int brev2c(int x) { return ((x & 1) << 1) | ((x >> 1) & 1); }

// v[t] *= w_64^(STEP D r(t)) = 2^(S STEP D r(t)) for t = T .. R-1, r(t) the
// bit-reversed t (the frequency held at position t after a DIF of R points)
template <int S, int STEP, int D, int R, int T> struct Rot {
    __device__ __forceinline__ static void run(uint64_t v[8]) {
        if constexpr (T < R) {
            constexpr int r = R == 8 ? brev3c(T) : R == 4 ? brev2c(T) : T;
            v[T] = mulpow<S * STEP * D * r>(v[T]);
            Rot<S, STEP, D, R, T + 1>::run(v);
        }
    }
};
// the same with a warp-uniform run-time digit d in [0, 8)
template <int S, int STEP, int R> __device__ __forceinline__ void rot(uint64_t v[8], int d) {
    switch (d) {
        case 0: break;
        case 1: Rot<S, STEP, 1, R, 1>::run(v); break;
        case 2: Rot<S, STEP, 2, R, 1>::run(v); break;
        case 3: Rot<S, STEP, 3, R, 1>::run(v); break;
        case 4: Rot<S, STEP, 4, R, 1>::run(v); break;
        case 5: Rot<S, STEP, 5, R, 1>::run(v); break;
        case 6: Rot<S, STEP, 6, R, 1>::run(v); break;
        default: Rot<S, STEP, 7, R, 1>::run(v); break;
    }
}

// ---------------------------------------------------------------- 8 / 4-point kernels
// In each DFT below the twiddle w_8^t = 2^(8 S t) (w_4 = 2^(16 S)); a twiddle
// -C (Pow2::NEG) is applied by swapping the operands of the difference (DIF)
// or of the two outputs (DIT).  Bounds: inputs < 2^64; comments give the
// bound of every intermediate; every subk<K> has its subtrahend < K p
// (p > 2^63, so K p > 2^(63 + log2 K)).

// DIF levels of span 2 and 1 of the 8-point kernel below (shared by dif8 and
// dif8_zh): inputs s_i < 2^65, d0 < 2^66, d1..d3 < 2^64
template <int S>
__device__ __forceinline__ void dif8_l23(uint64_t v[8], const U3& s0, const U3& s1, const U3& s2, const U3& s3,
                                         const U3& d0, uint64_t d1, uint64_t d2, uint64_t d3);

// DIF, natural in, bit-reversed out (positions of the radix-2 network)
template <int S> __device__ __forceinline__ void dif8(uint64_t v[8]) {
    typedef Pow2<8 * S> W1;
    typedef Pow2<16 * S> W2;
    typedef Pow2<24 * S> W3;
    // level span 4
    const U3 s0 = add(v[0], v[4]), s1 = add(v[1], v[5]), s2 = add(v[2], v[6]), s3 = add(v[3], v[7]);   // < 2^65
    const U3 d0 = subk<2>(v[0], v[4]);                                                                     // < 2^66
    const uint64_t d1 = mul2k<W1::KR>(fold(W1::NEG ? subk<2>(v[5], v[1]) : subk<2>(v[1], v[5])));
    const uint64_t d2 = mul2k<W2::KR>(fold(W2::NEG ? subk<2>(v[6], v[2]) : subk<2>(v[2], v[6])));
    const uint64_t d3 = mul2k<W3::KR>(fold(W3::NEG ? subk<2>(v[7], v[3]) : subk<2>(v[3], v[7])));
    dif8_l23<S>(v, s0, s1, s2, s3, d0, d1, d2, d3);
}

// the same with v[4..7] = 0 (the upper half of a zero-padded column): the
// span-4 level is v_i, v_i w_8^i -- no sums, differences or folds (the
// generic kernel cannot see through its inline-PTX carry chains)
template <int S> __device__ __forceinline__ void dif8_zh(uint64_t v[8]) {
    typedef Pow2<8 * S> W1;
    typedef Pow2<16 * S> W2;
    typedef Pow2<24 * S> W3;
    const uint64_t d1 = mul2k<W1::KR>(W1::NEG ? neg(v[1]) : v[1]);
    const uint64_t d2 = mul2k<W2::KR>(W2::NEG ? neg(v[2]) : v[2]);
    const uint64_t d3 = mul2k<W3::KR>(W3::NEG ? neg(v[3]) : v[3]);
    dif8_l23<S>(v, mk(v[0]), mk(v[1]), mk(v[2]), mk(v[3]), mk(v[0]), d1, d2, d3);
}

template <int S>
__device__ __forceinline__ void dif8_l23(uint64_t v[8], const U3& s0, const U3& s1, const U3& s2, const U3& s3,
                                         const U3& d0, uint64_t d1, uint64_t d2, uint64_t d3) {
    typedef Pow2<16 * S> W2;
    // level span 2 (twiddles 1, w_4)
    const U3 a0 = add(s0, s2);                                                        // < 2^66
    const U3 a2 = subk<4>(s0, s2);                                                    // < 2^67
    const U3 a1 = add(s1, s3);                                                        // < 2^66
    const uint64_t a3 = mul2k<W2::KR>(fold(W2::NEG ? subk<4>(s3, s1) : subk<4>(s1, s3)));
    const U3 b0 = add(d0, d2);                                                        // < 2^67
    const U3 b2 = subk<2>(d0, d2);                                                    // < 2^67
    const U3 b1 = add(d1, d3);                                                        // < 2^65
    const uint64_t b3 = mul2k<W2::KR>(fold(W2::NEG ? subk<2>(d3, d1) : subk<2>(d1, d3)));
    // level span 1 (twiddle 1); all outputs < 2^68
    v[0] = fold(add(a0, a1));
    v[1] = fold(subk<8>(a0, a1));
    v[2] = fold(add(a2, a3));
    v[3] = fold(subk<2>(a2, a3));
    v[4] = fold(add(b0, b1));
    v[5] = fold(subk<4>(b0, b1));
    v[6] = fold(add(b2, b3));
    v[7] = fold(subk<2>(b2, b3));
}

// DIT, bit-reversed in, natural out; S = exponent of the (inverse) w_64
template <int S> __device__ __forceinline__ void dit8(uint64_t v[8]) {
    typedef Pow2<8 * S> W1;
    typedef Pow2<16 * S> W2;
    typedef Pow2<24 * S> W3;
    // level span 1
    const U3 e0 = add(v[0], v[1]), e2 = add(v[2], v[3]), e4 = add(v[4], v[5]), e6 = add(v[6], v[7]);   // < 2^65
    const U3 e1 = subk<2>(v[0], v[1]), e3 = subk<2>(v[2], v[3]);                                           // < 2^66
    const U3 e5 = subk<2>(v[4], v[5]), e7 = subk<2>(v[6], v[7]);
    // level span 2: pairs (0,2) w = 1, (1,3) w = w_4
    const U3 f0 = add(e0, e2);                  // < 2^66
    const U3 f2 = subk<4>(e0, e2);              // < 2^67
    const uint64_t t3 = mul2k<W2::KR>(fold(e3));
    const U3 f1 = W2::NEG ? subk<2>(e1, t3) : add(e1, t3);   // < 2^67
    const U3 f3 = W2::NEG ? add(e1, t3) : subk<2>(e1, t3);
    const U3 f4 = add(e4, e6);
    const U3 f6 = subk<4>(e4, e6);
    const uint64_t t7 = mul2k<W2::KR>(fold(e7));
    const U3 f5 = W2::NEG ? subk<2>(e5, t7) : add(e5, t7);
    const U3 f7 = W2::NEG ? add(e5, t7) : subk<2>(e5, t7);
    // level span 4: pairs (t, t+4) with w_8^t; outputs < 2^68
    v[0] = fold(add(f0, f4));
    v[4] = fold(subk<8>(f0, f4));               // f4 < 2^66
    const uint64_t u1 = mul2k<W1::KR>(fold(f5));
    const uint64_t u2 = mul2k<W2::KR>(fold(f6));
    const uint64_t u3 = mul2k<W3::KR>(fold(f7));
    v[1] = fold(W1::NEG ? subk<2>(f1, u1) : add(f1, u1));
    v[5] = fold(W1::NEG ? add(f1, u1) : subk<2>(f1, u1));
    v[2] = fold(W2::NEG ? subk<2>(f2, u2) : add(f2, u2));
    v[6] = fold(W2::NEG ? add(f2, u2) : subk<2>(f2, u2));
    v[3] = fold(W3::NEG ? subk<2>(f3, u3) : add(f3, u3));
    v[7] = fold(W3::NEG ? add(f3, u3) : subk<2>(f3, u3));
}

template <int S> __device__ __forceinline__ void dif4(uint64_t v[4]) {
    typedef Pow2<16 * S> W2;
    const U3 s0 = add(v[0], v[2]), s1 = add(v[1], v[3]);           // < 2^65
    const U3 d0 = subk<2>(v[0], v[2]);                              // < 2^66
    const uint64_t d1 = mul2k<W2::KR>(fold(W2::NEG ? subk<2>(v[3], v[1]) : subk<2>(v[1], v[3])));
    v[0] = fold(add(s0, s1));
    v[1] = fold(subk<4>(s0, s1));
    v[2] = fold(add(d0, d1));
    v[3] = fold(subk<2>(d0, d1));
}
template <int S> __device__ __forceinline__ void dit4(uint64_t v[4]) {
    typedef Pow2<16 * S> W2;
    const U3 e0 = add(v[0], v[1]), e2 = add(v[2], v[3]);           // < 2^65
    const U3 e1 = subk<2>(v[0], v[1]), e3 = subk<2>(v[2], v[3]);   // < 2^66
    const uint64_t t = mul2k<W2::KR>(fold(e3));
    v[0] = fold(add(e0, e2));
    v[2] = fold(subk<4>(e0, e2));
    v[1] = fold(W2::NEG ? subk<2>(e1, t) : add(e1, t));
    v[3] = fold(W2::NEG ? add(e1, t) : subk<2>(e1, t));
}

__device__ __forceinline__ int brev3(int x) { return ((x & 1) << 2) | (x & 2) | ((x >> 2) & 1); }
__device__ __forceinline__ int brev2(int x) { return ((x & 1) << 1) | ((x >> 1) & 1); }

// 2-point DFT (NA = 16 tiles): (x + y, x - y), the same in both directions
__device__ __forceinline__ void dft2(uint64_t v[2]) {
    const uint64_t x = v[0], y = v[1];
    v[0] = fold(add(x, y));
    v[1] = fold(subk<2>(x, y));
}

// chunk q of the stages over the b digits -> (A, the digit d, sub-transform ct):
// lanes take consecutive A; when NA < 32 they also span sub-transforms so that
// d stays warp-uniform (rot's switch)
template <int NA, int CT> __device__ __forceinline__ void decode_a(int q, int& A, int& d, int& ct) {
    A = q % NA;
    if constexpr (NA >= 32) {
        d = (q / NA) & 7;
        ct = q / (NA * 8);
    } else {
        static_assert(NA * CT >= 32 && CT % (32 / NA) == 0, "warp-uniform digit needs 32 / NA sub-transforms");
        ct = (q / NA) % CT;
        d = (q / (NA * CT)) & 7;
    }
}

// ---------------------------------------------------------------- tile passes
// One length-LN sub-transform per (c, h): element j of it at Lay::addr(c, h*LN + j);
// full[TS * e] = w_LN^e (natural powers, e < LN); the 64-th roots w_64^e = 2^(S e)
// are shifts (rot), the digit they depend on being warp-uniform.
// LN = NA * 64 with NA in {16, 32, 64}; RA = NA / 8.
// stage A of dif_ln on RA values in registers: the RA-point DFT over ah
// (j = 512 ah + 64 al + b), then w_NA^(al r) (al warp-uniform)
template <int RA, int S> __device__ __forceinline__ void dif_a(uint64_t v[8], int al) {
    if constexpr (RA == 8) dif8<S>(v);
    else if constexpr (RA == 4) dif4<S>(v);
    else dft2(v);
    rot<S, 8 / RA, RA>(v, al);
}

template <class Lay, int LN, int H, int NT, int S>
__device__ __forceinline__ void dif_ln_bcd(uint64_t* s, const uint64_t* __restrict__ full, int TS, int LQ);

template <class Lay, int LN, int H, int NT, int S>
__device__ __forceinline__ void dif_ln(uint64_t* s, const uint64_t* __restrict__ full, int TS, int LQ) {
    constexpr int NA = LN / 64, RA = NA / 8, C = Lay::C;
    constexpr int CT = C * H;
    // stage A: RA-point DFTs over ah (j = 512 ah + 64 al + b), then w_NA^(al r)
    for (int q = threadIdx.x; q < CT * 512; q += NT) {
        const int b = q & 63, al = (q >> 6) & 7, ct = q >> 9;
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 64 * al + b);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < RA; t++) v[t] = p0[Lay::off(512 * t)];
        dif_a<RA, S>(v, al);
#pragma unroll
        for (int t = 0; t < RA; t++) p0[Lay::off(512 * t)] = v[t];
    }
    __syncthreads();
    dif_ln_bcd<Lay, LN, H, NT, S>(s, full, TS, LQ);
}

// stages B-D of dif_ln (stage A's output in s)
template <class Lay, int LN, int H, int NT, int S>
__device__ __forceinline__ void dif_ln_bcd(uint64_t* s, const uint64_t* __restrict__ full, int TS, int LQ) {
    constexpr int NA = LN / 64, RA = NA / 8, C = Lay::C;
    constexpr int CT = C * H;
    // stage B: 8-point DFTs over al (j = 512 P + 64 al + b), then w_LN^(b k_a)
    for (int q = threadIdx.x; q < CT * RA * 64; q += NT) {
        const int b = q & 63, P = (q >> 6) % RA, ct = q / (64 * RA);
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 512 * P + b);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(64 * t)];
        dif8<S>(v);
        const int r = RA == 8 ? brev3(P) : RA == 4 ? brev2(P) : P;
#pragma unroll
        for (int t = 0; t < 8; t++) {
            const int ka = r + RA * brev3(t);
            v[t] = FpG::mul(v[t], __ldg(full + TS * (b * ka)));
        }
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(64 * t)] = v[t];
    }
    __syncthreads();
    // stage C: 8-point DFTs over bh (j = 64 A + 8 bh + bl), then w_64^(bl r)
    for (int q = threadIdx.x; q < CT * NA * 8; q += NT) {
        int A, bl, ct;
        decode_a<NA, CT>(q, A, bl, ct);
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 64 * A + bl);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(8 * t)];
        dif8<S>(v);
        rot<S, 1, 8>(v, bl);            // w_64^(bl r), bl warp-uniform
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(8 * t)] = v[t];
    }
    __syncthreads();
    // stage D: 8-point DFTs over bl (j = 64 A + 8 P + bl)
    for (int q = threadIdx.x; q < CT * NA * 8; q += NT) {
        int A, P, ct;
        decode_a<NA, CT>(q, A, P, ct);
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 64 * A + 8 * P);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(t)];
        dif8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(t)] = v[t];
    }
    __syncthreads();
}

template <class Lay, int LN, int H, int NT, int S>
__device__ __forceinline__ void dit_ln(uint64_t* s, const uint64_t* __restrict__ full, int TS, int LQ) {
    constexpr int NA = LN / 64, RA = NA / 8, C = Lay::C;
    constexpr int CT = C * H;
    // stage D': inverse 8-point over the bl digit
    for (int q = threadIdx.x; q < CT * NA * 8; q += NT) {
        int A, P, ct;
        decode_a<NA, CT>(q, A, P, ct);
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 64 * A + 8 * P);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(t)];
        dit8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(t)] = v[t];
    }
    __syncthreads();
    // stage C': w_64^-(bl r) then inverse 8-point over bh
    for (int q = threadIdx.x; q < CT * NA * 8; q += NT) {
        int A, bl, ct;
        decode_a<NA, CT>(q, A, bl, ct);
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 64 * A + bl);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(8 * t)];
        rot<S, 1, 8>(v, bl);
        dit8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(8 * t)] = v[t];
    }
    __syncthreads();
    // stage B': w_LN^-(b k_a) then inverse 8-point over al
    for (int q = threadIdx.x; q < CT * RA * 64; q += NT) {
        const int b = q & 63, P = (q >> 6) % RA, ct = q / (64 * RA);
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 512 * P + b);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(64 * t)];
        const int r = RA == 8 ? brev3(P) : RA == 4 ? brev2(P) : P;
#pragma unroll
        for (int t = 0; t < 8; t++) {
            const int ka = r + RA * brev3(t);
            v[t] = FpG::mul(v[t], __ldg(full + TS * (b * ka)));
        }
        dit8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(64 * t)] = v[t];
    }
    __syncthreads();
    // stage A': w_NA^-(al r) then inverse RA-point over ah
    for (int q = threadIdx.x; q < CT * 512; q += NT) {
        const int b = q & 63, al = (q >> 6) & 7, ct = q >> 9;
        const int c = ct / H, h = ct % H;
        uint64_t* p0 = s + Lay::addr(c, h * LN + 64 * al + b);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < RA; t++) v[t] = p0[Lay::off(512 * t)];
        rot<S, 8 / RA, RA>(v, al);
        if constexpr (RA == 8) dit8<S>(v);
        else if constexpr (RA == 4) dit4<S>(v);
        else dft2(v);
#pragma unroll
        for (int t = 0; t < RA; t++) p0[Lay::off(512 * t)] = v[t];
    }
    __syncthreads();
}

// dit_ln for one 4096-point sub-transform per column (H = 1), split so that a
// tile's first half can be transformed while its second half is still in
// flight: stages D', C', B' touch only the rows of one 2048-row half
// (D', C': rows 64 A + [0, 64) with A in [32 hh, 32 hh + 32); B': rows
// 512 P + [0, 512) with P in [4 hh, 4 hh + 4)), stage A' needs both
template <class Lay, int NT, int S>
__device__ __forceinline__ void dit4096_half(uint64_t* s, const uint64_t* __restrict__ full, int hh) {
    constexpr int C = Lay::C;
    for (int q = threadIdx.x; q < C * 32 * 8; q += NT) {       // D': 8-point over bl
        const int A = 32 * hh + (q & 31), P = (q >> 5) & 7, c = q >> 8;
        uint64_t* p0 = s + Lay::addr(c, 64 * A + 8 * P);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(t)];
        dit8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(t)] = v[t];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < C * 32 * 8; q += NT) {       // C': w_64^-(bl r), 8-point over bh
        const int A = 32 * hh + (q & 31), bl = (q >> 5) & 7, c = q >> 8;   // bl warp-uniform
        uint64_t* p0 = s + Lay::addr(c, 64 * A + bl);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(8 * t)];
        rot<S, 1, 8>(v, bl);
        dit8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(8 * t)] = v[t];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < C * 4 * 64; q += NT) {       // B': w_4096^-(b k_a), 8-point over al
        const int b = q & 63, P = 4 * hh + ((q >> 6) & 3), c = q >> 8;
        uint64_t* p0 = s + Lay::addr(c, 512 * P + b);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(64 * t)];
        const int r = brev3(P);
#pragma unroll
        for (int t = 0; t < 8; t++) {
            const int ka = r + 8 * brev3(t);
            v[t] = FpG::mul(v[t], __ldg(full + b * ka));
        }
        dit8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(64 * t)] = v[t];
    }
    __syncthreads();
}
template <class Lay, int NT, int S>
__device__ __forceinline__ void dit4096_a(uint64_t* s) {
    constexpr int C = Lay::C;
    for (int q = threadIdx.x; q < C * 512; q += NT) {           // A': w_64^-(al r), 8-point over ah
        const int b = q & 63, al = (q >> 6) & 7, c = q >> 9;
        uint64_t* p0 = s + Lay::addr(c, 64 * al + b);
        uint64_t v[8];
#pragma unroll
        for (int t = 0; t < 8; t++) v[t] = p0[Lay::off(512 * t)];
        rot<S, 1, 8>(v, al);
        dit8<S>(v);
#pragma unroll
        for (int t = 0; t < 8; t++) p0[Lay::off(512 * t)] = v[t];
    }
    __syncthreads();
}

// Whole-tile transforms, L = 2^LOGL in {2^11, 2^12, 2^13}; full = w_L^e, e < L.
template <class Lay, int LOGL, int NT>
__device__ __forceinline__ void tile_dif(uint64_t* s, const uint64_t* __restrict__ full) {
    constexpr int L = 1 << LOGL, C = Lay::C;
    if constexpr (LOGL == 13) {
        // radix-2 level of span 4096 (twiddle w_8192^j), then two 4096-point halves
        for (int q = threadIdx.x; q < C * 4096; q += NT) {
            const int j = q & 4095, c = q >> 12;
            uint64_t* px = s + Lay::addr(c, j);
            uint64_t* py = s + Lay::addr(c, j + 4096);
            const uint64_t x = *px, y = *py;
            *px = FpG::add(x, y);
            *py = FpG::mul(FpG::sub(x, y), __ldg(full + j));
        }
        __syncthreads();
        dif_ln<Lay, 4096, 2, NT, S_FWD>(s, full, 2, L / 64);
    } else {
        dif_ln<Lay, L, 1, NT, S_FWD>(s, full, 1, L / 64);
    }
}
template <class Lay, int LOGL, int NT>
__device__ __forceinline__ void tile_dit(uint64_t* s, const uint64_t* __restrict__ full) {
    constexpr int L = 1 << LOGL, C = Lay::C;
    if constexpr (LOGL == 13) {
        dit_ln<Lay, 4096, 2, NT, S_INV>(s, full, 2, L / 64);
        for (int q = threadIdx.x; q < C * 4096; q += NT) {
            const int j = q & 4095, c = q >> 12;
            uint64_t* px = s + Lay::addr(c, j);
            uint64_t* py = s + Lay::addr(c, j + 4096);
            const uint64_t x = *px, t = FpG::mul(*py, __ldg(full + j));
            *px = FpG::add(x, t);
            *py = FpG::sub(x, t);
        }
        __syncthreads();
    } else {
        dit_ln<Lay, L, 1, NT, S_INV>(s, full, 1, L / 64);
    }
}

}  // namespace gold
}  // namespace mm
