// ntt_core.cuh -- shared-memory tile transforms for sm_100a, compile-time shaped.
//
// A "tile" is C independent length-L transforms (L = 2^LOGL) held in shared
// memory.  Butterfly levels run in register groups of radix RR = 2^r: a thread
// loads RR elements of one transform, runs r levels in registers and writes
// them back; groups are separated by __syncthreads().  Every size is a
// template parameter, so all index arithmetic folds into immediate offsets
// (one base address per chunk of RR elements).
//
//   forward  = decimation in frequency (Gentleman-Sande): natural in,
//              bit-mirrored out -- the TFT order TFT_w of P:893 with l = n;
//   inverse  = decimation in time (Cooley-Tukey): bit-mirrored in, natural
//              out, root w^-1 (inverse of Algorithm 1's TFFT).
//
// Twiddles: per-level table tw[m + i] = w_{2m}^i (0 <= i < m, m = 1 .. L/2);
// for 32-bit moduli each entry carries the fixed-multiplicand companion
// floor(w 2^32 / p) (Function 8).  Butterflies whose twiddle is
// w^0 = 1 at compile time skip the product.
//
// Shared-memory layouts (conflict-free for every group of the transform):
//   RowLayout<T, LOGL, C> : transform c at c*SROW, element j at j + (j >> 4)
//                           (one pad element per 16), SROW = 16 mod 32 banks.
//   ColLayout<T, LOGL, C> : element (j, c) at j*C + c (the global row-major
//                           order of a column tile), used when C*sizeof(T) = 128 B
//                           so that the 32 lanes of a warp share one base.
#pragma once
#include "arith.cuh"

namespace mm {

__device__ __forceinline__ int brev(int i, int k) { return k == 0 ? 0 : (int)(__brev((unsigned)i) >> (32 - k)); }

template <int X> struct Log2 { enum { v = 1 + Log2<X / 2>::v }; };
template <> struct Log2<1> { enum { v = 0 }; };

template <class T, int LOGL, int C_> struct RowLayout {
    static constexpr int L = 1 << LOGL;
    static constexpr int C = C_;
    static constexpr int WORDS = sizeof(T) / 4;
    static constexpr int PADL = L + (L >> 4);
    // row pitch in elements: PADL rounded up so that pitch*WORDS = 16 (mod 32) banks
    static constexpr int SROW = [] {
        int s = PADL;
        while (((s * WORDS) & 31) != 16 && L >= 16) s++;
        return s;
    }();
    static constexpr int ELEMS = C * SROW;
    static constexpr bool COL = false;
    __device__ __forceinline__ static int addr(int c, int j) { return c * SROW + j + (j >> 4); }
    // chunk -> (c, b) with b the position of the chunk inside its transform
    template <int PER> __device__ __forceinline__ static void split(int ch, int& c, int& b) {
        c = ch / PER;
        b = ch % PER;
    }
    // base address of element j = base (per chunk) + OFF(t*M) with OFF(x) = x + (x >> 4)
    __device__ __forceinline__ static int chunk_base(int c, int base) { return c * SROW + base + (base >> 4); }
    __host__ __device__ static constexpr int off(int x) { return x + (x >> 4); }
};

template <class T, int LOGL, int C_> struct ColLayout {
    static constexpr int L = 1 << LOGL;
    static constexpr int C = C_;
    static constexpr int ELEMS = C * L;
    static constexpr bool COL = true;
    __device__ __forceinline__ static int addr(int c, int j) { return j * C + c; }
    template <int PER> __device__ __forceinline__ static void split(int ch, int& c, int& b) {
        c = ch % C;
        b = ch / C;
    }
    __device__ __forceinline__ static int chunk_base(int c, int base) { return base * C + c; }
    __host__ __device__ static constexpr int off(int x) { return x * C; }
};

// ---------------------------------------------------------------- DIF group
// Levels S0 .. S0+r-1 (spans L/2^(S0+1) ... L/2^(S0+r)).
template <class F, class Lay, int LOGL, int S0, int r, int NT>
__device__ __forceinline__ void dif_group(const F& f, typename F::T* s, const typename F::W* tw) {
    typedef typename F::T T;
    constexpr int RR = 1 << r;
    constexpr int L = 1 << LOGL;
    constexpr int lm = LOGL - S0 - r;          // log2 of the span of the last level of the group
    constexpr int M = 1 << lm;
    constexpr int PER = L / RR;
    constexpr int CHUNKS = Lay::C * PER;
#pragma unroll 1
    for (int ch = threadIdx.x; ch < CHUNKS; ch += NT) {
        int c, b;
        Lay::template split<PER>(ch, c, b);
        const int lo = b & (M - 1), hi = b >> lm;
        const int base = lo + (hi << (lm + r));
        T* p = s + Lay::chunk_base(c, base);
        const typename F::W* twp = tw + lo;
        T v[RR];
#pragma unroll
        for (int t = 0; t < RR; t++) v[t] = p[Lay::off(t * M)];
#pragma unroll
        for (int q = 0; q < r; q++) {
            const int h = RR >> (q + 1);
            const int m = M * h;
#pragma unroll
            for (int t = 0; t < RR; t++) {
                if (t & h) continue;
                const int k = (t & (h - 1)) * M;
                if (M == 1 && k == 0) f.dif1(v[t], v[t + h]);         // twiddle w^0 = 1
                else f.dif(v[t], v[t + h], twp[m + k]);
            }
        }
#pragma unroll
        for (int t = 0; t < RR; t++) p[Lay::off(t * M)] = v[t];
    }
}

// ---------------------------------------------------------------- DIT group
// Spans 2^S0 .. 2^(S0+r-1).
template <class F, class Lay, int LOGL, int S0, int r, int NT>
__device__ __forceinline__ void dit_group(const F& f, typename F::T* s, const typename F::W* tw) {
    typedef typename F::T T;
    constexpr int RR = 1 << r;
    constexpr int L = 1 << LOGL;
    constexpr int M = 1 << S0;                 // span of the first level of the group
    constexpr int PER = L / RR;
    constexpr int CHUNKS = Lay::C * PER;
#pragma unroll 1
    for (int ch = threadIdx.x; ch < CHUNKS; ch += NT) {
        int c, b;
        Lay::template split<PER>(ch, c, b);
        const int lo = b & (M - 1), hi = b >> S0;
        const int base = lo + (hi << (S0 + r));
        T* p = s + Lay::chunk_base(c, base);
        const typename F::W* twp = tw + lo;
        T v[RR];
#pragma unroll
        for (int t = 0; t < RR; t++) v[t] = p[Lay::off(t * M)];
#pragma unroll
        for (int q = 0; q < r; q++) {
            const int h = 1 << q;
            const int m = M * h;
#pragma unroll
            for (int t = 0; t < RR; t++) {
                if (t & h) continue;
                const int k = (t & (h - 1)) * M;
                if (M == 1 && k == 0) f.dit1(v[t], v[t + h]);
                else f.dit(v[t], v[t + h], twp[m + k]);
            }
        }
#pragma unroll
        for (int t = 0; t < RR; t++) p[Lay::off(t * M)] = v[t];
    }
}

template <class F, class Lay, int LOGL, int S0, int RL, int NT> struct DifGroups {
    __device__ __forceinline__ static void run(const F& f, typename F::T* s, const typename F::W* tw) {
        constexpr int r = (LOGL - S0) < RL ? (LOGL - S0) : RL;
        dif_group<F, Lay, LOGL, S0, r, NT>(f, s, tw);
        __syncthreads();
        DifGroups<F, Lay, LOGL, S0 + r, RL, NT>::run(f, s, tw);
    }
};
template <class F, class Lay, int LOGL, int RL, int NT> struct DifGroups<F, Lay, LOGL, LOGL, RL, NT> {
    __device__ __forceinline__ static void run(const F&, typename F::T*, const typename F::W*) {}
};

// DIT runs the small spans first; the first group takes the remainder so the
// later (larger-span, per-lane twiddle) groups are full radix.
template <class F, class Lay, int LOGL, int S0, int RL, int NT> struct DitGroups {
    __device__ __forceinline__ static void run(const F& f, typename F::T* s, const typename F::W* tw) {
        constexpr int rem = (LOGL - S0) % RL;
        constexpr int r = (S0 == 0 && rem != 0) ? rem : ((LOGL - S0) < RL ? (LOGL - S0) : RL);
        dit_group<F, Lay, LOGL, S0, r, NT>(f, s, tw);
        __syncthreads();
        DitGroups<F, Lay, LOGL, S0 + r, RL, NT>::run(f, s, tw);
    }
};
template <class F, class Lay, int LOGL, int RL, int NT> struct DitGroups<F, Lay, LOGL, LOGL, RL, NT> {
    __device__ __forceinline__ static void run(const F&, typename F::T*, const typename F::W*) {}
};

// Full forward / inverse transform of the tile (caller synchronises before).
template <class F, class Lay, int LOGL, int RL, int NT>
__device__ __forceinline__ void tile_dif(const F& f, typename F::T* s, const typename F::W* tw) {
    DifGroups<F, Lay, LOGL, 0, RL, NT>::run(f, s, tw);
}
template <class F, class Lay, int LOGL, int RL, int NT>
__device__ __forceinline__ void tile_dit(const F& f, typename F::T* s, const typename F::W* tw) {
    DitGroups<F, Lay, LOGL, 0, RL, NT>::run(f, s, tw);
}

}  // namespace mm
