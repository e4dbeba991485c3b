// ntt_core.cuh -- shared-memory tile transforms for sm_100a.
//
// A "tile" is C independent length-L transforms held in shared memory
// (transform c occupies a padded row of the tile).  Each CTA performs the
// butterfly stages in register groups of radix R = 2^r: a thread loads R
// elements of one transform, runs r butterfly levels in registers, and
// writes them back; groups are separated by __syncthreads().
//
//   forward  = decimation in frequency (Gentleman-Sande): natural in,
//              bit-mirrored out -- the TFT order TFT_w of P:893 with l = n;
//   inverse  = decimation in time (Cooley-Tukey): bit-mirrored in, natural
//              out, root w^-1 (inverse of Algorithm 1's TFFT).
//
// Twiddles come from a per-level table tw[m + i] = w_{2m}^i (0 <= i < m,
// m = 1, 2, ..., L/2), staged in shared memory; for 32-bit moduli each entry
// carries its fixed-multiplicand companion floor(w 2^32 / p).
#pragma once
#include "arith.cuh"

namespace mm {

// Padded shared-memory index: one pad word per 32 banks worth of elements.
template <class T> __device__ __forceinline__ int spad(int j);
template <> __device__ __forceinline__ int spad<uint32_t>(int j) { return j + (j >> 5); }
template <> __device__ __forceinline__ int spad<uint64_t>(int j) { return j + (j >> 4); }
template <class T> __host__ __device__ constexpr int spad_len(int L) {
    return sizeof(T) == 4 ? L + (L >> 5) : L + (L >> 4);
}

__device__ __forceinline__ int ilog2i(int x) { return 31 - __clz(x); }

// One DIF group: stages s0 .. s0+RL-1 of a length-L (= 2^k) transform,
// RL = log2(RR).  Chunks of RR elements: transform c, base b.
template <class F, int RR>
__device__ __forceinline__ void dif_group(const F& f, typename F::T* s, int srow, int C, int k, int s0,
                                          const typename F::W* tw) {
    typedef typename F::T T;
    constexpr int RL = RR == 1 ? 0 : (RR == 2 ? 1 : (RR == 4 ? 2 : (RR == 8 ? 3 : (RR == 16 ? 4 : 5))));
    const int L = 1 << k;
    const int lm = k - s0 - RL;           // log2 of the span of the last stage of the group
    const int m_last = 1 << lm;
    const int per = L / RR;
    const int chunks = C * per;
    for (int ch = threadIdx.x; ch < chunks; ch += blockDim.x) {
        int c = ch / per, b = ch - c * per;
        int lo = b & (m_last - 1), hi = b >> lm;
        int base = lo + (hi << (lm + RL));
        T* row = s + c * srow;
        T v[RR];
#pragma unroll
        for (int t = 0; t < RR; t++) v[t] = row[spad<T>(base + t * m_last)];
#pragma unroll
        for (int q = 0; q < RL; q++) {
            const int h = RR >> (q + 1);           // partner offset in t-space
            const int m = m_last * h;              // span of this stage
#pragma unroll
            for (int t = 0; t < RR; t++) {
                if (t & h) continue;
                int widx = m + lo + (t & (h - 1)) * m_last;
                f.dif(v[t], v[t + h], tw[widx]);
            }
        }
#pragma unroll
        for (int t = 0; t < RR; t++) row[spad<T>(base + t * m_last)] = v[t];
    }
}

// One DIT group: spans 2^s0 .. 2^(s0+RL-1).
template <class F, int RR>
__device__ __forceinline__ void dit_group(const F& f, typename F::T* s, int srow, int C, int k, int s0,
                                          const typename F::W* tw) {
    typedef typename F::T T;
    constexpr int RL = RR == 1 ? 0 : (RR == 2 ? 1 : (RR == 4 ? 2 : (RR == 8 ? 3 : (RR == 16 ? 4 : 5))));
    const int L = 1 << k;
    const int mf = 1 << s0;               // span of the first stage of the group
    const int per = L / RR;
    const int chunks = C * per;
    for (int ch = threadIdx.x; ch < chunks; ch += blockDim.x) {
        int c = ch / per, b = ch - c * per;
        int lo = b & (mf - 1), hi = b >> s0;
        int base = lo + (hi << (s0 + RL));
        T* row = s + c * srow;
        T v[RR];
#pragma unroll
        for (int t = 0; t < RR; t++) v[t] = row[spad<T>(base + t * mf)];
#pragma unroll
        for (int q = 0; q < RL; q++) {
            const int h = 1 << q;
            const int m = mf * h;
#pragma unroll
            for (int t = 0; t < RR; t++) {
                if (t & h) continue;
                int widx = m + lo + (t & (h - 1)) * mf;
                f.dit(v[t], v[t + h], tw[widx]);
            }
        }
#pragma unroll
        for (int t = 0; t < RR; t++) row[spad<T>(base + t * mf)] = v[t];
    }
}

// Full forward (DIF) transform of the C rows of a tile, radix-R groups.
// Caller must __syncthreads() before (data ready) ; this ends synchronised.
template <class F, int R>
__device__ __forceinline__ void tile_dif(const F& f, typename F::T* s, int srow, int C, int k,
                                         const typename F::W* tw) {
    constexpr int RL = R == 2 ? 1 : (R == 4 ? 2 : (R == 8 ? 3 : (R == 16 ? 4 : 5)));
    int s0 = 0;
    while (s0 < k) {
        int r = k - s0 < RL ? k - s0 : RL;
        switch (r) {
            case 1: dif_group<F, 2>(f, s, srow, C, k, s0, tw); break;
            case 2: dif_group<F, 4>(f, s, srow, C, k, s0, tw); break;
            case 3: if (RL >= 3) dif_group<F, (R >= 8 ? 8 : 2)>(f, s, srow, C, k, s0, tw); break;
            case 4: if (RL >= 4) dif_group<F, (R >= 16 ? 16 : 2)>(f, s, srow, C, k, s0, tw); break;
            default: if (RL >= 5) dif_group<F, (R >= 32 ? 32 : 2)>(f, s, srow, C, k, s0, tw); break;
        }
        s0 += r;
        __syncthreads();
    }
}

template <class F, int R>
__device__ __forceinline__ void tile_dit(const F& f, typename F::T* s, int srow, int C, int k,
                                         const typename F::W* tw) {
    constexpr int RL = R == 2 ? 1 : (R == 4 ? 2 : (R == 8 ? 3 : (R == 16 ? 4 : 5)));
    int s0 = 0;
    while (s0 < k) {
        int r = k - s0 < RL ? k - s0 : RL;
        switch (r) {
            case 1: dit_group<F, 2>(f, s, srow, C, k, s0, tw); break;
            case 2: dit_group<F, 4>(f, s, srow, C, k, s0, tw); break;
            case 3: if (RL >= 3) dit_group<F, (R >= 8 ? 8 : 2)>(f, s, srow, C, k, s0, tw); break;
            case 4: if (RL >= 4) dit_group<F, (R >= 16 ? 16 : 2)>(f, s, srow, C, k, s0, tw); break;
            default: if (RL >= 5) dit_group<F, (R >= 32 ? 32 : 2)>(f, s, srow, C, k, s0, tw); break;
        }
        s0 += r;
        __syncthreads();
    }
}

__device__ __forceinline__ int brev(int i, int k) { return k == 0 ? 0 : (int)(__brev((unsigned)i) >> (32 - k)); }

}  // namespace mm
