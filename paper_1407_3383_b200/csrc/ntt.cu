// ntt.cu -- batched NTT plans, forward / inverse transforms, the four-step
// passes of Algorithm 1, polynomial and integer products.
//
// Layout in HBM: `batch` rows of n = 2^k elements, row-major, contiguous.
//   k <= 12 : one pass; a CTA holds C whole rows in shared memory.
//   k  > 12 : Algorithm 1 with l = n, n = n2 x n1, a[j2 n1 + j1]:
//     column pass : column TFFTs (length n2, root w^n1, DIF -> rows in
//                   bit-mirrored order i2) + twiddle w^(j1 [i2]_k2)   (steps 1-2)
//     row pass    : row TFFTs (length n1, root w^n2, DIF)             (steps 3-4)
//   and the output position i2 n1 + i1 holds ahat_{[i2 n1 + i1]_k} (P:913,
//   Proposition 15), i.e. the TFT order with no transposition at all.
//   The inverse runs the steps backwards with w^-1.
#include "common.h"
#include <cuda.h>
#include "ntt_kernels.cuh"
#include "fast32.h"
#include "tft.h"
#include "jobs.h"
#include <new>
#include <string.h>
#include <type_traits>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

namespace mm {

// ---------------------------------------------------------------- bit-mirror permutation
template <class T>
__global__ void k_bitrev_perm(const T* __restrict__ in, T* __restrict__ out, int k, long long batch) {
    const long long n = 1ll << k;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n * batch;
         i += (long long)gridDim.x * blockDim.x) {
        long long b = i >> k, j = i & (n - 1);
        unsigned long long rj = __brevll((unsigned long long)j) >> (64 - k);
        out[i] = in[b * n + (long long)rj];
    }
}

// Tiled form for k >= 10.  Write j = (a : 5 bits | m : k - 10 bits | b : 5 bits);
// its mirror is ([b] | [m] | [a]).  A tile is the 32 x 32 pairs (a, b) of one m:
// it is read as 32 runs of 32 consecutive elements (run a at (a | m | 0)) and
// written as 32 runs of 32 consecutive elements (run [b] at ([b] | [m] | 0)),
// transposed through shared memory, so both sides move whole 128- / 256-byte
// lines (the element-wise form reads one element per sector).
template <class T>
__global__ void __launch_bounds__(256) k_bitrev_tiled(const T* __restrict__ in, T* __restrict__ out, int k, long long batch) {
    __shared__ T tile[32][33];
    const int km = k - 10;
    const long long ntiles = batch << km;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int rtx = (int)(__brev((unsigned)tx) >> 27);
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long long b = t >> km;
        const unsigned m = (unsigned)(t & ((1ll << km) - 1));
        const unsigned rm = km ? __brev(m) >> (32 - km) : 0u;
        const T* src = in + (b << k) + ((long long)m << 5) + tx;
        T* dst = out + (b << k) + ((long long)rm << 5) + tx;
#pragma unroll
        for (int a = ty; a < 32; a += 8) tile[a][tx] = src[(long long)a << (k - 5)];
        __syncthreads();
        // out[(rb | rm | ra)] = in[([ra] | m | [rb])] = tile[[ra]][[rb]], ra = tx
#pragma unroll
        for (int rb = ty; rb < 32; rb += 8) dst[(long long)rb << (k - 5)] = tile[rtx][__brev((unsigned)rb) >> 27];
        __syncthreads();
    }
}

// ---------------------------------------------------------------- twiddle tables (device)
__device__ __forceinline__ uint32_t dmulmod32(uint32_t a, uint32_t b, uint32_t p) {
    return (uint32_t)(((uint64_t)a * b) % p);
}
__device__ uint32_t dpow32(uint32_t b, uint64_t e, uint32_t p) {
    uint32_t r = 1;
    while (e) {
        if (e & 1) r = dmulmod32(r, b, p);
        b = dmulmod32(b, b, p);
        e >>= 1;
    }
    return r;
}
__device__ uint64_t dpowG(uint64_t b, uint64_t e) {
    uint64_t r = 1;
    while (e) {
        if (e & 1) r = FpG::mul(r, b);
        b = FpG::mul(b, b);
        e >>= 1;
    }
    return FpG::canon(r);
}
__device__ __forceinline__ void tw_set(uint2* t, long long i, uint32_t w, uint32_t p) {
    t[i] = make_uint2(w, (uint32_t)(((uint64_t)w << 32) / p));   // (w, psi)
}
__device__ __forceinline__ void tw_set(uint64_t* t, long long i, uint64_t w, uint64_t) { t[i] = w; }
// FP64 plans (word_bits 52): exponents in exact integer arithmetic mod p < 2^50,
// tables hold the residues as doubles
struct D50 {
    uint64_t v;
    __host__ __device__ D50(uint64_t x = 0) : v(x) {}
};
__device__ __forceinline__ uint64_t dmulmod50(uint64_t a, uint64_t b, uint64_t p) {
    return (uint64_t)(((unsigned __int128)a * b) % p);
}
__device__ __forceinline__ void tw_set(double* t, long long i, D50 w, uint64_t) { t[i] = (double)w.v; }
__device__ D50 tw_pow(D50 w, uint64_t e, uint64_t p) {
    uint64_t r = 1, b = w.v % p;
    while (e) {
        if (e & 1) r = dmulmod50(r, b, p);
        b = dmulmod50(b, b, p);
        e >>= 1;
    }
    return D50(r);
}
__device__ __forceinline__ uint64_t tw_pow(uint32_t w, uint64_t e, uint64_t p) { return dpow32(w, e, (uint32_t)p); }
__device__ __forceinline__ uint64_t tw_pow(uint64_t w, uint64_t e, uint64_t) { return dpowG(w, e); }

// level table for a length-L transform with root w_L: tw[m + i] = w_L^(i L / 2m)
template <class W, class E>
__global__ void k_level_table(W* tw, int k, E w, uint64_t p) {
    const long long L = 1ll << k;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < L;
         idx += (long long)gridDim.x * blockDim.x) {
        if (idx == 0) { tw_set(tw, 0, (E)1, p); continue; }
        int lm = 63 - __clzll(idx);
        long long m = 1ll << lm, i = idx - m;
        uint64_t e = (uint64_t)i << (k - 1 - lm);
        tw_set(tw, idx, (E)tw_pow(w, e, p), p);
    }
}
// power table: t[i] = w^(i * step) for i < cnt
template <class W, class E>
__global__ void k_pow_table(W* t, long long cnt, E w, uint64_t step, uint64_t p) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x)
        tw_set(t, i, (E)tw_pow(w, (uint64_t)i * step, p), p);
}

// full step-2 table: t[i2 n1 + j1] = w^(j1 [i2]_k2)
template <class W, class E>
__global__ void k_fs_table(W* t, int k1, int k2, E w, uint64_t p) {
    const long long cnt = 1ll << (k1 + k2);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
        long long i2 = i >> k1, j1 = i & ((1ll << k1) - 1);
        uint64_t e = (uint64_t)j1 * (uint64_t)brev((int)i2, k2);
        tw_set(t, i, (E)tw_pow(w, e, p), p);
    }
}

// scaled step-2 table for the 32-bit fused product: t[i2 n1 + j1] = w^(j1 [i2]_k2) s mod p
__global__ void k_fs_table_scaled32(uint2* t, int k1, int k2, uint32_t w, uint32_t s, uint32_t p) {
    const long long cnt = 1ll << (k1 + k2);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
        long long i2 = i >> k1, j1 = i & ((1ll << k1) - 1);
        uint64_t e = (uint64_t)j1 * (uint64_t)brev((int)i2, k2);
        tw_set(t, i, dmulmod32(dpow32(w, e, p), s, p), p);
    }
}

// ---------------------------------------------------------------- carries (int_mul)
// The product coefficients c_k (exact integers) are evaluated at 2^W (P:973,
// "A(2^h) = a") digit by digit: s_j = sum_t digit_t(c_{j-t}) (T digits of W
// bits per coefficient); u_j = (s_j mod 2^W) + (s_{j-1} >> W) < 2^W + T;
// w_j = u_j mod 2^W, g_j = u_j >> W in {0,1}; carry chain
// C_{j+1} = g_j | (w_j == 2^W - 1 & C_j); out_j = (w_j + C_j) mod 2^W.
// Dig16: Goldilocks path, c_k < 2^56 in a u64, 16-bit limbs (T = 4).
// Dig32x3: three-prime path, c_k < 2^86 as three 32-bit words, 32-bit limbs (T = 3).
struct Dig16 {
    typedef uint16_t Out;
    enum { W = 16 };
    const uint64_t* c;
    long long nc;
    __device__ __forceinline__ uint64_t s_at(long long j) const {
        uint64_t s = 0;
#pragma unroll
        for (int t = 0; t < 4; t++) {
            long long k = j - t;
            if (k >= 0 && k < nc) s += (c[k] >> (16 * t)) & 0xFFFF;
        }
        return s;
    }
};
struct Dig32x3 {
    typedef uint32_t Out;
    enum { W = 32 };
    const uint32_t* w;   // coefficient k at w[3k], w[3k+1], w[3k+2] (little-endian words)
    long long nc;
    __device__ __forceinline__ uint64_t s_at(long long j) const {
        uint64_t s = 0;
#pragma unroll
        for (int t = 0; t < 3; t++) {
            long long k = j - t;
            if (k >= 0 && k < nc) s += w[3 * k + t];
        }
        return s;
    }
};
// many independent products back to back: entry e owns limbs [e nout, (e+1) nout)
// and coefficients w[3 (e nc + k) ..], k < nc; digit sums never cross entries
// (each entry's value fits its nout limbs, so its carry out is 0).
struct Dig32x3Batch {
    typedef uint32_t Out;
    enum { W = 32 };
    const uint32_t* w;
    long long nc, nout;
    __device__ __forceinline__ uint64_t s_at(long long j) const {
        const long long e = j / nout, jl = j - e * nout;
        const uint32_t* we = w + 3 * e * nc;
        uint64_t s = 0;
#pragma unroll
        for (int t = 0; t < 3; t++) {
            long long k = jl - t;
            if (k >= 0 && k < nc) s += we[3 * k + t];
        }
        return s;
    }
};
template <class D>
__device__ __forceinline__ void carry_gp(const D& d, long long j, uint32_t& w, uint32_t& g) {
    constexpr uint64_t M = (D::W == 32) ? 0xFFFFFFFFull : ((1ull << D::W) - 1);
    const uint64_t sj = d.s_at(j);
    const uint64_t sp = j > 0 ? d.s_at(j - 1) : 0;
    const uint64_t u = (sj & M) + (sp >> D::W);
    w = (uint32_t)(u & M);
    g = (uint32_t)(u >> D::W);
}
template <class D> __device__ __forceinline__ bool all_ones(uint32_t w) {
    return D::W == 32 ? w == 0xFFFFFFFFu : w == ((1u << D::W) - 1);
}
// (G,P) composition: applying segment lo then hi: G = Ghi | (Phi & Glo), P = Phi & Plo
constexpr int CARRY_T = 256, CARRY_E = 16, CARRY_B = CARRY_T * CARRY_E;

__device__ __forceinline__ uint32_t gp_comb(uint32_t lo, uint32_t hi) {   // bit0 = G, bit1 = P
    uint32_t G = (hi & 1) | ((hi >> 1) & lo & 1);
    uint32_t P = (hi >> 1) & (lo >> 1) & 1;
    return G | (P << 1);
}

// block-exclusive scan of (G,P) over threads; returns the thread's carry-in
// relative to the block start (assuming block carry-in = cin).
__device__ uint32_t block_carry_in(uint32_t mine, uint32_t cin, uint32_t* sh) {
    // inclusive warp scan
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = gp_comb(y, x);
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 2u;   // identity: G=0,P=1
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v = gp_comb(y, v);
        }
        sh[32 + lane] = v;   // inclusive over warps
    }
    __syncthreads();
    uint32_t excl_w = wid > 0 ? sh[32 + wid - 1] : 2u;
    uint32_t excl_l = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) excl_l = 2u;
    uint32_t pre = gp_comb(excl_w, excl_l);      // exclusive prefix within block
    uint32_t res = (pre & 1) | ((pre >> 1) & cin);
    __syncthreads();
    return res;
}

template <class D>
__global__ void __launch_bounds__(CARRY_T) k_carry_reduce(D d, long long nout, uint32_t* __restrict__ agg) {
    __shared__ uint32_t sh[64];
    long long j0 = (long long)blockIdx.x * CARRY_B + (long long)threadIdx.x * CARRY_E;
    uint32_t acc = 2u;   // identity
    for (int e = 0; e < CARRY_E; e++) {
        long long j = j0 + e;
        uint32_t gp = 2u;
        if (j < nout) {
            uint32_t w, g;
            carry_gp(d, j, w, g);
            gp = g | ((all_ones<D>(w) ? 1u : 0u) << 1);
        }
        acc = gp_comb(acc, gp);
    }
    // reduce over the block (inclusive scan, take the last)
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = acc;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = gp_comb(y, x);
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t v = 2u;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) v = gp_comb(v, sh[w]);
        agg[blockIdx.x] = v;
    }
}

// scan of block aggregates -> carry-in per block.  Up to 16 aggregates per
// thread: each thread combines its run of E consecutive ones, one block scan
// gives the carry into every run, and the run is walked again (one pass of
// barriers instead of one per 1024 aggregates); longer inputs go in chunks.
__global__ void k_carry_scan(uint32_t* agg, long long nblk) {
    __shared__ uint32_t sh[64];
    __shared__ uint32_t carry;
    if (nblk <= 16ll * blockDim.x) {
        const int E = (int)((nblk + blockDim.x - 1) / blockDim.x);
        const long long i0 = (long long)threadIdx.x * E;
        uint32_t v[16];
#pragma unroll
        for (int e = 0; e < 16; e++) v[e] = (e < E && i0 + e < nblk) ? agg[i0 + e] : 2u;   // all loads in flight
        uint32_t loc = 2u;                                   // identity: G = 0, P = 1
#pragma unroll
        for (int e = 0; e < 16; e++) loc = gp_comb(loc, v[e]);
        uint32_t c = block_carry_in(loc, 0u, sh);            // carry into this run
#pragma unroll
        for (int e = 0; e < 16; e++) {
            if (e < E && i0 + e < nblk) agg[i0 + e] = c;
            c = (v[e] & 1) | ((v[e] >> 1) & c);
        }
        return;
    }
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < nblk; base += blockDim.x) {
        long long i = base + threadIdx.x;
        uint32_t mine = i < nblk ? agg[i] : 2u;
        uint32_t cin = block_carry_in(mine, carry, sh);
        __syncthreads();
        if (i < nblk) agg[i] = cin;     // carry into block i
        // carry out of this chunk = carry-in of last + its own
        if (threadIdx.x == blockDim.x - 1) carry = (mine & 1) | ((mine >> 1) & cin);
        __syncthreads();
    }
}

template <class D>
__global__ void __launch_bounds__(CARRY_T) k_carry_apply(D d, long long nout, const uint32_t* __restrict__ cin_blk,
                                                         typename D::Out* __restrict__ out) {
    __shared__ uint32_t sh[64];
    long long j0 = (long long)blockIdx.x * CARRY_B + (long long)threadIdx.x * CARRY_E;
    uint32_t w[CARRY_E], g[CARRY_E];
    uint32_t acc = 2u;
#pragma unroll
    for (int e = 0; e < CARRY_E; e++) {
        long long j = j0 + e;
        w[e] = 0; g[e] = 0;
        uint32_t gp = 2u;
        if (j < nout) {
            carry_gp(d, j, w[e], g[e]);
            gp = g[e] | ((all_ones<D>(w[e]) ? 1u : 0u) << 1);
        }
        acc = gp_comb(acc, gp);
    }
    uint32_t C = block_carry_in(acc, cin_blk[blockIdx.x], sh);
#pragma unroll
    for (int e = 0; e < CARRY_E; e++) {
        long long j = j0 + e;
        if (j < nout) out[j] = (typename D::Out)(w[e] + C);    // mod 2^W by the cast
        C = g[e] | ((all_ones<D>(w[e]) ? 1u : 0u) & C);
    }
}

// Dig16 fast path: a CTA stages the coefficients [jb - 4, jb + CARRY_B) of its
// limb block in shared memory once (coalesced, one pad word per 16 so the
// 16-apart thread windows do not collide), then every thread forms its 16 digit
// sums from a 20-coefficient register window (the generic path reloads 8
// coefficients per limb from global memory).
constexpr int C16_SM = CARRY_B + 4 + (CARRY_B + 4) / 16 + 1;
__device__ __forceinline__ int c16_pad(int r) { return r + (r >> 4); }
// Coefficient pairs (16-byte loads when the window is aligned), all of a
// thread's loads in flight before its shared stores (the one-load-at-a-time
// loop left the carry pass latency-bound).
__device__ __forceinline__ void c16_stage(uint64_t* sc, const uint64_t* __restrict__ c, long long nc, long long jb) {
    constexpr int NP = (CARRY_B + 4) / 2, U = (NP + CARRY_T - 1) / CARRY_T;
    static_assert((CARRY_B + 4) % 2 == 0, "pairs");
    const long long k0 = jb - 4;
    const bool vec = (((uintptr_t)(c + k0)) & 15) == 0 && k0 >= 0 && k0 + 2 * NP <= nc;
    ulonglong2 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int pr = threadIdx.x + u * CARRY_T;
        if (pr < NP) {
            if (vec) {
                v[u] = __ldg((const ulonglong2*)(c + k0) + pr);
            } else {
                const long long k = k0 + 2 * pr;
                v[u].x = (k >= 0 && k < nc) ? __ldg(c + k) : 0ull;
                v[u].y = (k + 1 >= 0 && k + 1 < nc) ? __ldg(c + k + 1) : 0ull;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int pr = threadIdx.x + u * CARRY_T;
        if (pr < NP) {
            sc[c16_pad(2 * pr)] = v[u].x;
            sc[c16_pad(2 * pr + 1)] = v[u].y;
        }
    }
}
// w[e], g[e] for limbs j = jb + 16 t + e (see the Dig16 comment above)
__device__ __forceinline__ void c16_wg(const uint64_t* sc, uint32_t* w, uint32_t* g) {
    uint64_t cc[20];
#pragma unroll
    for (int u = 0; u < 20; u++) cc[u] = sc[c16_pad(16 * threadIdx.x + u)];
    uint32_t S[17];
#pragma unroll
    for (int q = 0; q < 17; q++) {
        uint32_t t = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) t += (uint32_t)(cc[q + 3 - u] >> (16 * u)) & 0xFFFFu;
        S[q] = t;
    }
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const uint32_t v = (S[e + 1] & 0xFFFFu) + (S[e] >> 16);
        w[e] = v & 0xFFFFu;
        g[e] = v >> 16;
    }
}
__global__ void __launch_bounds__(CARRY_T) k_carry16_reduce(const uint64_t* __restrict__ c, long long nc, long long nout,
                                                            uint32_t* __restrict__ agg) {
    __shared__ uint64_t sc[C16_SM];
    __shared__ uint32_t sh[64];
    const long long jb = (long long)blockIdx.x * CARRY_B;
    c16_stage(sc, c, nc, jb);
    __syncthreads();
    uint32_t w[16], g[16];
    c16_wg(sc, w, g);
    uint32_t acc = 2u;
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const long long j = jb + 16 * threadIdx.x + e;
        acc = gp_comb(acc, j < nout ? (g[e] | ((w[e] == 0xFFFFu ? 1u : 0u) << 1)) : 2u);
    }
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = acc;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = gp_comb(y, x);
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t v = 2u;
        for (int q = 0; q < (int)(blockDim.x >> 5); q++) v = gp_comb(v, sh[q]);
        agg[blockIdx.x] = v;
    }
}
__global__ void __launch_bounds__(CARRY_T) k_carry16_apply(const uint64_t* __restrict__ c, long long nc, long long nout,
                                                           const uint32_t* __restrict__ cin_blk, uint16_t* __restrict__ out) {
    __shared__ uint64_t sc[C16_SM];
    __shared__ uint32_t sh[64];
    const long long jb = (long long)blockIdx.x * CARRY_B;
    c16_stage(sc, c, nc, jb);
    __syncthreads();
    uint32_t w[16], g[16];
    c16_wg(sc, w, g);
    uint32_t acc = 2u;
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const long long j = jb + 16 * threadIdx.x + e;
        acc = gp_comb(acc, j < nout ? (g[e] | ((w[e] == 0xFFFFu ? 1u : 0u) << 1)) : 2u);
    }
    uint32_t C = block_carry_in(acc, cin_blk[blockIdx.x], sh);
    const long long j0 = jb + 16 * threadIdx.x;
    uint32_t o[8];
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const uint32_t limb = (w[e] + C) & 0xFFFFu;
        C = g[e] | ((w[e] == 0xFFFFu ? 1u : 0u) & C);
        if (e & 1) o[e >> 1] |= limb << 16; else o[e >> 1] = limb;
    }
    if (j0 + 16 <= nout && ((((uintptr_t)(out + j0)) & 15) == 0)) {   // two 16-byte stores
        uint4* d = (uint4*)(out + j0);
        d[0] = make_uint4(o[0], o[1], o[2], o[3]);
        d[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
        for (int e = 0; e < 16; e++)
            if (j0 + e < nout) out[j0 + e] = (uint16_t)(o[e >> 1] >> (16 * (e & 1)));
    }
}

// Single-pass carries (decoupled look-back): a CTA takes the next block index
// from a ticket (so every predecessor is already running), publishes its
// (G, P) aggregate, walks back over its predecessors' published words until an
// inclusive prefix, publishes its own inclusive prefix and applies its carry-in
// -- the coefficients are read once instead of twice.  status[b] = flag << 32 |
// (G, P), flag 1 = aggregate, 2 = inclusive prefix; one 64-bit word so flag and
// value travel together (release / acquire at gpu scope).
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__global__ void __launch_bounds__(CARRY_T) k_carry16_fused(const uint64_t* __restrict__ c, long long nc, long long nout,
                                                           unsigned long long* status, unsigned* ticket,
                                                           uint16_t* __restrict__ out) {
    __shared__ uint64_t sc[C16_SM];
    __shared__ uint32_t sh[64];
    __shared__ uint32_t s_bid, s_cin;
    if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
    __syncthreads();
    const long long bid = s_bid;
    const long long jb = bid * CARRY_B;
    c16_stage(sc, c, nc, jb);
    __syncthreads();
    uint32_t w[16], g[16];
    c16_wg(sc, w, g);
    uint32_t acc = 2u;
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const long long j = jb + 16 * threadIdx.x + e;
        acc = gp_comb(acc, j < nout ? (g[e] | ((w[e] == 0xFFFFu ? 1u : 0u) << 1)) : 2u);
    }
    uint32_t C;
    {   // block aggregate; every thread's exclusive prefix within the block is
        // formed while warp 0 looks back (two barriers instead of four)
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        uint32_t x = acc;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = gp_comb(y, x);
        }
        if (lane == 31) sh[wid] = x;
        __syncthreads();
        uint32_t wpre = 2u;                                  // identity: G = 0, P = 1
        for (int q = 0; q < wid; q++) wpre = gp_comb(wpre, sh[q]);
        uint32_t excl_l = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) excl_l = 2u;
        const uint32_t pre = gp_comb(wpre, excl_l);
        if (wid == 0) {
            // warp 0: publish the aggregate, then look back 32 predecessors at a
            // time (lane l reads block k - l) until an inclusive prefix appears
            uint32_t agg = 2u;
            for (int q = 0; q < (int)(blockDim.x >> 5); q++) agg = gp_comb(agg, sh[q]);
            if (bid == 0) {
                if (lane == 0) {
                    st_release64(status, (2ull << 32) | agg);
                    s_cin = 0;
                }
            } else {
                if (lane == 0) st_release64(status + bid, (1ull << 32) | agg);
                uint32_t run = 2u;                         // identity: G = 0, P = 1
                for (long long k = bid - 1;; k -= 32) {
                    const long long kk = k - lane;
                    unsigned long long v = (2ull << 32) | 2u;   // before block 0: identity, inclusive
                    if (kk >= 0)
                        do { v = ld_acquire64(status + kk); } while ((v >> 32) == 0);
                    const unsigned inc = __ballot_sync(0xffffffffu, (v >> 32) == 2);
                    const int stop = inc ? __ffs(inc) - 1 : 31;    // nearest inclusive prefix
                    uint32_t x2 = lane <= stop ? (uint32_t)v : 2u;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {          // far (higher lane) before near
                        const uint32_t y = __shfl_down_sync(0xffffffffu, x2, o);
                        if (lane + o < 32) x2 = gp_comb(y, x2);
                    }
                    run = gp_comb(__shfl_sync(0xffffffffu, x2, 0), run);
                    if (inc) break;
                }
                if (lane == 0) {
                    st_release64(status + bid, (2ull << 32) | gp_comb(run, agg));
                    s_cin = run & 1u;                      // carry into the block (G of the prefix)
                }
            }
        }
        __syncthreads();
        C = (pre & 1) | ((pre >> 1) & s_cin);             // carry into this thread's first limb
    }
    const long long j0 = jb + 16 * threadIdx.x;
    uint32_t o[8];
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const uint32_t limb = (w[e] + C) & 0xFFFFu;
        C = g[e] | ((w[e] == 0xFFFFu ? 1u : 0u) & C);
        if (e & 1) o[e >> 1] |= limb << 16; else o[e >> 1] = limb;
    }
    if (j0 + 16 <= nout && ((((uintptr_t)(out + j0)) & 15) == 0)) {
        uint4* d = (uint4*)(out + j0);
        d[0] = make_uint4(o[0], o[1], o[2], o[3]);
        d[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
        for (int e = 0; e < 16; e++)
            if (j0 + e < nout) out[j0 + e] = (uint16_t)(o[e >> 1] >> (16 * (e & 1)));
    }
}

// ---------------------------------------------------------------- carries over column blocks (sharded int_mul)
// A rank of the sharded product holds coefficients c_j, j = r n1 + col0 + i
// (row r < nrows, i < c1): one chunk of c1 consecutive j per row.  The digit
// sums at the start of a chunk need the 4 coefficients before it (halo):
// halo[r] = the last 4 coefficients of the preceding chunk, i.e. of the same
// row on the previous rank, or -- on rank 0 (shift) -- of row r - 1 on the last
// rank.  Coefficients with global index outside [0, nc) are zero.
struct ChunkRef {
    const uint64_t* coef;
    const uint64_t* halo;
    long long c1, n1, col0, nc, nout;
    int shift;
    __device__ __forceinline__ uint64_t cf(long long r, long long i) const {
        if (i >= 0) return coef[r * c1 + i];
        const long long hr = shift ? r - 1 : r;
        return hr >= 0 ? halo[hr * 4 + 4 + i] : 0;
    }
    __device__ __forceinline__ uint64_t s_at(long long r, long long i) const {
        const long long jg = r * n1 + col0 + i;
        uint64_t s = 0;
#pragma unroll
        for (int t = 0; t < 4; t++)
            if (jg - t >= 0 && jg - t < nc) s += (cf(r, i - t) >> (16 * t)) & 0xFFFF;
        return s;
    }
    __device__ __forceinline__ void gp(long long r, long long i, uint32_t& w, uint32_t& g) const {
        const uint64_t sj = s_at(r, i);
        const uint64_t sp = (r * n1 + col0 + i > 0) ? s_at(r, i - 1) : 0;
        const uint64_t u = (sj & 0xFFFF) + (sp >> 16);
        w = (uint32_t)(u & 0xFFFF);
        g = (uint32_t)(u >> 16);
    }
};
__global__ void k_chunk_halo(const uint64_t* __restrict__ coef, long long nrows, long long c1, uint64_t* __restrict__ halo) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nrows * 4; i += (long long)gridDim.x * blockDim.x)
        halo[i] = coef[(i >> 2) * c1 + c1 - 4 + (i & 3)];
}
// one CTA per chunk: (G, P) aggregate of its digits (identity beyond nout)
__global__ void __launch_bounds__(256) k_chunk_reduce(ChunkRef R, uint32_t* __restrict__ agg) {
    __shared__ uint32_t sh[64];
    const long long r = blockIdx.x;
    const int E = (int)((R.c1 + blockDim.x - 1) / blockDim.x);
    uint32_t acc = 2u;
    for (int e = 0; e < E; e++) {
        const long long i = (long long)threadIdx.x * E + e;
        uint32_t gpv = 2u;
        if (i < R.c1 && r * R.n1 + R.col0 + i < R.nout) {
            uint32_t w, g;
            R.gp(r, i, w, g);
            gpv = g | ((w == 0xFFFF ? 1u : 0u) << 1);
        }
        acc = gp_comb(acc, gpv);
    }
    // block reduction of the (G, P) pairs in thread order
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = acc;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = gp_comb(y, x);
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t v = 2u;
        for (int q = 0; q < (int)(blockDim.x >> 5); q++) v = gp_comb(v, sh[q]);
        agg[r] = v;
    }
}
// sequential scan of chunk aggregates in natural chunk order q = r G + g, stored at
// agg[g nrows + r] (the all-gathered layout); replaced by the carry into each chunk
__global__ void k_chunk_scan(uint32_t* agg, long long G, long long nrows) {
    __shared__ uint32_t sh[64];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const long long nq = G * nrows;
    for (long long base = 0; base < nq; base += blockDim.x) {
        const long long q = base + threadIdx.x;
        const long long at = q < nq ? (q % G) * nrows + q / G : 0;
        const uint32_t mine = q < nq ? agg[at] : 2u;
        const uint32_t cin = block_carry_in(mine, carry, sh);
        __syncthreads();
        if (q < nq) agg[at] = cin;
        if (threadIdx.x == blockDim.x - 1) carry = (mine & 1) | ((mine >> 1) & cin);
        __syncthreads();
    }
}
__global__ void __launch_bounds__(256) k_chunk_apply(ChunkRef R, const uint32_t* __restrict__ cin_chunk,
                                                     uint16_t* __restrict__ out) {
    __shared__ uint32_t sh[64];
    const long long r = blockIdx.x;
    const int E = (int)((R.c1 + blockDim.x - 1) / blockDim.x);
    uint32_t acc = 2u;
    for (int e = 0; e < E; e++) {
        const long long i = (long long)threadIdx.x * E + e;
        uint32_t gpv = 2u;
        if (i < R.c1 && r * R.n1 + R.col0 + i < R.nout) {
            uint32_t w, g;
            R.gp(r, i, w, g);
            gpv = g | ((w == 0xFFFF ? 1u : 0u) << 1);
        }
        acc = gp_comb(acc, gpv);
    }
    uint32_t C = block_carry_in(acc, cin_chunk[r], sh);
    for (int e = 0; e < E; e++) {
        const long long i = (long long)threadIdx.x * E + e;
        if (i >= R.c1) break;
        uint32_t w = 0, g = 0;
        const bool live = r * R.n1 + R.col0 + i < R.nout;
        if (live) R.gp(r, i, w, g);
        out[r * R.c1 + i] = live ? (uint16_t)(w + C) : (uint16_t)0;
        C = g | ((w == 0xFFFF ? 1u : 0u) & C);
    }
}

// ---------------------------------------------------------------- polynomial matrix product
// At every evaluation point f < L: Chat_f = Ahat_f Bhat_f, an (m x kk) (kk x n)
// product over Z/pZ.  A CTA owns FB consecutive points and stages the
// matching slices of Ahat [m kk][L] and Bhat [kk n][L] in shared memory as
// [f][row][col]; each output sums kk products of residues exactly (64-bit
// accumulators, high words folded every 16 terms), reduced once.
// 4 x 4 register blocks: a thread owns C[i0..i0+3][j0..j0+3] at one point and
// loads 4 + 4 shared values per 16 products.
// 4-byte global -> shared copy that does not block the issuing thread (LDGSTS):
// the staging loops issue all their loads back to back
__device__ __forceinline__ void cp_async4s(uint32_t* dst, const uint32_t* src) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
// v mod p for any v < 2^64 by Barrett with mu = floor(2^64 / p): q = hi(v mu)
// underestimates floor(v / p) by at most 2 (p < 2^31)
__device__ __forceinline__ uint32_t mod64_barrett(uint64_t v, uint32_t p, uint64_t mu) {
    const uint64_t q = __umul64hi(v, mu);
    uint64_t r = v - q * p;
    r = r >= p ? r - p : r;
    r = r >= p ? r - p : r;
    return (uint32_t)r;
}
// (hi 2^32 + lo) mod p, hi < 2^64, lo < 2^32
__device__ __forceinline__ uint32_t mod96_barrett(uint64_t hi, uint64_t lo, uint32_t p, uint64_t mu) {
    const uint64_t t = mod64_barrett(hi, p, mu);
    return mod64_barrett((t << 32) | lo, p, mu);
}
__global__ void __launch_bounds__(256) k_point_matmul_any(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                                                      uint32_t* __restrict__ C, int m, int kk, int n, long long L,
                                                      int FB, uint32_t p, uint64_t r64) {
    extern __shared__ uint32_t sm[];
    const int sa = m * kk, sb = kk * n;
    uint32_t* SA = sm;                        // [FB][m][kk]
    uint32_t* SB = sm + (size_t)FB * sa;      // [FB][kk][n]
    const int mb = (m + 3) >> 2, nb = (n + 3) >> 2;
    for (long long f0 = (long long)blockIdx.x * FB; f0 < L; f0 += (long long)gridDim.x * FB) {
        const int nf = (int)(L - f0 < FB ? L - f0 : FB);
        __syncthreads();
        for (int e = threadIdx.x; e < nf * sa; e += blockDim.x) {
            const int f = e % nf, rc = e / nf;          // consecutive threads: consecutive points
            cp_async4s(SA + f * sa + rc, A + (long long)rc * L + f0 + f);
        }
        for (int e = threadIdx.x; e < nf * sb; e += blockDim.x) {
            const int f = e % nf, rc = e / nf;
            cp_async4s(SB + f * sb + rc, B + (long long)rc * L + f0 + f);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        const int nblk = nf * mb * nb;
        for (int o = threadIdx.x; o < nblk; o += blockDim.x) {
            const int jb = o % nb, ib = (o / nb) % mb, f = o / (mb * nb);
            const int i0 = ib * 4, j0 = jb * 4;
            const uint32_t* a = SA + f * sa;
            const uint32_t* bb = SB + f * sb;
            // products < 2^60 (residues < p < 2^30): 16 of them fit a u64 on top of a
            // value < 2^32, so every 16 terms the high word moves to hi (IMAD.WIDE.U32
            // accumulates in 64 bits in one instruction)
            uint64_t acc[4][4], hi[4][4];
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int v = 0; v < 4; v++) { acc[u][v] = 0; hi[u][v] = 0; }
            const uint32_t* ar[4];
            bool rv[4], cv[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                rv[u] = i0 + u < m;
                cv[u] = j0 + u < n;
                ar[u] = a + (rv[u] ? i0 + u : 0) * kk;
            }
            const int jc = j0 + 3 < n ? j0 : 0;
            for (int l0 = 0; l0 < kk; l0 += 16) {
                const int le = kk - l0 < 16 ? kk - l0 : 16;
                for (int l = l0; l < l0 + le; l++) {
                    uint32_t x[4], y[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) x[u] = rv[u] ? ar[u][l] : 0u;
                    if (j0 + 3 < n) {
#pragma unroll
                        for (int v = 0; v < 4; v++) y[v] = bb[l * n + jc + v];
                    } else {
#pragma unroll
                        for (int v = 0; v < 4; v++) y[v] = cv[v] ? bb[l * n + j0 + v] : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++)
#pragma unroll
                        for (int v = 0; v < 4; v++) acc[u][v] += (uint64_t)x[u] * y[v];
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        hi[u][v] += acc[u][v] >> 32;
                        acc[u][v] &= 0xFFFFFFFFull;
                    }
            }
            const uint64_t r32 = (uint64_t)(((uint64_t)1 << 32) % p);
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int v = 0; v < 4; v++)
                    if (rv[u] && cv[v])
                        C[(long long)((i0 + u) * n + j0 + v) * L + f0 + f] =
                            (uint32_t)(((hi[u][v] % p) * r32 + acc[u][v]) % p);
        }
    }
}

// [R][Cn] -> [Cn][R] u32 transpose through 32 x 33 shared tiles (coalesced both
// ways).  With rm > 0 the R input rows are an rm x rk matrix (row i rk + l) and
// land at output column l rm + i (its transpose), else at column r.
__global__ void __launch_bounds__(256) k_transpose32(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                     long long R, long long Cn, int rm = 0, int rk = 1) {
    __shared__ uint32_t t[32][33];
    const long long tiles_c = (Cn + 31) / 32, tiles = ((R + 31) / 32) * tiles_c;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (long long b = blockIdx.x; b < tiles; b += gridDim.x) {
        const long long r0 = (b / tiles_c) * 32, c0 = (b % tiles_c) * 32;
        for (int y = ty; y < 32; y += 8)
            if (r0 + y < R && c0 + tx < Cn) t[y][tx] = in[(r0 + y) * Cn + c0 + tx];
        __syncthreads();
        long long oc = r0 + tx;
        if (rm > 0 && oc < R) {
            const long long i = oc / rk, l = oc - i * rk;
            oc = l * rm + i;
        }
        for (int y = ty; y < 32; y += 8)
            if (c0 + y < Cn && r0 + tx < R) out[(c0 + y) * R + oc] = t[tx][y];
        __syncthreads();
    }
}
// point-major operands: A_f = At[f][m kk], B_f = Bt[f][kk n]; a CTA copies the
// slices of FB consecutive points contiguously (16-byte loads), each thread
// owns 4 x 4 output blocks: per term 4 broadcast words of A and one 16-byte
// load of B (m, n multiples of 4); output Ct[f][m n].
__global__ void __launch_bounds__(256, 2) k_point_matmul_pm(const uint32_t* __restrict__ At,
                                                            const uint32_t* __restrict__ Bt, uint32_t* __restrict__ Ct,
                                                            int m, int kk, int n, long long L, int FB, uint32_t p,
                                                            uint64_t mu) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int sa = m * kk, sb = kk * n;
    const int mb = m >> 2, nb = n >> 2;
    uint32_t* SA = sm;                  // [FB][m][kk]
    uint32_t* SB = sm + FB * sa;        // [FB][kk][n]
    for (long long f0 = (long long)blockIdx.x * FB; f0 < L; f0 += (long long)gridDim.x * FB) {
        const int nf = (int)(L - f0 < FB ? L - f0 : FB);
        __syncthreads();
        const uint4* gA = (const uint4*)(At + f0 * sa);
        for (int e = threadIdx.x; e < nf * sa / 4; e += blockDim.x) ((uint4*)SA)[e] = gA[e];
        const uint4* gB = (const uint4*)(Bt + f0 * sb);
        for (int e = threadIdx.x; e < nf * sb / 4; e += blockDim.x) ((uint4*)SB)[e] = gB[e];
        __syncthreads();
        const int nblk = nf * mb * nb;
        for (int o = threadIdx.x; o < nblk; o += blockDim.x) {
            const int jb = o % nb, ib = (o / nb) % mb, f = o / (mb * nb);
            const uint32_t* a = SA + f * sa + ib * 4 * kk;
            const uint32_t* bb = SB + f * sb + jb * 4;
            uint64_t acc[4][4], hi[4][4];
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int v = 0; v < 4; v++) { acc[u][v] = 0; hi[u][v] = 0; }
            for (int l0 = 0; l0 < kk; l0 += 16) {
                const int le = kk - l0 < 16 ? kk - l0 : 16;
#pragma unroll 4
                for (int l = l0; l < l0 + le; l++) {
                    const uint4 yb = *(const uint4*)(bb + l * n);
                    const uint32_t x[4] = {a[l], a[kk + l], a[2 * kk + l], a[3 * kk + l]};
                    const uint32_t y[4] = {yb.x, yb.y, yb.z, yb.w};
#pragma unroll
                    for (int u = 0; u < 4; u++)
#pragma unroll
                        for (int v = 0; v < 4; v++) acc[u][v] += (uint64_t)x[u] * y[v];
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        hi[u][v] += acc[u][v] >> 32;
                        acc[u][v] &= 0xFFFFFFFFull;
                    }
            }
            uint32_t* cf = Ct + (f0 + f) * (long long)(m * n) + (ib * 4) * n + jb * 4;
#pragma unroll
            for (int u = 0; u < 4; u++) {
                uint4 r;
                r.x = mod96_barrett(hi[u][0], acc[u][0], p, mu);
                r.y = mod96_barrett(hi[u][1], acc[u][1], p, mu);
                r.z = mod96_barrett(hi[u][2], acc[u][2], p, mu);
                r.w = mod96_barrett(hi[u][3], acc[u][3], p, mu);
                *(uint4*)(cf + u * n) = r;
            }
        }
    }
}

// ---------------------------------------------------------------- three-prime integer product
// p1 = 998244353, p2 = 985661441, p3 = 943718401, 32-bit chunks (h = 32).
struct Crt3 {
    uint32_t p1, p2, p3;
    uint32_t i12, i13, i23;   // p1^-1 mod p2, p1^-1 mod p3, p2^-1 mod p3
    uint64_t p12;             // p1 p2
};
__global__ void k_residues3(const uint32_t* __restrict__ x, long long n, uint32_t* __restrict__ r, long long stride,
                            Crt3 K) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint32_t v = x[i];
        r[i] = v % K.p1;
        r[stride + i] = v % K.p2;
        r[2 * stride + i] = v % K.p3;
    }
}
// Garner: c = x1 + p1 x2 + p1 p2 x3 < p1 p2 p3 < 2^90 from c mod p1, p2, p3 -> three 32-bit words
__global__ void k_crt3(const uint32_t* __restrict__ c, long long stride, long long n, uint32_t* __restrict__ w, Crt3 K) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const uint32_t x1 = c[k], r2 = c[stride + k], r3 = c[2 * stride + k];
        const uint32_t t2 = (uint32_t)(((uint64_t)(r2 + K.p2 - x1 % K.p2) % K.p2 * K.i12) % K.p2);
        const uint32_t t3 = (uint32_t)(((uint64_t)(r3 + K.p3 - x1 % K.p3) % K.p3 * K.i13) % K.p3);
        const uint32_t x3 = (uint32_t)(((uint64_t)(t3 + K.p3 - t2 % K.p3) % K.p3 * K.i23) % K.p3);
        const uint64_t lo = (uint64_t)x1 + (uint64_t)K.p1 * t2;           // < 2^61
        const uint64_t ml = K.p12 * x3, mh = __umul64hi(K.p12, (uint64_t)x3);
        const uint64_t s = lo + ml;
        const uint64_t hi = mh + (s < lo ? 1 : 0);
        w[3 * k] = (uint32_t)s;
        w[3 * k + 1] = (uint32_t)(s >> 32);
        w[3 * k + 2] = (uint32_t)hi;
    }
}

// ---------------------------------------------------------------- fused Garner CRT + carries (three-prime path)
// One pass from the three residue products to 32-bit limbs: a CTA of the
// single-pass look-back carry (k_carry16_fused's scheme) stages the
// coefficients its 4096 limbs need, rebuilding each from c mod p1, p2, p3 by
// Garner (c = x1 + p1 t2 + p1 p2 x3 < p1 p2 p3, three 32-bit words) with
// Shoup products instead of 64-bit divisions, then forms digit sums
// s_j = w0(c_j) + w1(c_{j-1}) + w2(c_{j-2}) and the (generate, propagate) chain.
// Limb positions: entry e = j / nout, local jl = j - e nout; coefficient jl of
// entry e (residue q at Cp[q stride + e nc + jl]) exists for jl < nc, the
// positions jl in [nc, nout) are zero (nout - nc >= 1 keeps entries apart:
// a limb's digit sum reaches 2 positions back, and positions of the previous
// entry that close are its zero tail when nout - nc = 2, or absent when E = 1).
struct Crt3S {
    uint32_t p1, p2, p3;
    uint32_t i12, i12s, i13, i13s, i23, i23s;   // inverses and their Shoup companions
    uint64_t p12;
};
__device__ __forceinline__ uint32_t shoup_mul(uint32_t x, uint32_t w, uint32_t ws, uint32_t p) {
    const uint32_t q = __umulhi(x, ws);
    const uint32_t r = x * w - q * p;        // in [0, 2p)
    return r >= p ? r - p : r;
}
__device__ __forceinline__ void garner3(uint32_t r1, uint32_t r2, uint32_t r3, const Crt3S& K, uint32_t* w) {
    const uint32_t x1 = r1;
    const uint32_t x1m2 = x1 >= K.p2 ? x1 - K.p2 : x1;                 // x1 < p1 < 2 p2
    const uint32_t d2 = r2 >= x1m2 ? r2 - x1m2 : r2 + K.p2 - x1m2;
    const uint32_t t2 = shoup_mul(d2, K.i12, K.i12s, K.p2);           // (r2 - x1) / p1 mod p2
    const uint32_t x1m3 = x1 >= K.p3 ? x1 - K.p3 : x1;                 // x1 < 2 p3
    const uint32_t d3 = r3 >= x1m3 ? r3 - x1m3 : r3 + K.p3 - x1m3;
    const uint32_t t3 = shoup_mul(d3, K.i13, K.i13s, K.p3);           // (r3 - x1) / p1 mod p3
    const uint32_t t2m3 = t2 >= K.p3 ? t2 - K.p3 : t2;                 // t2 < p2 < 2 p3
    const uint32_t e3 = t3 >= t2m3 ? t3 - t2m3 : t3 + K.p3 - t2m3;
    const uint32_t x3 = shoup_mul(e3, K.i23, K.i23s, K.p3);           // (t3 - t2) / p2 mod p3
    const uint64_t lo = (uint64_t)x1 + (uint64_t)K.p1 * t2;            // < 2^60
    const uint64_t ml = K.p12 * x3, mh = __umul64hi(K.p12, (uint64_t)x3);
    const uint64_t sum = lo + ml;
    w[0] = (uint32_t)sum;
    w[1] = (uint32_t)(sum >> 32);
    w[2] = (uint32_t)(mh + (sum < lo ? 1 : 0));
}
constexpr int CC_HALO = 3;                                  // positions before a block: s_{jb-1} reaches jb - 3
__global__ void __launch_bounds__(CARRY_T) k_crt_carry32(const uint32_t* __restrict__ Cp, long long stride,
                                                         long long nc, long long nout, long long nall, Crt3S K,
                                                         unsigned long long* status, unsigned* ticket,
                                                         uint32_t* __restrict__ out) {
    extern __shared__ uint32_t sw_dyn[];                    // the three words of every staged position
    uint32_t (*sw)[CARRY_B + CC_HALO + 1] = (uint32_t (*)[CARRY_B + CC_HALO + 1])sw_dyn;
    __shared__ uint32_t sh[64];
    __shared__ uint32_t s_bid, s_cin;
    if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
    __syncthreads();
    const long long bid = s_bid;
    const long long jb = bid * CARRY_B;
    // stage: 4 positions per thread per round, loads of a round issued together
    constexpr int NPOS = CARRY_B + CC_HALO, ROUNDS = (NPOS + 4 * CARRY_T - 1) / (4 * CARRY_T);
#pragma unroll 1
    for (int rd = 0; rd < ROUNDS; rd++) {
        uint32_t r1[4], r2[4], r3[4];
        bool live[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int r = threadIdx.x + (rd * 4 + u) * CARRY_T;
            const long long q = jb - CC_HALO + r;
            long long at = 0;
            live[u] = false;
            if (r < NPOS && q >= 0 && q < nall) {
                const long long e = q / nout, jl = q - e * nout;
                live[u] = jl < nc;
                at = e * nc + jl;
            }
            r1[u] = live[u] ? __ldg(Cp + at) : 0u;
            r2[u] = live[u] ? __ldg(Cp + stride + at) : 0u;
            r3[u] = live[u] ? __ldg(Cp + 2 * stride + at) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int r = threadIdx.x + (rd * 4 + u) * CARRY_T;
            if (r >= NPOS) continue;
            uint32_t w[3] = {0u, 0u, 0u};
            if (live[u]) garner3(r1[u], r2[u], r3[u], K, w);
            sw[0][r] = w[0];
            sw[1][r] = w[1];
            sw[2][r] = w[2];
        }
    }
    __syncthreads();
    // limbs j = jb + 16 t + e: s_j = w0(c_j) + w1(c_{j-1}) + w2(c_{j-2}); u_j = (s_j mod 2^32) + (s_{j-1} >> 32)
    uint32_t w[16], g[16];
    {
        const int base = CC_HALO + 16 * (int)threadIdx.x;    // staged index of limb j0
        // s_{j0 - 1}; positions before 0 are staged as zeros, so s_{-1} = 0
        uint64_t sprev = (uint64_t)sw[0][base - 1] + sw[1][base - 2] + sw[2][base - 3];
#pragma unroll
        for (int e = 0; e < 16; e++) {
            const int i = base + e;
            const uint64_t sj = (uint64_t)sw[0][i] + sw[1][i - 1] + sw[2][i - 2];
            const uint64_t u = (sj & 0xFFFFFFFFull) + (sprev >> 32);
            w[e] = (uint32_t)u;
            g[e] = (uint32_t)(u >> 32);
            sprev = sj;
        }
    }
    uint32_t acc = 2u;
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const long long j = jb + 16 * threadIdx.x + e;
        acc = gp_comb(acc, j < nall ? (g[e] | ((w[e] == 0xFFFFFFFFu ? 1u : 0u) << 1)) : 2u);
    }
    {   // block aggregate, publication and decoupled look-back (as k_carry16_fused)
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        uint32_t x = acc;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = gp_comb(y, x);
        }
        if (lane == 31) sh[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t agg = 2u;
            for (int q = 0; q < (int)(blockDim.x >> 5); q++) agg = gp_comb(agg, sh[q]);
            if (bid == 0) {
                if (lane == 0) {
                    st_release64(status, (2ull << 32) | agg);
                    s_cin = 0;
                }
            } else {
                if (lane == 0) st_release64(status + bid, (1ull << 32) | agg);
                uint32_t run = 2u;
                for (long long k = bid - 1;; k -= 32) {
                    const long long kk = k - lane;
                    unsigned long long v = (2ull << 32) | 2u;
                    if (kk >= 0)
                        do { v = ld_acquire64(status + kk); } while ((v >> 32) == 0);
                    const unsigned inc = __ballot_sync(0xffffffffu, (v >> 32) == 2);
                    const int stop = inc ? __ffs(inc) - 1 : 31;
                    uint32_t x2 = lane <= stop ? (uint32_t)v : 2u;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_down_sync(0xffffffffu, x2, o);
                        if (lane + o < 32) x2 = gp_comb(y, x2);
                    }
                    run = gp_comb(__shfl_sync(0xffffffffu, x2, 0), run);
                    if (inc) break;
                }
                if (lane == 0) {
                    st_release64(status + bid, (2ull << 32) | gp_comb(run, agg));
                    s_cin = run & 1u;
                }
            }
        }
        __syncthreads();
    }
    uint32_t C = block_carry_in(acc, s_cin, sh);
    const long long j0 = jb + 16 * threadIdx.x;
    uint32_t o[16];
#pragma unroll
    for (int e = 0; e < 16; e++) {
        o[e] = w[e] + C;
        C = g[e] | ((w[e] == 0xFFFFFFFFu ? 1u : 0u) & C);
    }
    if (j0 + 16 <= nall && ((((uintptr_t)(out + j0)) & 15) == 0)) {
        uint4* d = (uint4*)(out + j0);
#pragma unroll
        for (int i = 0; i < 4; i++) d[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
    } else {
#pragma unroll
        for (int e = 0; e < 16; e++)
            if (j0 + e < nall) out[j0 + e] = o[e];
    }
}

}  // namespace mm

using namespace mm;

// ====================================================================== plans
struct mm_ntt_plan {
    int word_bits;
    uint64_t p, omega;
    int k, k1, k2;           // n = 2^k = n2 * n1, n1 = 2^k1 (rows), n2 = 2^k2 (cols)
    size_t batch;
    void* lvl_f1 = nullptr;  // level tables for n1 (or n when single pass)
    void* lvl_i1 = nullptr;
    void* lvl_f2 = nullptr;  // level tables for n2
    void* lvl_i2 = nullptr;
    void* fs_lo_f = nullptr; // four-step twiddles w^e split at fs_h bits
    void* fs_hi_f = nullptr;
    void* fs_lo_i = nullptr;
    void* fs_hi_i = nullptr;
    void* fs_full_f = nullptr; // full step-2 tables [i2][j1] (small n only)
    void* fs_full_i = nullptr;
    int fs_h = 0;
    uint64_t ninv;           // n^-1 mod p
    uint64_t ninv_r;         // n^-1 2^32 mod p (32-bit: after REDC)
    uint32_t pinv;           // p^-1 mod 2^32
    // specialised 2^16 = 256 x 256 path (ntt_fast32.cu), 32-bit only
    bool fast16 = false;
    void* fs_pm_i = nullptr;   // inverse step-2 table times n^-1 2^32
    void* fs_ni_i = nullptr;   // inverse step-2 table times n^-1 (standalone inverse)
    mm::f32::Tw15 tw_f1, tw_i1, tw_f2, tw_i2;   // level-table entries 1..15 (host copies)
};

namespace mm {

template <class F> static F make_field(const mm_ntt_plan* P);
template <> Fp32 make_field<Fp32>(const mm_ntt_plan* P) {
    Fp32 f;
    f.p = (uint32_t)P->p;
    f.p2 = 2 * (uint32_t)P->p;
    f.pinv = P->pinv;
    f.pr = (uint32_t)((1ull << 32) / P->p);
    return f;
}
template <> FpG make_field<FpG>(const mm_ntt_plan*) { return FpG(); }
template <> FpD make_field<FpD>(const mm_ntt_plan* P) {
    FpD f;
    f.p = (double)P->p;
    f.u = 1.0 / f.p;
    return f;
}

static inline uint2 mkw32(uint64_t w, uint64_t p) {
    return make_uint2((uint32_t)w, (uint32_t)(((u128)w << 32) / p));
}
template <class W> static W host_w(uint64_t w, uint64_t p);
template <> uint2 host_w<uint2>(uint64_t w, uint64_t p) { return mkw32(w, p); }
template <> uint64_t host_w<uint64_t>(uint64_t w, uint64_t) { return w; }
template <> double host_w<double>(uint64_t w, uint64_t) { return (double)w; }

static size_t esize(int word_bits) { return word_bits == 32 ? 4 : 8; }


constexpr int MAX_BLOCK_LOG = 12;   // single-pass limit (longer transforms use Algorithm 1)

// explicit instantiations live in ntt_inst32.cu / ntt_inst64.cu
extern template mm_status launch_rows<Fp32, false, uint32_t, uint32_t>(const Fp32&, const RowArgs<Fp32>&, cudaStream_t);
extern template mm_status launch_rows<Fp32, true, uint32_t, uint32_t>(const Fp32&, const RowArgs<Fp32>&, cudaStream_t);
extern template mm_status launch_cols<Fp32, false, uint32_t, uint32_t>(const Fp32&, const ColArgs<Fp32>&, cudaStream_t);
extern template mm_status launch_cols<Fp32, true, uint32_t, uint32_t>(const Fp32&, const ColArgs<Fp32>&, cudaStream_t);
extern template mm_status launch_pmul<Fp32, uint32_t, uint32_t>(const Fp32&, const PmulArgs<Fp32>&, cudaStream_t);
extern template mm_status launch_rows<FpG, false, uint64_t, uint64_t>(const FpG&, const RowArgs<FpG>&, cudaStream_t);
extern template mm_status launch_rows<FpG, true, uint64_t, uint64_t>(const FpG&, const RowArgs<FpG>&, cudaStream_t);
extern template mm_status launch_cols<FpG, false, uint64_t, uint64_t>(const FpG&, const ColArgs<FpG>&, cudaStream_t);
extern template mm_status launch_cols<FpG, true, uint64_t, uint64_t>(const FpG&, const ColArgs<FpG>&, cudaStream_t);
extern template mm_status launch_cols<FpG, false, uint16_t, uint64_t>(const FpG&, const ColArgs<FpG>&, cudaStream_t);
extern template mm_status launch_pmul<FpG, uint64_t, uint64_t>(const FpG&, const PmulArgs<FpG>&, cudaStream_t);
extern template mm_status launch_pmul<FpG, uint16_t, uint64_t>(const FpG&, const PmulArgs<FpG>&, cudaStream_t);
extern template mm_status launch_rows<FpD, false, double, double>(const FpD&, const RowArgs<FpD>&, cudaStream_t);
extern template mm_status launch_rows<FpD, true, double, double>(const FpD&, const RowArgs<FpD>&, cudaStream_t);
extern template mm_status launch_cols<FpD, false, double, double>(const FpD&, const ColArgs<FpD>&, cudaStream_t);
extern template mm_status launch_cols<FpD, true, double, double>(const FpD&, const ColArgs<FpD>&, cudaStream_t);
extern template mm_status launch_pmul<FpD, double, double>(const FpD&, const PmulArgs<FpD>&, cudaStream_t);

// ---- plan construction
// entries 1..15 of the level table of a length-2^k transform with root r: tw[m + i] = r^(i 2^k / 2m)
static void tw15(f32::Tw15* T, uint64_t r, int k, uint64_t p) {
    T->w[0] = make_uint2(0, 0);
    for (int m = 1; m <= 8; m <<= 1)
        for (int i = 0; i < m; i++) T->w[m + i] = mkw32(hpowmod(r, (uint64_t)i << (k - 1 - (31 - __builtin_clz(m))), p), p);
}
// Goldilocks plans append the natural powers w^e (e < L) after the level table:
// gold.cuh's tiles read their 64-th-root and w_L^(b k_a) twiddles there.
template <class W, class E>
static mm_status build_level(void** dst, int k, E w, uint64_t p) {
    size_t L = (size_t)1 << k;
    constexpr bool NAT = std::is_same<W, uint64_t>::value;
    MM_CUDA_TRY(cudaMalloc(dst, (NAT ? 2 : 1) * L * sizeof(W)));
    int grid = (int)((L + 255) / 256 < 4096 ? (L + 255) / 256 : 4096);
    {
        LaunchScope ls("twiddle_level_table", 0);
        k_level_table<W, E><<<grid, 256>>>((W*)*dst, k, w, p);
        if (NAT) k_pow_table<W, E><<<grid, 256>>>((W*)*dst + L, (long long)L, w, 1, p);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
template <class W, class E>
static mm_status build_pow(void** dst, long long cnt, E w, uint64_t step, uint64_t p) {
    MM_CUDA_TRY(cudaMalloc(dst, (size_t)cnt * sizeof(W)));
    int grid = (int)((cnt + 255) / 256 < 4096 ? (cnt + 255) / 256 : 4096);
    {
        LaunchScope ls("twiddle_pow_table", 0);
        k_pow_table<W, E><<<grid, 256>>>((W*)*dst, cnt, w, step, p);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

template <class W, class E>
static mm_status build_fs_full(void** dst, int k1, int k2, E w, uint64_t p) {
    long long cnt = 1ll << (k1 + k2);
    MM_CUDA_TRY(cudaMalloc(dst, (size_t)cnt * sizeof(W)));
    int grid = (int)((cnt + 255) / 256 < 4096 ? (cnt + 255) / 256 : 4096);
    {
        LaunchScope ls("twiddle_fs_table", 0);
        k_fs_table<W, E><<<grid, 256>>>((W*)*dst, k1, k2, w, p);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

template <class W, class E>
static mm_status build_tables(mm_ntt_plan* P) {
    uint64_t p = P->p, w = P->omega;
    uint64_t winv = hpowmod(w, p - 2, p);
    int k = P->k;
    mm_status s;
    if (P->k2 == 0) {
        if ((s = build_level<W, E>(&P->lvl_f1, k, (E)w, p)) != MM_OK) return s;
        if ((s = build_level<W, E>(&P->lvl_i1, k, (E)winv, p)) != MM_OK) return s;
    } else {
        // rows: length n1 with root w^n2; columns: length n2 with root w^n1 (Algorithm 1 steps 1, 3)
        uint64_t n1 = 1ull << P->k1, n2 = 1ull << P->k2;
        if ((s = build_level<W, E>(&P->lvl_f1, P->k1, (E)hpowmod(w, n2, p), p)) != MM_OK) return s;
        if ((s = build_level<W, E>(&P->lvl_i1, P->k1, (E)hpowmod(winv, n2, p), p)) != MM_OK) return s;
        if ((s = build_level<W, E>(&P->lvl_f2, P->k2, (E)hpowmod(w, n1, p), p)) != MM_OK) return s;
        if ((s = build_level<W, E>(&P->lvl_i2, P->k2, (E)hpowmod(winv, n1, p), p)) != MM_OK) return s;
        // step 2 twiddles w^e, e < n, e = e_lo + 2^h e_hi
        int h = (k + 1) / 2;
        P->fs_h = h;
        long long nlo = 1ll << h, nhi = 1ll << (k - h);
        if ((s = build_pow<W, E>(&P->fs_lo_f, nlo, (E)w, 1, p)) != MM_OK) return s;
        if ((s = build_pow<W, E>(&P->fs_hi_f, nhi, (E)w, 1ull << h, p)) != MM_OK) return s;
        if ((s = build_pow<W, E>(&P->fs_lo_i, nlo, (E)winv, 1, p)) != MM_OK) return s;
        if ((s = build_pow<W, E>(&P->fs_hi_i, nhi, (E)winv, 1ull << h, p)) != MM_OK) return s;
        // full tables TW[i2 n1 + j1] = w^(+-j1 [i2]) up to 32 MiB each (n <= 2^22),
        // always for Goldilocks plans: the passes are ALU-bound and one table
        // word (8 B streamed beside the pass's 8-16 B per element) replaces two
        // split-table loads and one of two products per element (64 x 2^20
        // 32-bit forward 0.63 -> 0.52 ms, three-prime Table-16 product 0.256 ->
        // 0.224 ms against the former 2 MiB L2-resident limit)
        if (((size_t)1 << k) * sizeof(W) <= ((size_t)32 << 20) || P->word_bits == 64) {
            if ((s = build_fs_full<W, E>(&P->fs_full_f, P->k1, P->k2, (E)w, p)) != MM_OK) return s;
            if ((s = build_fs_full<W, E>(&P->fs_full_i, P->k1, P->k2, (E)winv, p)) != MM_OK) return s;
        }
        if (P->word_bits == 32 && P->k1 == 8 && P->k2 == 8) {
            // the specialised 256 x 256 kernels: host copies of the small level-table
            // entries, and the inverse step-2 table with n^-1 2^32 folded in
            uint64_t r1 = hpowmod(w, n2, p), r1i = hpowmod(winv, n2, p);
            uint64_t r2 = hpowmod(w, n1, p), r2i = hpowmod(winv, n1, p);
            tw15(&P->tw_f1, r1, P->k1, p);
            tw15(&P->tw_i1, r1i, P->k1, p);
            tw15(&P->tw_f2, r2, P->k2, p);
            tw15(&P->tw_i2, r2i, P->k2, p);
            MM_CUDA_TRY(cudaMalloc(&P->fs_pm_i, ((size_t)1 << k) * sizeof(uint2)));
            MM_CUDA_TRY(cudaMalloc(&P->fs_ni_i, ((size_t)1 << k) * sizeof(uint2)));
            {
                LaunchScope ls("twiddle_fs_table", 0);
                k_fs_table_scaled32<<<256, 256>>>((uint2*)P->fs_pm_i, P->k1, P->k2, (uint32_t)winv,
                                                  (uint32_t)P->ninv_r, (uint32_t)p);
                k_fs_table_scaled32<<<256, 256>>>((uint2*)P->fs_ni_i, P->k1, P->k2, (uint32_t)winv,
                                                  (uint32_t)P->ninv, (uint32_t)p);
            }
            MM_LAUNCH_CHECK();
            P->fast16 = true;
        }
    }
    MM_CUDA_TRY(cudaDeviceSynchronize());
    return MM_OK;
}

static void free_plan(mm_ntt_plan* P) {
    if (!P) return;
    void* bufs[] = {P->lvl_f1,  P->lvl_i1,  P->lvl_f2,    P->lvl_i2,    P->fs_lo_f, P->fs_hi_f,
                    P->fs_lo_i, P->fs_hi_i, P->fs_full_f, P->fs_full_i, P->fs_pm_i, P->fs_ni_i};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete P;
}

static mm_status check_modulus(int word_bits, uint64_t p, int log2n) {
    if (word_bits == 32) {
        if (p < 3 || !(p & 1) || !hprime(p)) return set_err(MM_E_INVALID_MODULUS, "p=%llu is not an odd prime", (unsigned long long)p);
        if (p >= (1ull << 30)) return set_err(MM_E_PROFILE, "32-bit NTT needs p < 2^30 (lazy butterflies in [0,4p)), got %llu", (unsigned long long)p);
        if (log2n < 1 || log2n > 24) return set_err(MM_E_UNSUPPORTED_SIZE, "log2n=%d out of [1,24]", log2n);
    } else if (word_bits == 64) {
        if (p != FpG::P) return set_err(MM_E_INVALID_MODULUS, "64-bit NTT supports only p = 2^64 - 2^32 + 1");
        if (log2n < 1 || log2n > 25) return set_err(MM_E_UNSUPPORTED_SIZE, "log2n=%d out of [1,25]", log2n);
    } else if (word_bits == 52) {
        if (p < 3 || !(p & 1) || !hprime(p)) return set_err(MM_E_INVALID_MODULUS, "p=%llu is not an odd prime", (unsigned long long)p);
        if (p >= (1ull << 50))
            return set_err(MM_E_PROFILE, "FP64 NTT needs p < 2^50 (Function 16: m <= l - 2), got %llu", (unsigned long long)p);
        if (log2n < 1 || log2n > 25) return set_err(MM_E_UNSUPPORTED_SIZE, "log2n=%d out of [1,25]", log2n);
    } else {
        return set_err(MM_E_ARG, "word_bits must be 32, 64 or 52 (FP64 residues)");
    }
    if (log2n > two_adicity(p)) return set_err(MM_E_UNSUPPORTED_SIZE, "2^%d does not divide p-1", log2n);
    return MM_OK;
}

// longest one-pass transform: 2^13 points for 64-bit and 32-bit words (a 32 KiB
// row tile; against the 2^6 x 2^7 split: forward 1.59 -> 1.09 ms per 2^28
// elements, products of 4096 x 4096 coefficients 4.31 -> 2.98 ms per 2^27;
// MMNTT_ONEPASS32_13=0 restores the split), 2^12 for FP64 residues
static int onepass_log(int word_bits) {
    static const bool w32 = !(getenv("MMNTT_ONEPASS32_13") && atoi(getenv("MMNTT_ONEPASS32_13")) == 0);
    return word_bits == 64 || (word_bits == 32 && w32) ? MAX_BLOCK_LOG + 1 : MAX_BLOCK_LOG;
}

static mm_status plan_create(int word_bits, uint64_t p, int log2n, uint64_t omega, size_t batch, mm_ntt_plan** out) {
    mm_status s = check_modulus(word_bits, p, log2n);
    if (s != MM_OK) return s;
    uint64_t n = 1ull << log2n;
    omega %= p;
    if (hpowmod(omega, n / 2, p) != p - 1)
        return set_err(MM_E_BAD_ROOT, "omega^(n/2) != p-1: omega is not a primitive 2^%d-th root", log2n);
    mm_ntt_plan* P = new (std::nothrow) mm_ntt_plan;
    if (!P) return set_err(MM_E_ARG, "out of host memory");
    P->word_bits = word_bits;
    P->p = p;
    P->omega = omega;
    P->k = log2n;
    P->batch = batch;
    // Goldilocks rows of 2^13 points run in one pass (512-thread CTAs, gold.cuh)
    if (log2n <= onepass_log(word_bits)) {
        P->k1 = log2n;
        P->k2 = 0;
    } else {
        // n1 (row length, contiguous) >= n2 (column length, strided); the
        // column pass keeps <= 2^10 (32-bit) / 2^11 (64-bit) points per column
        // tile so that several CTAs share an SM; rows go up to 2^13.
        int cap = word_bits == 32 ? 10 : 11;
        int k2 = log2n / 2 < cap ? log2n / 2 : cap;
        if (log2n - k2 > 13) k2 = log2n - 13;
        // Goldilocks: the 2^13-point rows run on gold.cuh's tiles, short columns
        // on the interleaved generic tiles (2^19..2^21: 10-11 % faster than the
        // balanced split; 2^18, 2^22, 2^23 measured slower)
        if (word_bits == 64 && log2n >= 19 && log2n <= 21) k2 = log2n - 13;   // measured: tools/time_split.py
        // 32-bit: 2^8-point columns up to 2^21 (tools/exp_split32.py, per 2^28
        // elements: 2^18 forward 2.21 -> 1.55 ms, 2^20 2.31 -> 1.55 ms against the
        // 2^9 / 2^10-point columns of the balanced split; 2^22 would need 2^14-point
        // rows and keeps 2^10 x 2^12; MMNTT_SPLIT32_BALANCED=1 restores the old rule)
        static const bool bal32 = getenv("MMNTT_SPLIT32_BALANCED") && atoi(getenv("MMNTT_SPLIT32_BALANCED")) != 0;
        if (word_bits == 32 && log2n >= 17 && log2n <= 21 && !bal32) k2 = 8;
        if (const char* e = getenv("MMNTT_K2_32"))   // 32-bit split experiments (tools/exp_split32.py)
            if (word_bits == 32 && atoi(e) >= log2n - 13 && atoi(e) >= 1 && atoi(e) <= 10 && atoi(e) < log2n) k2 = atoi(e);
        if (const char* e = getenv("MMNTT_K2_64"))   // split experiments (tools/time_g.py)
            if (word_bits == 64 && atoi(e) >= log2n - 13 && atoi(e) <= 12 && atoi(e) < log2n) k2 = atoi(e);
        P->k2 = k2;
        P->k1 = log2n - k2;
    }
    P->ninv = hpowmod(n % p, p - 2, p);
    P->ninv_r = word_bits == 32 ? hmulmod(P->ninv, ((u128)1 << 32) % p, p) : P->ninv;
    P->pinv = word_bits == 32 ? inv_mod_2_32((uint32_t)p) : 0;
    s = word_bits == 32   ? build_tables<uint2, uint32_t>(P)
        : word_bits == 52 ? build_tables<double, D50>(P)
                          : build_tables<uint64_t, uint64_t>(P);
    if (s != MM_OK) {
        free_plan(P);
        return s;
    }
    *out = P;
    return MM_OK;
}

// NATURAL-order transforms on the four-step path go through a bit-mirror
// permutation of a temporary: a stream-ordered allocation
// (alloc_async / cudaFreeAsync from the library's memory pool), so the
// plan holds no mutable workspace and calls on different streams sharing a
// plan never touch the same buffer, and nothing here synchronises.
template <class T>
static mm_status bitrev_rows(const void* in, void* out, int k, long long batch, cudaStream_t st) {
    {
        LaunchScope ls("bitrev_permute", st);
        // MMNTT_BITREV_TILED=0 selects the element-wise form (comparison runs)
        static const bool tiled = !(getenv("MMNTT_BITREV_TILED") && atoi(getenv("MMNTT_BITREV_TILED")) == 0);
        if (k >= 10 && tiled) k_bitrev_tiled<T><<<num_sms() * 8, 256, 0, st>>>((const T*)in, (T*)out, k, batch);
        else k_bitrev_perm<T><<<num_sms() * 8, 256, 0, st>>>((const T*)in, (T*)out, k, batch);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

// ---- fork streams for sub-batch concurrency (product_impl) ----------------------
constexpr int MAX_FORK = 4;
struct Fork {
    cudaStream_t s[MAX_FORK];
    cudaEvent_t fork, join[MAX_FORK];
    std::mutex mu;
};
static std::mutex g_fork_mu;
static std::map<int, Fork*> g_forks;
static int g_product_streams = 2;
static int product_streams() { return g_product_streams; }
static mm_status fork_streams(Fork** out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_fork_mu);
    Fork*& F = g_forks[dev];
    if (!F) {
        Fork* f = new (std::nothrow) Fork;
        if (!f) return set_err(MM_E_ARG, "out of host memory");
        for (int i = 0; i < MAX_FORK; i++) {
            MM_CUDA_TRY(cudaStreamCreateWithFlags(&f->s[i], cudaStreamNonBlocking));
            MM_CUDA_TRY(cudaEventCreateWithFlags(&f->join[i], cudaEventDisableTiming));
        }
        MM_CUDA_TRY(cudaEventCreateWithFlags(&f->fork, cudaEventDisableTiming));
        F = f;
    }
    *out = F;
    return MM_OK;
}

// fn(in + r0 n, out + r0 n, rows, stream) over the fork streams, sub-batches of
// the batch forked from and joined back into st (one call on st when the
// concurrency is 1 or the batch is a single transform)
template <class T, class Fn>
static mm_status forked(const T* in, T* out, long long batch, long long n, cudaStream_t st, Fn fn) {
    const int ns = (int)(product_streams() < batch ? product_streams() : batch);
    if (ns < 2) return fn(in, out, batch, st);
    Fork* FK = nullptr;
    mm_status s = fork_streams(&FK);
    if (s != MM_OK) return s;
    std::lock_guard<std::mutex> lk(FK->mu);
    MM_CUDA_TRY(cudaEventRecord(FK->fork, st));
    long long r0 = 0;
    for (int h = 0; h < ns; h++) {
        const long long rows = batch / ns + (h < batch % ns ? 1 : 0);
        MM_CUDA_TRY(cudaStreamWaitEvent(FK->s[h], FK->fork, 0));
        if ((s = fn(in + r0 * n, out + r0 * n, rows, FK->s[h])) != MM_OK) return s;
        MM_CUDA_TRY(cudaEventRecord(FK->join[h], FK->s[h]));
        MM_CUDA_TRY(cudaStreamWaitEvent(st, FK->join[h], 0));
        r0 += rows;
    }
    return MM_OK;
}

// ---- forward / inverse drivers ------------------------------------------------------
template <class F>
static mm_status fwd_impl(mm_ntt_plan* P, const void* in, void* out, mm_order order, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    const long long n = 1ll << P->k;
    if (P->k2 == 0) {
        RowArgs<F> a{};
        a.in = in; a.out = out;
        a.nrows = (long long)P->batch;
        a.in_rs = a.out_rs = n;
        a.in_len = a.out_len = n;
        a.k = P->k;
        a.perm = order == MM_ORDER_NATURAL;
        a.canon = 1;
        a.lvl = (const W*)P->lvl_f1;
        return launch_rows<F, false, T, T>(f, a, st);
    }
    if constexpr (sizeof(T) == 4) {
        if (order == MM_ORDER_NATURAL && P->fast16 && ((uintptr_t)out & 15) == 0) {
            // 256 x 256: column pass into a temporary, natural-order row pass into out
            void* tmp = nullptr;
            MM_CUDA_TRY(alloc_async(&tmp, (size_t)n * P->batch * sizeof(T), st));
            const f32::Fld ff{(uint32_t)P->p, 2 * (uint32_t)P->p, P->pinv};
            f32::ColFwdArgs cf{};
            cf.in = (const uint32_t*)in; cf.out = (uint32_t*)tmp;
            cf.nbatch = (long long)P->batch;
            cf.in_bs = cf.in_len = cf.out_bs = n;
            cf.lvl = (const uint2*)P->lvl_f2;
            cf.fs = (const uint2*)P->fs_full_f;
            cf.tc = P->tw_f2;
            cf.f = ff;
            mm_status s = f32::launch_col_fwd(cf, st);
            if (s == MM_OK) {
                f32::RowArgs32 ra{};
                ra.in = (const uint32_t*)tmp; ra.out = (uint32_t*)out;
                ra.nrows = (long long)P->batch << 8;
                ra.lvl = (const uint2*)P->lvl_f1;
                ra.tc = P->tw_f1;
                ra.f = ff;
                s = f32::launch_row_fwd_nat(ra, st);
            }
            cudaFreeAsync(tmp, st);
            return s;
        }
    }
    if (order == MM_ORDER_NATURAL) {   // Algorithm 1's TFT order into a temporary, then the permutation
        void* tmp = nullptr;
        MM_CUDA_TRY(alloc_async(&tmp, (size_t)n * P->batch * sizeof(T), st));
        mm_status s = fwd_impl<F>(P, in, tmp, MM_ORDER_BITREV, st);
        if (s == MM_OK) s = bitrev_rows<T>(tmp, out, P->k, (long long)P->batch, st);
        cudaFreeAsync(tmp, st);
        return s;
    }
    if constexpr (sizeof(T) == 4) {
        if (P->fast16 && ((uintptr_t)out & 15) == 0) {
            // 2^16 = 256 x 256: the specialised column and row passes (ntt_fast32.cu)
            const f32::Fld ff{(uint32_t)P->p, 2 * (uint32_t)P->p, P->pinv};
            f32::ColFwdArgs cf{};
            cf.in = (const uint32_t*)in; cf.out = (uint32_t*)out;
            cf.nbatch = (long long)P->batch;
            cf.in_bs = cf.in_len = cf.out_bs = n;
            cf.lvl = (const uint2*)P->lvl_f2;
            cf.fs = (const uint2*)P->fs_full_f;
            cf.tc = P->tw_f2;
            cf.f = ff;
            mm_status s = f32::launch_col_fwd(cf, st);
            if (s != MM_OK) return s;
            f32::RowArgs32 ra{};
            ra.in = (const uint32_t*)out; ra.out = (uint32_t*)out;
            ra.nrows = (long long)P->batch << 8;
            ra.lvl = (const uint2*)P->lvl_f1;
            ra.tc = P->tw_f1;
            ra.f = ff;
            return f32::launch_row_fwd(ra, st);
        }
    }
    // column pass: in -> out, then row pass: out -> out (bit-mirrored result),
    // for nb transforms from gin to gout on stream gs
    auto four_step = [&](const void* gin, void* gout, long long nb, cudaStream_t gs) -> mm_status {
        ColArgs<F> c{};
        c.in = gin; c.out = gout;
        c.ncols = 1ll << P->k1;
        c.nbatch = nb;
        c.in_rs = c.out_rs = 1ll << P->k1;
        c.in_bs = c.out_bs = n;
        c.in_len = c.out_len = n;
        c.col0 = 0;
        c.n1 = 1ll << P->k1;
        c.k = P->k2;
        c.fs = 1;
        c.lvl = (const W*)P->lvl_f2;
        c.fs_lo = (const W*)P->fs_lo_f;
        c.fs_hi = (const W*)P->fs_hi_f;
        c.fs_full = (const W*)P->fs_full_f;
        c.fs_h = P->fs_h;
        mm_status s = launch_cols<F, false, T, T>(f, c, gs);
        if (s != MM_OK) return s;
        RowArgs<F> a{};
        a.in = gout; a.out = gout;
        a.nrows = nb << P->k2;
        a.in_rs = a.out_rs = 1ll << P->k1;
        a.in_len = a.out_len = 1ll << P->k1;
        a.k = P->k1;
        a.canon = 1;
        a.lvl = (const W*)P->lvl_f1;
        return launch_rows<F, false, T, T>(f, a, gs);
    };
    // 64-bit four-step batches run as sub-batches on the fork streams (the
    // latency-bound column pass of one overlaps the row pass of the other:
    // C4 3.25 -> 3.04 ms on B200, tools/exp_streams2.py)
    // (not when both passes are the whole-SM TMA / bulk-copy Goldilocks kernels,
    // which cannot share an SM: C4 forward 2.76 forked vs 2.73 ms one stream)
    const bool whole_sm = std::is_same<F, FpG>::value && P->k1 == 13 && P->k2 == 11 && gold_tma_enabled();
    if (sizeof(T) == 8 && !whole_sm) return forked((const T*)in, (T*)out, (long long)P->batch, n, st, four_step);
    return four_step(in, out, (long long)P->batch, st);
}

template <class F>
static mm_status inv_impl(mm_ntt_plan* P, const void* in, void* out, mm_order order, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    const long long n = 1ll << P->k;
    W sc = host_w<W>(P->ninv, P->p);
    if (P->k2 == 0) {
        RowArgs<F> a{};
        a.in = in; a.out = out;
        a.nrows = (long long)P->batch;
        a.in_rs = a.out_rs = n;
        a.in_len = a.out_len = n;
        a.k = P->k;
        a.perm = order == MM_ORDER_NATURAL;
        a.scale = 1; a.sc = sc;
        a.canon = 1;
        a.lvl = (const W*)P->lvl_i1;
        return launch_rows<F, true, T, T>(f, a, st);
    }
    mm_status s;
    const void* src = in;
    if constexpr (sizeof(T) == 4) {
        if (order == MM_ORDER_NATURAL && P->fast16 && ((uintptr_t)in & 15) == 0 && ((uintptr_t)out & 15) == 0) {
            // 256 x 256: natural-order inverse row pass into a temporary, column pass into out
            void* tmp = nullptr;
            MM_CUDA_TRY(alloc_async(&tmp, (size_t)n * P->batch * sizeof(T), st));
            const f32::Fld ff{(uint32_t)P->p, 2 * (uint32_t)P->p, P->pinv};
            f32::RowArgs32 ra{};
            ra.in = (const uint32_t*)in; ra.out = (uint32_t*)tmp;
            ra.nrows = (long long)P->batch << 8;
            ra.lvl = (const uint2*)P->lvl_i1;
            ra.fsi = (const uint2*)P->fs_ni_i;
            ra.tc = P->tw_i1;
            ra.f = ff;
            s = f32::launch_row_inv_nat(ra, st);
            if (s == MM_OK) {
                f32::ColInvArgs ci{};
                ci.in = (const uint32_t*)tmp; ci.out = (uint32_t*)out;
                ci.nbatch = (long long)P->batch;
                ci.in_bs = n;
                ci.out_bs = ci.out_len = n;
                ci.lvl = (const uint2*)P->lvl_i2;
                ci.tc = P->tw_i2;
                ci.f = ff;
                s = f32::launch_col_inv(ci, st);
            }
            cudaFreeAsync(tmp, st);
            return s;
        }
    }
    if (order == MM_ORDER_NATURAL) {   // permute into a temporary, then the TFT-order inverse
        void* tmp = nullptr;
        MM_CUDA_TRY(alloc_async(&tmp, (size_t)n * P->batch * sizeof(T), st));
        s = bitrev_rows<T>(in, tmp, P->k, (long long)P->batch, st);
        if (s == MM_OK) s = inv_impl<F>(P, tmp, out, MM_ORDER_BITREV, st);
        cudaFreeAsync(tmp, st);
        return s;
    }
    if constexpr (sizeof(T) == 4) {
        if (P->fast16 && ((uintptr_t)src & 15) == 0 && ((uintptr_t)out & 15) == 0) {
            const f32::Fld ff{(uint32_t)P->p, 2 * (uint32_t)P->p, P->pinv};
            f32::RowArgs32 ra{};
            ra.in = (const uint32_t*)src; ra.out = (uint32_t*)out;
            ra.nrows = (long long)P->batch << 8;
            ra.lvl = (const uint2*)P->lvl_i1;
            ra.fsi = (const uint2*)P->fs_ni_i;
            ra.tc = P->tw_i1;
            ra.f = ff;
            if ((s = f32::launch_row_inv(ra, st)) != MM_OK) return s;
            f32::ColInvArgs ci{};
            ci.in = (const uint32_t*)out; ci.out = (uint32_t*)out;
            ci.nbatch = (long long)P->batch;
            ci.in_bs = n;
            ci.out_bs = ci.out_len = n;
            ci.lvl = (const uint2*)P->lvl_i2;
            ci.tc = P->tw_i2;
            ci.f = ff;
            return f32::launch_col_inv(ci, st);
        }
    }
    auto four_step = [&](const void* gin, void* gout, long long nb, cudaStream_t gs) -> mm_status {
        // inverse row pass (DIT over j1 + twiddle w^-(j1 [i2])): gin -> gout
        RowArgs<F> a{};
        a.in = gin; a.out = gout;
        a.nrows = nb << P->k2;
        a.in_rs = a.out_rs = 1ll << P->k1;
        a.in_len = a.out_len = 1ll << P->k1;
        a.k = P->k1;
        a.fs = 1; a.k2 = P->k2; a.row0 = 0;
        a.lvl = (const W*)P->lvl_i1;
        a.fs_lo = (const W*)P->fs_lo_i;
        a.fs_hi = (const W*)P->fs_hi_i;
        a.fs_full = (const W*)P->fs_full_i;
        a.fs_h = P->fs_h;
        mm_status s2 = launch_rows<F, true, T, T>(f, a, gs);
        if (s2 != MM_OK) return s2;
        // inverse column pass (DIT over i2, n^-1, canonical): gout -> gout
        ColArgs<F> c{};
        c.in = gout; c.out = gout;
        c.ncols = 1ll << P->k1;
        c.nbatch = nb;
        c.in_rs = c.out_rs = 1ll << P->k1;
        c.in_bs = c.out_bs = n;
        c.in_len = c.out_len = n;
        c.n1 = 1ll << P->k1;
        c.k = P->k2;
        c.scale = 1; c.sc = sc; c.canon = 1;
        c.lvl = (const W*)P->lvl_i2;
        return launch_cols<F, true, T, T>(f, c, gs);
    };
    (void)s;
    if (sizeof(T) == 8) return forked((const T*)src, (T*)out, (long long)P->batch, n, st, four_step);
    return four_step(src, out, (long long)P->batch, st);
}

// ---- forward with zero-padded input rows / inverse with truncated output rows ----------
// rows: `rows` transforms; input row r at in + r in_rs with in_len valid elements
// (zeros beyond); output BITREV rows of n (canonical).
template <class F>
static mm_status fwd_pad_impl(mm_ntt_plan* P, const void* in, long long rows, long long in_rs, long long in_len,
                              void* out, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    const long long n = 1ll << P->k;
    if constexpr (sizeof(T) == 4) {
        if (P->fast16 && ((uintptr_t)out & 15) == 0) {   // 256 x 256: the specialised passes
            const f32::Fld ff{(uint32_t)P->p, 2 * (uint32_t)P->p, P->pinv};
            f32::ColFwdArgs cf{};
            cf.in = (const uint32_t*)in; cf.out = (uint32_t*)out;
            cf.nbatch = rows;
            cf.in_bs = in_rs; cf.in_len = in_len; cf.out_bs = n;
            cf.lvl = (const uint2*)P->lvl_f2;
            cf.fs = (const uint2*)P->fs_full_f;
            cf.tc = P->tw_f2;
            cf.f = ff;
            mm_status s = f32::launch_col_fwd(cf, st);
            if (s != MM_OK) return s;
            f32::RowArgs32 ra{};
            ra.in = (const uint32_t*)out; ra.out = (uint32_t*)out;
            ra.nrows = rows << 8;
            ra.lvl = (const uint2*)P->lvl_f1;
            ra.tc = P->tw_f1;
            ra.f = ff;
            return f32::launch_row_fwd(ra, st);
        }
    }
    if (P->k2 == 0) {
        RowArgs<F> a{};
        a.in = in; a.out = out;
        a.nrows = rows;
        a.in_rs = in_rs; a.out_rs = n;
        a.in_len = in_len; a.out_len = n;
        a.k = P->k;
        a.canon = 1;
        a.lvl = (const W*)P->lvl_f1;
        return launch_rows<F, false, T, T>(f, a, st);
    }
    ColArgs<F> c{};
    c.in = in; c.out = out;
    c.ncols = 1ll << P->k1;
    c.nbatch = rows;
    c.in_rs = c.out_rs = 1ll << P->k1;
    c.in_bs = in_rs; c.out_bs = n;
    c.in_len = in_len; c.out_len = n;
    c.n1 = 1ll << P->k1;
    c.k = P->k2;
    c.fs = 1;
    c.lvl = (const W*)P->lvl_f2;
    c.fs_lo = (const W*)P->fs_lo_f;
    c.fs_hi = (const W*)P->fs_hi_f;
    c.fs_full = (const W*)P->fs_full_f;
    c.fs_h = P->fs_h;
    mm_status s = launch_cols<F, false, T, T>(f, c, st);
    if (s != MM_OK) return s;
    RowArgs<F> a{};
    a.in = out; a.out = out;
    a.nrows = rows << P->k2;
    a.in_rs = a.out_rs = 1ll << P->k1;
    a.in_len = a.out_len = 1ll << P->k1;
    a.k = P->k1;
    a.canon = 1;
    a.lvl = (const W*)P->lvl_f1;
    return launch_rows<F, false, T, T>(f, a, st);
}
// BITREV input rows of n (in place allowed for the row pass: `in` is overwritten
// on the four-step path); output row r at out + r out_rs, first out_len
// coefficients, times n^-1, canonical.
template <class F>
static mm_status inv_trunc_impl(mm_ntt_plan* P, void* in, long long rows, void* out, long long out_rs,
                                long long out_len, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    const long long n = 1ll << P->k;
    W sc = host_w<W>(P->ninv, P->p);
    if constexpr (sizeof(T) == 4) {
        if (P->fast16 && ((uintptr_t)in & 15) == 0) {
            const f32::Fld ff{(uint32_t)P->p, 2 * (uint32_t)P->p, P->pinv};
            f32::RowArgs32 ra{};
            ra.in = (const uint32_t*)in; ra.out = (uint32_t*)in;
            ra.nrows = rows << 8;
            ra.lvl = (const uint2*)P->lvl_i1;
            ra.fsi = (const uint2*)P->fs_ni_i;
            ra.tc = P->tw_i1;
            ra.f = ff;
            mm_status s = f32::launch_row_inv(ra, st);
            if (s != MM_OK) return s;
            f32::ColInvArgs ci{};
            ci.in = (const uint32_t*)in; ci.out = (uint32_t*)out;
            ci.nbatch = rows;
            ci.in_bs = n;
            ci.out_bs = out_rs;
            ci.out_len = out_len;
            ci.lvl = (const uint2*)P->lvl_i2;
            ci.tc = P->tw_i2;
            ci.f = ff;
            return f32::launch_col_inv(ci, st);
        }
    }
    if (P->k2 == 0) {
        RowArgs<F> a{};
        a.in = in; a.out = out;
        a.nrows = rows;
        a.in_rs = n; a.out_rs = out_rs;
        a.in_len = n; a.out_len = out_len;
        a.k = P->k;
        a.scale = 1; a.sc = sc;
        a.canon = 1;
        a.lvl = (const W*)P->lvl_i1;
        return launch_rows<F, true, T, T>(f, a, st);
    }
    RowArgs<F> a{};
    a.in = in; a.out = in;
    a.nrows = rows << P->k2;
    a.in_rs = a.out_rs = 1ll << P->k1;
    a.in_len = a.out_len = 1ll << P->k1;
    a.k = P->k1;
    a.fs = 1; a.k2 = P->k2; a.row0 = 0;
    a.lvl = (const W*)P->lvl_i1;
    a.fs_lo = (const W*)P->fs_lo_i;
    a.fs_hi = (const W*)P->fs_hi_i;
    a.fs_full = (const W*)P->fs_full_i;
    a.fs_h = P->fs_h;
    mm_status s = launch_rows<F, true, T, T>(f, a, st);
    if (s != MM_OK) return s;
    ColArgs<F> c{};
    c.in = in; c.out = out;
    c.ncols = 1ll << P->k1;
    c.nbatch = rows;
    c.in_rs = c.out_rs = 1ll << P->k1;
    c.in_bs = n; c.out_bs = out_rs;
    c.in_len = n; c.out_len = out_len;
    c.n1 = 1ll << P->k1;
    c.k = P->k2;
    c.scale = 1; c.sc = sc; c.canon = 1;
    c.lvl = (const W*)P->lvl_i2;
    return launch_cols<F, true, T, T>(f, c, st);
}

// ---- dist building blocks ---------------------------------------------------------
template <class F>
static mm_status fwd_cols_impl(mm_ntt_plan* P, const void* in, void* out, size_t col0, size_t ncols, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    ColArgs<F> c{};
    c.in = in; c.out = out;
    c.ncols = (long long)ncols;
    c.nbatch = 1;
    c.in_rs = c.out_rs = (long long)ncols;
    c.in_bs = c.out_bs = 0;
    c.in_len = c.out_len = 1ll << P->k;
    c.col0 = (long long)col0;
    c.n1 = 1ll << P->k1;
    c.k = P->k2;
    c.fs = 1;
    c.lvl = (const W*)P->lvl_f2;
    c.fs_lo = (const W*)P->fs_lo_f;
    c.fs_hi = (const W*)P->fs_hi_f;
    c.fs_full = (const W*)P->fs_full_f;
    c.fs_h = P->fs_h;
    return launch_cols<F, false, T, T>(f, c, st);
}
template <class F>
static mm_status rows_impl(mm_ntt_plan* P, const void* in, void* out, size_t row0, size_t nrows, bool inv,
                           cudaStream_t st, int seg_log = 0, long long seg_stride = 0) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    RowArgs<F> a{};
    a.in = in; a.out = out;
    a.nrows = (long long)nrows;
    a.in_rs = a.out_rs = 1ll << P->k1;
    // segmented side: forward reads segmented rows, inverse writes them (row stride = segment length)
    if (seg_log) {
        if (!inv) { a.in_seg_log = seg_log; a.in_seg_stride = seg_stride; a.in_rs = 1ll << seg_log; }
        else { a.out_seg_log = seg_log; a.out_seg_stride = seg_stride; a.out_rs = 1ll << seg_log; }
    }
    a.in_len = a.out_len = 1ll << P->k1;
    a.k = P->k1;
    a.row0 = (long long)row0;
    a.k2 = P->k2;
    if (!inv) {
        a.canon = 1;
        a.lvl = (const W*)P->lvl_f1;
        return launch_rows<F, false, T, T>(f, a, st);
    }
    a.fs = 1;
    a.lvl = (const W*)P->lvl_i1;
    a.fs_lo = (const W*)P->fs_lo_i;
    a.fs_hi = (const W*)P->fs_hi_i;
    a.fs_full = (const W*)P->fs_full_i;
    a.fs_h = P->fs_h;
    return launch_rows<F, true, T, T>(f, a, st);
}
template <class F>
static mm_status inv_cols_impl(mm_ntt_plan* P, const void* in, void* out, size_t col0, size_t ncols, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    ColArgs<F> c{};
    c.in = in; c.out = out;
    c.ncols = (long long)ncols;
    c.nbatch = 1;
    c.in_rs = c.out_rs = (long long)ncols;
    c.in_len = c.out_len = 1ll << P->k;
    c.col0 = (long long)col0;
    c.n1 = 1ll << P->k1;
    c.k = P->k2;
    c.scale = 1; c.sc = host_w<W>(P->ninv, P->p); c.canon = 1;
    c.lvl = (const W*)P->lvl_i2;
    return launch_cols<F, true, T, T>(f, c, st);
}

// ---- cached plans + workspaces for poly_mul / int_mul ----------------------------
static std::mutex g_cache_mu;
static std::map<std::tuple<int, uint64_t, int, uint64_t, int>, mm_ntt_plan*> g_plans;   // (bits,p,k,omega,dev)
struct WsKey { int dev; cudaStream_t st; bool operator<(const WsKey& o) const { return dev != o.dev ? dev < o.dev : st < o.st; } };
static std::map<WsKey, std::pair<void*, size_t>> g_ws;

static mm_status cached_plan(int bits, uint64_t p, int k, uint64_t omega, mm_ntt_plan** out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_cache_mu);
    auto key = std::make_tuple(bits, p, k, omega, dev);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) { *out = it->second; return MM_OK; }
    mm_ntt_plan* P = nullptr;
    mm_status s = plan_create(bits, p, k, omega, 1, &P);
    if (s != MM_OK) return s;
    g_plans[key] = P;
    *out = P;
    return MM_OK;
}

static mm_status stream_ws(cudaStream_t st, size_t bytes, void** out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_cache_mu);
    auto& e = g_ws[WsKey{dev, st}];
    if (e.second < bytes) {   // grow in stream order: the old buffer is freed after the work queued on it
        if (e.first) {
            cudaFreeAsync(e.first, st);
            e.first = nullptr;
            e.second = 0;
        }
        MM_CUDA_TRY(alloc_async(&e.first, bytes, st));
        e.second = bytes;
    }
    *out = e.first;
    return MM_OK;
}

// further per-stream workspaces for drivers that call product_impl (which owns
// the first): slot 1 for int_mul_u32 / poly_matmul, slot 2 for int_matmul
struct WsSlotKey {
    int dev, slot;
    cudaStream_t st;
    bool operator<(const WsSlotKey& o) const {
        if (dev != o.dev) return dev < o.dev;
        if (slot != o.slot) return slot < o.slot;
        return st < o.st;
    }
};
static std::map<WsSlotKey, std::pair<void*, size_t>> g_ws_slots;
static mm_status stream_ws_slot(cudaStream_t st, int slot, size_t bytes, void** out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_cache_mu);
    auto& e = g_ws_slots[WsSlotKey{dev, slot, st}];
    if (e.second < bytes) {
        if (e.first) {
            cudaFreeAsync(e.first, st);
            e.first = nullptr;
            e.second = 0;
        }
        MM_CUDA_TRY(alloc_async(&e.first, bytes, st));
        e.second = bytes;
    }
    *out = e.first;
    return MM_OK;
}
static mm_status stream_ws2(cudaStream_t st, size_t bytes, void** out) { return stream_ws_slot(st, 1, bytes, out); }

// n = 2^16 = 256 x 256, p < 2^30: the specialised passes of ntt_fast32.cu
static mm_status fast16_product(mm_ntt_plan* P, const uint32_t* a, long long la, long long lda, const uint32_t* b,
                                long long lb, long long ldb, uint32_t* c, long long lc, long long ldc, long long batch,
                                uint32_t* WA, uint32_t* WB, cudaStream_t st) {
    const f32::Fld f{(uint32_t)P->p, 2 * (uint32_t)P->p, P->pinv};
    const long long n = 1ll << P->k;
    mm_status s;
    for (int op = 0; op < 2; op++) {
        f32::ColFwdArgs cf{};
        cf.in = op == 0 ? a : b;
        cf.out = op == 0 ? WA : WB;
        cf.nbatch = batch;
        cf.in_bs = op == 0 ? lda : ldb;
        cf.in_len = op == 0 ? la : lb;
        cf.out_bs = n;
        cf.lvl = (const uint2*)P->lvl_f2;
        cf.fs = (const uint2*)P->fs_full_f;
        cf.tc = P->tw_f2;
        cf.f = f;
        if ((s = f32::launch_col_fwd(cf, st)) != MM_OK) return s;
    }
    f32::RowPmulArgs rp{};
    rp.A = WA; rp.B = WB; rp.C = WA;
    rp.nrows = batch << P->k2;
    rp.lvl_f = (const uint2*)P->lvl_f1;
    rp.lvl_i = (const uint2*)P->lvl_i1;
    rp.fsi = (const uint2*)P->fs_pm_i;
    rp.tf = P->tw_f1;
    rp.ti = P->tw_i1;
    rp.f = f;
    if ((s = f32::launch_row_pmul(rp, st)) != MM_OK) return s;
    f32::ColInvArgs ci{};
    ci.in = WA; ci.out = c;
    ci.nbatch = batch;
    ci.in_bs = n;
    ci.out_bs = ldc;
    ci.out_len = lc;
    ci.lvl = (const uint2*)P->lvl_i2;
    ci.tc = P->tw_i2;
    ci.f = f;
    return f32::launch_col_inv(ci, st);
}

// c = a * b for `batch` rows; TIn = input element type (uint16 limbs for int_mul)
template <class F, class TIn, class TOut>
static mm_status product_impl(mm_ntt_plan* P, const TIn* a, long long la, const TIn* b, long long lb, TOut* c,
                              long long lc, long long batch, cudaStream_t st, long long lda = -1, long long ldb = -1,
                              long long ldc = -1) {
    if (lda < 0) lda = la;
    if (ldb < 0) ldb = lb;
    if (ldc < 0) ldc = lc;
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    W sc = host_w<W>(P->ninv_r, P->p);   // n^-1 (x 2^32 for the 32-bit REDC product)
    if (P->k2 == 0) {
        PmulArgs<F> m{};
        m.a = a; m.b = b; m.c = c;
        m.nrows = batch;
        m.a_rs = lda; m.b_rs = ldb; m.c_rs = ldc;
        m.la = la; m.lb = lb; m.lc = lc;
        m.k = P->k;
        m.sc = sc;
        m.canon = 1;
        m.lvl_f = (const W*)P->lvl_f1;
        m.lvl_i = (const W*)P->lvl_i1;
        return launch_pmul<F, TIn, TOut>(f, m, st);
    }
    const long long n = 1ll << P->k, n1 = 1ll << P->k1;
    if constexpr (sizeof(T) == 4 && sizeof(TIn) == 4 && sizeof(TOut) == 4) {
        if (P->fast16) {
            // Large batches run as sub-batches on the library's fork streams
            // (forked from and joined back into `st` by events): one
            // sub-batch's HBM-heavy column passes overlap another's ALU-bound
            // product rows, and each kernel's tail overlaps the other stream's
            // work (C3: 2.21 -> 2.08 ms on B200, tools/exp_streams.py)
            const int ns = product_streams();
            if (ns > 1 && batch >= 128 * ns) {
                Fork* FK = nullptr;
                mm_status s = fork_streams(&FK);
                if (s != MM_OK) return s;
                std::lock_guard<std::mutex> lk(FK->mu);
                MM_CUDA_TRY(cudaEventRecord(FK->fork, st));
                long long r0 = 0;
                for (int h = 0; h < ns; h++) {
                    const long long rows = batch / ns + (h < batch % ns ? 1 : 0);
                    MM_CUDA_TRY(cudaStreamWaitEvent(FK->s[h], FK->fork, 0));
                    void* wsh = nullptr;
                    if ((s = stream_ws(FK->s[h], (size_t)(2 * n * rows) * sizeof(T), &wsh)) != MM_OK) return s;
                    if ((s = fast16_product(P, (const uint32_t*)a + r0 * lda, la, lda, (const uint32_t*)b + r0 * ldb, lb,
                                            ldb, (uint32_t*)c + r0 * ldc, lc, ldc, rows, (uint32_t*)wsh,
                                            (uint32_t*)wsh + n * rows, FK->s[h])) != MM_OK)
                        return s;
                    MM_CUDA_TRY(cudaEventRecord(FK->join[h], FK->s[h]));
                    MM_CUDA_TRY(cudaStreamWaitEvent(st, FK->join[h], 0));
                    r0 += rows;
                }
                return MM_OK;
            }
            void* ws = nullptr;
            mm_status s = stream_ws(st, (size_t)(2 * n * batch) * sizeof(T), &ws);
            if (s != MM_OK) return s;
            return fast16_product(P, (const uint32_t*)a, la, lda, (const uint32_t*)b, lb, ldb, (uint32_t*)c, lc, ldc,
                                  batch, (uint32_t*)ws, (uint32_t*)ws + n * batch, st);
        }
    }
    void* ws = nullptr;
    mm_status s = stream_ws(st, (size_t)(2 * n * batch) * sizeof(T), &ws);
    if (s != MM_OK) return s;
    T* WA = (T*)ws;
    T* WB = WA + n * batch;
    // forward column passes (steps 1-2) for a and b, zero padding beyond la / lb;
    // 64-bit products: a's and b's passes on the two fork streams (concurrent)
    const bool fork2 = sizeof(T) == 8 && product_streams() > 1;
    Fork* FK = nullptr;
    std::unique_lock<std::mutex> flk;
    if (fork2) {
        if ((s = fork_streams(&FK)) != MM_OK) return s;
        flk = std::unique_lock<std::mutex>(FK->mu);
        MM_CUDA_TRY(cudaEventRecord(FK->fork, st));
    }
    for (int op = 0; op < 2; op++) {
        cudaStream_t cs = st;
        if (fork2) {
            cs = FK->s[op];
            MM_CUDA_TRY(cudaStreamWaitEvent(cs, FK->fork, 0));
        }
        ColArgs<F> cc{};
        cc.in = op == 0 ? (const void*)a : (const void*)b;
        cc.out = op == 0 ? WA : WB;
        cc.ncols = n1;
        cc.nbatch = batch;
        cc.in_rs = n1; cc.out_rs = n1;
        cc.in_bs = op == 0 ? lda : ldb; cc.out_bs = n;
        cc.in_len = op == 0 ? la : lb; cc.out_len = n;
        cc.n1 = n1;
        cc.k = P->k2;
        cc.fs = 1;
        cc.lvl = (const W*)P->lvl_f2;
        cc.fs_lo = (const W*)P->fs_lo_f;
        cc.fs_hi = (const W*)P->fs_hi_f;
        cc.fs_full = (const W*)P->fs_full_f;
        cc.fs_h = P->fs_h;
        if ((s = launch_cols<F, false, TIn, T>(f, cc, cs)) != MM_OK) return s;
        if (fork2) {
            MM_CUDA_TRY(cudaEventRecord(FK->join[op], cs));
            MM_CUDA_TRY(cudaStreamWaitEvent(st, FK->join[op], 0));
        }
    }
    if (fork2) flk.unlock();
    // fused row pass: steps 3-4 for both, pointwise product * n^-1, inverse step 4-3, inverse twiddle
    PmulArgs<F> m{};
    m.a = WA; m.b = WB; m.c = WA;
    m.nrows = batch << P->k2;
    m.a_rs = m.b_rs = m.c_rs = n1;
    m.la = m.lb = m.lc = n1;
    m.k = P->k1;
    m.fs = 1; m.k2 = P->k2; m.row0 = 0;
    m.sc = sc;
    m.lvl_f = (const W*)P->lvl_f1;
    m.lvl_i = (const W*)P->lvl_i1;
    m.fs_lo = (const W*)P->fs_lo_i;
    m.fs_hi = (const W*)P->fs_hi_i;
    m.fs_full = (const W*)P->fs_full_i;
    m.fs_h = P->fs_h;
    if ((s = launch_pmul<F, T, T>(f, m, st)) != MM_OK) return s;
    // inverse column pass (step 1 inverse), canonical, truncated to lc
    ColArgs<F> ci{};
    ci.in = WA; ci.out = c;
    ci.ncols = n1;
    ci.nbatch = batch;
    ci.in_rs = n1; ci.out_rs = n1;
    ci.in_bs = n; ci.out_bs = ldc;
    ci.in_len = n; ci.out_len = lc;
    ci.n1 = n1;
    ci.k = P->k2;
    ci.canon = 1;
    ci.lvl = (const W*)P->lvl_i2;
    return launch_cols<F, true, T, TOut>(f, ci, st);
}

// Remark 6: the three products of the three-prime method in one
// launch per pass -- row q of every batched operand is reduced mod p_q, with
// p_q's field constants and tables selected per tile.  R = residues [3][rs]
// (a at offset 0, b at offset na), Cp = products [3][lc]; the three plans
// share k (hence the split and the table geometry).
static mm_status product3_impl(mm_ntt_plan* const PL[3], const uint32_t* A, const uint32_t* B, const Crt3& K,
                               uint32_t* R, long long rs, long long na, long long nb, uint32_t* Cp, long long lc,
                               cudaStream_t st) {
    typedef uint2 W;
    mm_ntt_plan* P = PL[0];
    Fp32 f = make_field<Fp32>(P);
    const int rgrid = num_sms() * 8;
    // residues of operand op modulo the three primes -> R (a at 0, b at na)
    auto residues = [&](int op, cudaStream_t cs) -> mm_status {
        {
            LaunchScope ls("crt_residues", cs);
            k_residues3<<<rgrid, 256, 0, cs>>>(op ? B : A, op ? nb : na, R + (op ? na : 0), rs, K);
        }
        MM_LAUNCH_CHECK();
        return MM_OK;
    };
    if (P->k2 == 0) {
        for (int op = 0; op < 2; op++) {
            mm_status s = residues(op, st);
            if (s != MM_OK) return s;
        }
        // one-pass products: a product tile holds several rows, which would mix
        // moduli -- one launch per prime (these sizes are launch-latency bound)
        for (int q = 0; q < 3; q++) {
            mm_status s = product_impl<Fp32, uint32_t, uint32_t>(PL[q], R + q * rs, na, R + q * rs + na, nb, Cp + q * lc,
                                                                 lc, 1, st);
            if (s != MM_OK) return s;
        }
        return MM_OK;
    }
    const long long n = 1ll << P->k, n1 = 1ll << P->k1;
    void* ws = nullptr;
    mm_status s = stream_ws(st, (size_t)(6 * n) * sizeof(uint32_t), &ws);
    if (s != MM_OK) return s;
    uint32_t* WA = (uint32_t*)ws;
    uint32_t* WB = WA + 3 * n;
    // a's and b's forward column passes on the two fork streams: at Table-16
    // sizes each launch is a wave or two, so the two overlap
    const bool fork2 = product_streams() > 1;
    Fork* FK = nullptr;
    std::unique_lock<std::mutex> flk;
    if (fork2) {
        if ((s = fork_streams(&FK)) != MM_OK) return s;
        flk = std::unique_lock<std::mutex>(FK->mu);
        MM_CUDA_TRY(cudaEventRecord(FK->fork, st));
    }
    for (int op = 0; op < 2; op++) {
        cudaStream_t cs = st;
        if (fork2) {
            cs = FK->s[op];
            MM_CUDA_TRY(cudaStreamWaitEvent(cs, FK->fork, 0));
        }
        ColArgs<Fp32> cc{};
        // the raw 32-bit limbs, reduced modulo p_q by the loader of batch row q
        cc.in = op == 0 ? (const void*)A : (const void*)B;
        cc.reduce_in = 1;
        cc.out = op == 0 ? WA : WB;
        cc.ncols = n1;
        cc.nbatch = 3;
        cc.in_rs = n1; cc.out_rs = n1;
        cc.in_bs = 0; cc.out_bs = n;
        cc.in_len = op == 0 ? na : nb; cc.out_len = n;
        cc.n1 = n1;
        cc.k = P->k2;
        cc.fs = 1;
        cc.lvl = (const W*)P->lvl_f2;
        cc.fs_lo = (const W*)P->fs_lo_f;
        cc.fs_hi = (const W*)P->fs_hi_f;
        cc.fs_full = (const W*)P->fs_full_f;
        cc.fs_h = P->fs_h;
        cc.nmod = 3;
        cc.mod_span = 1;
        for (int q = 0; q < 3; q++) {
            cc.fm[q] = make_field<Fp32>(PL[q]);
            cc.lvlm[q] = (const W*)PL[q]->lvl_f2;
            cc.fslom[q] = (const W*)PL[q]->fs_lo_f;
            cc.fshim[q] = (const W*)PL[q]->fs_hi_f;
            cc.fsfullm[q] = (const W*)PL[q]->fs_full_f;
        }
        if ((s = launch_cols<Fp32, false, uint32_t, uint32_t>(f, cc, cs)) != MM_OK) return s;
        if (fork2) {
            MM_CUDA_TRY(cudaEventRecord(FK->join[op], cs));
            MM_CUDA_TRY(cudaStreamWaitEvent(st, FK->join[op], 0));
        }
    }
    if (fork2) flk.unlock();
    PmulArgs<Fp32> m{};
    m.a = WA; m.b = WB; m.c = WA;
    m.nrows = 3ll << P->k2;
    m.a_rs = m.b_rs = m.c_rs = n1;
    m.la = m.lb = m.lc = n1;
    m.k = P->k1;
    m.fs = 1; m.k2 = P->k2; m.row0 = 0;
    m.sc = host_w<W>(P->ninv_r, P->p);
    m.lvl_f = (const W*)P->lvl_f1;
    m.lvl_i = (const W*)P->lvl_i1;
    m.fs_lo = (const W*)P->fs_lo_i;
    m.fs_hi = (const W*)P->fs_hi_i;
    m.fs_full = (const W*)P->fs_full_i;
    m.fs_h = P->fs_h;
    m.nmod = 3;
    m.mod_span = 1ll << P->k2;
    for (int q = 0; q < 3; q++) {
        m.fm[q] = make_field<Fp32>(PL[q]);
        m.scm[q] = host_w<W>(PL[q]->ninv_r, PL[q]->p);
        m.lvlfm[q] = (const W*)PL[q]->lvl_f1;
        m.lvlim[q] = (const W*)PL[q]->lvl_i1;
        m.fslom[q] = (const W*)PL[q]->fs_lo_i;
        m.fshim[q] = (const W*)PL[q]->fs_hi_i;
        m.fsfullm[q] = (const W*)PL[q]->fs_full_i;
    }
    if ((s = launch_pmul<Fp32, uint32_t, uint32_t>(f, m, st)) != MM_OK) return s;
    ColArgs<Fp32> ci{};
    ci.in = WA; ci.out = Cp;
    ci.ncols = n1;
    ci.nbatch = 3;
    ci.in_rs = n1; ci.out_rs = n1;
    ci.in_bs = n; ci.out_bs = lc;
    ci.in_len = n; ci.out_len = lc;
    ci.n1 = n1;
    ci.k = P->k2;
    ci.canon = 1;
    ci.lvl = (const W*)P->lvl_i2;
    ci.nmod = 3;
    ci.mod_span = 1;
    for (int q = 0; q < 3; q++) {
        ci.fm[q] = make_field<Fp32>(PL[q]);
        ci.lvlm[q] = (const W*)PL[q]->lvl_i2;
    }
    return launch_cols<Fp32, true, uint32_t, uint32_t>(f, ci, st);
}

}  // namespace mm

// ====================================================================== C ABI
extern "C" mm_status mm_ntt_plan_create(int word_bits, uint64_t p, int log2n, uint64_t omega, size_t batch,
                                        mm_ntt_plan** plan) {
    if (!plan) return set_err(MM_E_ARG, "plan is null");
    *plan = nullptr;
    if (batch == 0) return set_err(MM_E_ARG, "batch must be >= 1");
    return plan_create(word_bits, p, log2n, omega, batch, plan);
}

extern "C" void mm_ntt_plan_destroy(mm_ntt_plan* plan) {
    if (plan) cudaDeviceSynchronize();
    free_plan(plan);
}

extern "C" mm_status mm_ntt_plan_info(const mm_ntt_plan* P, uint64_t out[6]) {
    if (!P || !out) return set_err(MM_E_ARG, "null argument");
    out[0] = 1ull << P->k1;
    out[1] = 1ull << P->k2;
    out[2] = P->k2 ? 2 : 1;
    out[3] = 0;                 // workspaces are stream-ordered allocations (none held by the plan)
    out[4] = (uint64_t)P->word_bits;
    out[5] = (uint64_t)P->batch;
    return MM_OK;
}

extern "C" mm_status mm_ntt_forward(const mm_ntt_plan* plan, const void* in, void* out, mm_order order, void* stream) {
    if (!plan || !in || !out) return set_err(MM_E_ARG, "null argument");
    if (order != MM_ORDER_NATURAL && order != MM_ORDER_BITREV) return set_err(MM_E_ARG, "bad order");
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    if (debug_checks()) {
        mm_status s = check_rows(in, P->word_bits, P->batch, 1ull << P->k, 1ull << P->k, P->p, st);
        if (s != MM_OK) return s;
    }
    if (P->word_bits == 52) return fwd_impl<FpD>(P, in, out, order, st);
    return P->word_bits == 32 ? fwd_impl<Fp32>(P, in, out, order, st) : fwd_impl<FpG>(P, in, out, order, st);
}

extern "C" mm_status mm_ntt_inverse(const mm_ntt_plan* plan, const void* in, void* out, mm_order order, void* stream) {
    if (!plan || !in || !out) return set_err(MM_E_ARG, "null argument");
    if (order != MM_ORDER_NATURAL && order != MM_ORDER_BITREV) return set_err(MM_E_ARG, "bad order");
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    if (debug_checks()) {
        mm_status s = check_rows(in, P->word_bits, P->batch, 1ull << P->k, 1ull << P->k, P->p, st);
        if (s != MM_OK) return s;
    }
    if (P->word_bits == 52) return inv_impl<FpD>(P, in, out, order, st);
    return P->word_bits == 32 ? inv_impl<Fp32>(P, in, out, order, st) : inv_impl<FpG>(P, in, out, order, st);
}

static mm_status dist_check(const mm_ntt_plan* P, const void* in, void* out, size_t off, size_t cnt, bool cols) {
    if (!P || !in || !out) return set_err(MM_E_ARG, "null argument");
    if (P->k2 == 0) return set_err(MM_E_UNSUPPORTED_SIZE, "four-step blocks need a two-pass plan (log2n > %d)",
                                   onepass_log(P->word_bits));
    if (P->word_bits == 52) return set_err(MM_E_ARG, "four-step blocks are built for 32- and 64-bit plans");
    size_t lim = cols ? (1ull << P->k1) : (1ull << P->k2);
    if (cnt == 0 || off + cnt > lim) return set_err(MM_E_ARG, "block [%zu, %zu) out of range %zu", off, off + cnt, lim);
    return MM_OK;
}

extern "C" mm_status mm_ntt_fwd_cols(const mm_ntt_plan* plan, const void* in, void* out, size_t col0, size_t ncols,
                                     void* stream) {
    mm_status s = dist_check(plan, in, out, col0, ncols, true);
    if (s != MM_OK) return s;
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    return P->word_bits == 32 ? fwd_cols_impl<Fp32>(P, in, out, col0, ncols, st)
                              : fwd_cols_impl<FpG>(P, in, out, col0, ncols, st);
}
extern "C" mm_status mm_ntt_fwd_rows(const mm_ntt_plan* plan, const void* in, void* out, size_t row0, size_t nrows,
                                     void* stream) {
    mm_status s = dist_check(plan, in, out, row0, nrows, false);
    if (s != MM_OK) return s;
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    return P->word_bits == 32 ? rows_impl<Fp32>(P, in, out, row0, nrows, false, st)
                              : rows_impl<FpG>(P, in, out, row0, nrows, false, st);
}
extern "C" mm_status mm_ntt_inv_rows(const mm_ntt_plan* plan, const void* in, void* out, size_t row0, size_t nrows,
                                     void* stream) {
    mm_status s = dist_check(plan, in, out, row0, nrows, false);
    if (s != MM_OK) return s;
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    return P->word_bits == 32 ? rows_impl<Fp32>(P, in, out, row0, nrows, true, st)
                              : rows_impl<FpG>(P, in, out, row0, nrows, true, st);
}
extern "C" mm_status mm_ntt_inv_cols(const mm_ntt_plan* plan, const void* in, void* out, size_t col0, size_t ncols,
                                     void* stream) {
    mm_status s = dist_check(plan, in, out, col0, ncols, true);
    if (s != MM_OK) return s;
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    return P->word_bits == 32 ? inv_cols_impl<Fp32>(P, in, out, col0, ncols, st)
                              : inv_cols_impl<FpG>(P, in, out, col0, ncols, st);
}

static mm_status seg_check(const mm_ntt_plan* P, size_t seg_len, size_t seg_stride, size_t nrows, int* seg_log) {
    int l = 0;
    while ((1ull << l) < seg_len) l++;
    if (seg_len == 0 || (1ull << l) != seg_len || seg_len > (1ull << P->k1) || ((1ull << P->k1) % seg_len) != 0)
        return set_err(MM_E_ARG, "segment length %zu must be a power of two dividing n1", seg_len);
    if (seg_stride < nrows * seg_len) return set_err(MM_E_ARG, "segment stride %zu < rows x segment length", seg_stride);
    *seg_log = l;
    return MM_OK;
}

extern "C" mm_status mm_ntt_fwd_rows_seg(const mm_ntt_plan* plan, const void* in, void* out, size_t row0, size_t nrows,
                                         size_t in_seg_len, size_t in_seg_stride, void* stream) {
    mm_status s = dist_check(plan, in, out, row0, nrows, false);
    if (s != MM_OK) return s;
    int sl = 0;
    if ((s = seg_check(plan, in_seg_len, in_seg_stride, nrows, &sl)) != MM_OK) return s;
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    return P->word_bits == 32 ? rows_impl<Fp32>(P, in, out, row0, nrows, false, st, sl, (long long)in_seg_stride)
                              : rows_impl<FpG>(P, in, out, row0, nrows, false, st, sl, (long long)in_seg_stride);
}
extern "C" mm_status mm_ntt_inv_rows_seg(const mm_ntt_plan* plan, const void* in, void* out, size_t row0, size_t nrows,
                                         size_t out_seg_len, size_t out_seg_stride, void* stream) {
    mm_status s = dist_check(plan, in, out, row0, nrows, false);
    if (s != MM_OK) return s;
    int sl = 0;
    if ((s = seg_check(plan, out_seg_len, out_seg_stride, nrows, &sl)) != MM_OK) return s;
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    return P->word_bits == 32 ? rows_impl<Fp32>(P, in, out, row0, nrows, true, st, sl, (long long)out_seg_stride)
                              : rows_impl<FpG>(P, in, out, row0, nrows, true, st, sl, (long long)out_seg_stride);
}

static bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

extern "C" mm_status mm_poly_mul_ld(int word_bits, uint64_t p, uint64_t g, const void* a, size_t la, size_t lda,
                                    const void* b, size_t lb, size_t ldb, void* c, size_t ldc, size_t batch,
                                    void* stream) {
    if (!a || !b || !c) return set_err(MM_E_ARG, "null argument");
    if (la == 0 || lb == 0 || batch == 0) return set_err(MM_E_ARG, "empty operands");
    size_t lc = la + lb - 1;
    if (lda < la || ldb < lb || ldc < lc) return set_err(MM_E_ARG, "leading dimension smaller than the row length");
    size_t es = esize(word_bits);
    const size_t ea = ((batch - 1) * lda + la) * es, eb = ((batch - 1) * ldb + lb) * es, ec = ((batch - 1) * ldc + lc) * es;
    if (overlaps(a, ea, c, ec) || overlaps(b, eb, c, ec)) return set_err(MM_E_ALIAS, "c aliases a or b");
    int k = 0;
    while ((1ull << k) < lc) k++;
    if (k == 0) k = 1;
    mm_status s = check_modulus(word_bits, p, k);
    if (s != MM_OK) return s;
    uint64_t omega = hpowmod(g % p, (p - 1) >> k, p);
    mm_ntt_plan* P = nullptr;
    if ((s = cached_plan(word_bits, p, k, omega, &P)) != MM_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if (debug_checks()) {
        if ((s = check_rows(a, word_bits, batch, la, lda, p, st)) != MM_OK) return s;
        if ((s = check_rows(b, word_bits, batch, lb, ldb, p, st)) != MM_OK) return s;
    }
    if (word_bits == 32)
        return product_impl<Fp32, uint32_t, uint32_t>(P, (const uint32_t*)a, (long long)la, (const uint32_t*)b,
                                                      (long long)lb, (uint32_t*)c, (long long)lc, (long long)batch, st,
                                                      (long long)lda, (long long)ldb, (long long)ldc);
    if (word_bits == 52)
        return product_impl<FpD, double, double>(P, (const double*)a, (long long)la, (const double*)b, (long long)lb,
                                                 (double*)c, (long long)lc, (long long)batch, st, (long long)lda,
                                                 (long long)ldb, (long long)ldc);
    return product_impl<FpG, uint64_t, uint64_t>(P, (const uint64_t*)a, (long long)la, (const uint64_t*)b, (long long)lb,
                                                 (uint64_t*)c, (long long)lc, (long long)batch, st, (long long)lda,
                                                 (long long)ldb, (long long)ldc);
}

extern "C" mm_status mm_poly_mul(int word_bits, uint64_t p, uint64_t g, const void* a, size_t la, const void* b,
                                 size_t lb, void* c, size_t batch, void* stream) {
    return mm_poly_mul_ld(word_bits, p, g, a, la, la, b, lb, lb, c, la + lb - 1, batch, stream);
}

// ---- host-buffer product: chunked H2D / compute / D2H pipeline -------------------
// Three device slots; H2D and D2H on their own streams, the products on the
// caller's stream, events between them, so chunk i+1 uploads and chunk i-1
// downloads while chunk i computes.  Device output rows use a 128-byte
// leading dimension; the D2H copy packs them (cudaMemcpy2DAsync).  Measured
// (tools/time_e2e.py, r12): 25.4-29.2 ms per C3 step for chunk sizes 48-128
// MiB, packed or aligned rows, with run-to-run spread larger than any
// setting's effect, against a 21.6 ms concurrent copy floor (pcie_probe).
struct HostPipe {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t in[3], done[3], freed[3];
    bool used[3] = {false, false, false};
    int next = 0;            // slot of the next chunk: the rotation continues across calls
    void* buf = nullptr;
    size_t bytes = 0;
    size_t layout = 0;       // slot size of the last call (slot k = buf + k layout)
    std::mutex mu;
};
static std::mutex g_pipe_mu;
static std::map<int, HostPipe*> g_pipes;

static mm_status host_pipe(HostPipe** out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_pipe_mu);
    HostPipe*& P = g_pipes[dev];
    if (!P) {
        HostPipe* h = new (std::nothrow) HostPipe;
        if (!h) return set_err(MM_E_ARG, "out of host memory");
        MM_CUDA_TRY(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
        MM_CUDA_TRY(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 3; i++) {
            MM_CUDA_TRY(cudaEventCreateWithFlags(&h->in[i], cudaEventDisableTiming));
            MM_CUDA_TRY(cudaEventCreateWithFlags(&h->done[i], cudaEventDisableTiming));
            MM_CUDA_TRY(cudaEventCreateWithFlags(&h->freed[i], cudaEventDisableTiming));
        }
        P = h;
    }
    *out = P;
    return MM_OK;
}

// Three slots of slot_bytes each.  When the slot size differs from the last
// call's, the new slots overlap other old ones, so the upload stream first
// waits for every pending download (otherwise only for its own slot's).
static mm_status pipe_reserve(HostPipe* H, size_t slot_bytes) {
    if (H->bytes < 3 * slot_bytes) {
        MM_CUDA_TRY(cudaDeviceSynchronize());
        if (H->buf) cudaFree(H->buf);
        H->buf = nullptr;
        H->bytes = 0;
        MM_CUDA_TRY(cudaMalloc(&H->buf, 3 * slot_bytes));
        H->bytes = 3 * slot_bytes;
        for (int i = 0; i < 3; i++) H->used[i] = false;
        H->next = 0;
    } else if (H->layout != slot_bytes) {
        for (int i = 0; i < 3; i++)
            if (H->used[i]) MM_CUDA_TRY(cudaStreamWaitEvent(H->h2d, H->freed[i], 0));
    }
    H->layout = slot_bytes;
    return MM_OK;
}

extern "C" mm_status mm_poly_mul_host(int word_bits, uint64_t p, uint64_t g, const void* a, size_t la, const void* b,
                                      size_t lb, void* c, size_t batch, void* stream) {
    if (!a || !b || !c) return set_err(MM_E_ARG, "null argument");
    if (la == 0 || lb == 0 || batch == 0) return set_err(MM_E_ARG, "empty operands");
    if (word_bits != 32 && word_bits != 64 && word_bits != 52) return set_err(MM_E_ARG, "word_bits must be 32, 64 or 52");
    const size_t es = esize(word_bits), lc = la + lb - 1;
    // MMNTT_HOST_PACKED=1: device output rows packed at lc (one 1-D download per
    // chunk) instead of 128-byte aligned rows (2-D download); MMNTT_HOST_CHUNK_MIB:
    // device traffic per chunk (default 96)
    static const bool packed = getenv("MMNTT_HOST_PACKED") && atoi(getenv("MMNTT_HOST_PACKED")) != 0;
    static const size_t chunk_mib = getenv("MMNTT_HOST_CHUNK_MIB") ? (size_t)atoi(getenv("MMNTT_HOST_CHUNK_MIB")) : 96;
    const size_t q = 128 / es, ldc = packed ? lc : (lc + q - 1) / q * q;
    const size_t per = (la + lb + ldc) * es;
    size_t ch = ((chunk_mib ? chunk_mib : 96) << 20) / per;   // device traffic per chunk
    if (ch < 1) ch = 1;
    if (ch > batch) ch = batch;
    HostPipe* H = nullptr;
    mm_status s = host_pipe(&H);
    if (s != MM_OK) return s;
    std::lock_guard<std::mutex> lk(H->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t slot_bytes = ch * per;
    if ((s = pipe_reserve(H, slot_bytes)) != MM_OK) return s;
    const size_t nch = (batch + ch - 1) / ch;
    int last = 0;
    for (size_t i = 0; i < nch; i++) {
        // slots rotate across calls too, so the next call's first upload waits
        // for the download of this call's third-to-last chunk, not its last
        const int k = (int)((H->next + i) % 3);
        const size_t r0 = i * ch, rows = batch - r0 < ch ? batch - r0 : ch;
        char* base = (char*)H->buf + k * slot_bytes;
        char* da = base;
        char* db = da + ch * la * es;
        char* dc = db + ch * lb * es;
        if (H->used[k]) MM_CUDA_TRY(cudaStreamWaitEvent(H->h2d, H->freed[k], 0));
        MM_CUDA_TRY(cudaMemcpyAsync(da, (const char*)a + r0 * la * es, rows * la * es, cudaMemcpyHostToDevice, H->h2d));
        MM_CUDA_TRY(cudaMemcpyAsync(db, (const char*)b + r0 * lb * es, rows * lb * es, cudaMemcpyHostToDevice, H->h2d));
        MM_CUDA_TRY(cudaEventRecord(H->in[k], H->h2d));
        MM_CUDA_TRY(cudaStreamWaitEvent(st, H->in[k], 0));
        if ((s = mm_poly_mul_ld(word_bits, p, g, da, la, la, db, lb, lb, dc, ldc, rows, stream)) != MM_OK) return s;
        MM_CUDA_TRY(cudaEventRecord(H->done[k], st));
        MM_CUDA_TRY(cudaStreamWaitEvent(H->d2h, H->done[k], 0));
        if (ldc == lc)
            MM_CUDA_TRY(cudaMemcpyAsync((char*)c + r0 * lc * es, dc, rows * lc * es, cudaMemcpyDeviceToHost, H->d2h));
        else
            MM_CUDA_TRY(cudaMemcpy2DAsync((char*)c + r0 * lc * es, lc * es, dc, ldc * es, lc * es, rows,
                                          cudaMemcpyDeviceToHost, H->d2h));
        MM_CUDA_TRY(cudaEventRecord(H->freed[k], H->d2h));
        H->used[k] = true;
        last = k;
    }
    H->next = (int)((H->next + nch) % 3);
    // the caller's stream is ordered after the last download
    MM_CUDA_TRY(cudaStreamWaitEvent(st, H->freed[last], 0));
    return MM_OK;
}

// ---- host-buffer transforms: the same three-slot pipeline over batch rows ---------
static mm_status ntt_host(const mm_ntt_plan* plan, const void* in, void* out, mm_order order, void* stream, bool inverse) {
    if (!plan || !in || !out) return set_err(MM_E_ARG, "null argument");
    if (order != MM_ORDER_NATURAL && order != MM_ORDER_BITREV) return set_err(MM_E_ARG, "bad order");
    static const size_t chunk_mib = getenv("MMNTT_HOST_CHUNK_MIB") ? (size_t)atoi(getenv("MMNTT_HOST_CHUNK_MIB")) : 96;
    const size_t es = esize(plan->word_bits), row = (es << plan->k), batch = plan->batch;
    size_t ch = ((chunk_mib ? chunk_mib : 96) << 20) / (2 * row);   // device traffic per chunk
    if (ch < 1) ch = 1;
    if (ch > batch) ch = batch;
    HostPipe* H = nullptr;
    mm_status s = host_pipe(&H);
    if (s != MM_OK) return s;
    std::lock_guard<std::mutex> lk(H->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t slot_bytes = 2 * ch * row;
    if ((s = pipe_reserve(H, slot_bytes)) != MM_OK) return s;
    const size_t nch = (batch + ch - 1) / ch;
    mm_ntt_plan Q = *plan;   // the tables do not depend on the batch: a chunk runs on a copy with its row count
    int last = 0;
    for (size_t i = 0; i < nch; i++) {
        const int k = (int)((H->next + i) % 3);
        const size_t r0 = i * ch, rows = batch - r0 < ch ? batch - r0 : ch;
        char* din = (char*)H->buf + k * slot_bytes;
        char* dout = din + ch * row;
        if (H->used[k]) MM_CUDA_TRY(cudaStreamWaitEvent(H->h2d, H->freed[k], 0));
        MM_CUDA_TRY(cudaMemcpyAsync(din, (const char*)in + r0 * row, rows * row, cudaMemcpyHostToDevice, H->h2d));
        MM_CUDA_TRY(cudaEventRecord(H->in[k], H->h2d));
        MM_CUDA_TRY(cudaStreamWaitEvent(st, H->in[k], 0));
        Q.batch = rows;
        s = inverse ? mm_ntt_inverse(&Q, din, dout, order, stream) : mm_ntt_forward(&Q, din, dout, order, stream);
        if (s != MM_OK) return s;
        MM_CUDA_TRY(cudaEventRecord(H->done[k], st));
        MM_CUDA_TRY(cudaStreamWaitEvent(H->d2h, H->done[k], 0));
        MM_CUDA_TRY(cudaMemcpyAsync((char*)out + r0 * row, dout, rows * row, cudaMemcpyDeviceToHost, H->d2h));
        MM_CUDA_TRY(cudaEventRecord(H->freed[k], H->d2h));
        H->used[k] = true;
        last = k;
    }
    H->next = (int)((H->next + nch) % 3);
    MM_CUDA_TRY(cudaStreamWaitEvent(st, H->freed[last], 0));
    return MM_OK;
}

extern "C" mm_status mm_ntt_forward_host(const mm_ntt_plan* plan, const void* in, void* out, mm_order order, void* stream) {
    return ntt_host(plan, in, out, order, stream, false);
}

extern "C" mm_status mm_ntt_inverse_host(const mm_ntt_plan* plan, const void* in, void* out, mm_order order, void* stream) {
    return ntt_host(plan, in, out, order, stream, true);
}

// ---- host-buffer elementwise operations: chunks of the vectors through the same slots
extern "C" mm_status mm_modop_u32_host(const mm_mod32* ctx, mm_host_op op, const uint32_t* x, const uint32_t* y,
                                       const uint32_t* y_shoup, uint32_t* z, size_t n, void* stream) {
    if (!ctx) return set_err(MM_E_ARG, "null context");
    if (op < MM_OP_ADD || op > MM_OP_MUL_MONTGOMERY) return set_err(MM_E_ARG, "bad operation");
    if (n == 0) return MM_OK;
    if (!x || !y || !z) return set_err(MM_E_ARG, "null argument");
    const bool shoup = op == MM_OP_MUL_SHOUP;
    if (shoup && !y_shoup) return set_err(MM_E_ARG, "SHOUP needs y_shoup");
    static const size_t chunk_mib = getenv("MMNTT_HOST_CHUNK_MIB") ? (size_t)atoi(getenv("MMNTT_HOST_CHUNK_MIB")) : 96;
    const size_t arrays = shoup ? 4 : 3;
    size_t ch = ((chunk_mib ? chunk_mib : 96) << 20) / (arrays * 4) & ~(size_t)3;   // elements per chunk, 16-byte multiples
    if (ch < 4) ch = 4;
    if (ch > n) ch = (n + 3) & ~(size_t)3;
    HostPipe* H = nullptr;
    mm_status s = host_pipe(&H);
    if (s != MM_OK) return s;
    std::lock_guard<std::mutex> lk(H->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t slot_bytes = arrays * ch * 4;
    if ((s = pipe_reserve(H, slot_bytes)) != MM_OK) return s;
    const size_t nch = (n + ch - 1) / ch;
    int last = 0;
    for (size_t i = 0; i < nch; i++) {
        const int k = (int)((H->next + i) % 3);
        const size_t e0 = i * ch, cnt = n - e0 < ch ? n - e0 : ch;
        uint32_t* dx = (uint32_t*)((char*)H->buf + k * slot_bytes);
        uint32_t* dy = dx + ch;
        uint32_t* dz = dy + ch;
        uint32_t* dys = dz + ch;
        if (H->used[k]) MM_CUDA_TRY(cudaStreamWaitEvent(H->h2d, H->freed[k], 0));
        MM_CUDA_TRY(cudaMemcpyAsync(dx, x + e0, cnt * 4, cudaMemcpyHostToDevice, H->h2d));
        MM_CUDA_TRY(cudaMemcpyAsync(dy, y + e0, cnt * 4, cudaMemcpyHostToDevice, H->h2d));
        if (shoup) MM_CUDA_TRY(cudaMemcpyAsync(dys, y_shoup + e0, cnt * 4, cudaMemcpyHostToDevice, H->h2d));
        MM_CUDA_TRY(cudaEventRecord(H->in[k], H->h2d));
        MM_CUDA_TRY(cudaStreamWaitEvent(st, H->in[k], 0));
        if (op == MM_OP_ADD) s = mm_modadd_u32(ctx, dx, dy, dz, cnt, stream);
        else if (op == MM_OP_SUB) s = mm_modsub_u32(ctx, dx, dy, dz, cnt, stream);
        else s = mm_modmul_u32(ctx, op == MM_OP_MUL_BARRETT ? MM_MUL_BARRETT : shoup ? MM_MUL_SHOUP : MM_MUL_MONTGOMERY,
                               dx, dy, shoup ? dys : nullptr, dz, cnt, stream);
        if (s != MM_OK) return s;
        MM_CUDA_TRY(cudaEventRecord(H->done[k], st));
        MM_CUDA_TRY(cudaStreamWaitEvent(H->d2h, H->done[k], 0));
        MM_CUDA_TRY(cudaMemcpyAsync(z + e0, dz, cnt * 4, cudaMemcpyDeviceToHost, H->d2h));
        MM_CUDA_TRY(cudaEventRecord(H->freed[k], H->d2h));
        H->used[k] = true;
        last = k;
    }
    H->next = (int)((H->next + nch) % 3);
    MM_CUDA_TRY(cudaStreamWaitEvent(st, H->freed[last], 0));
    return MM_OK;
}

extern "C" mm_status mm_set_product_streams(int n) {
    if (n < 1 || n > MAX_FORK) return set_err(MM_E_ARG, "product streams must be in [1, %d]", MAX_FORK);
    g_product_streams = n;
    return MM_OK;
}

// Release everything the library caches between calls: the poly_mul / int_mul
// plans (Goldilocks plans hold 2 n-word step-2 tables: 256 MiB at 2^24, 1 GiB
// at 2^26), the per-stream workspaces and the host-pipeline slots; then trim
// the device's default memory pool.  Synchronises the device; later calls
// rebuild what they need.
extern "C" mm_status mm_release_cached(void) {
    MM_CUDA_TRY(cudaDeviceSynchronize());
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        for (auto& kv : g_plans) free_plan(kv.second);
        g_plans.clear();
        for (auto& kv : g_ws)
            if (kv.second.first) cudaFreeAsync(kv.second.first, 0);
        g_ws.clear();
        for (auto& kv : g_ws_slots)
            if (kv.second.first) cudaFreeAsync(kv.second.first, 0);
        g_ws_slots.clear();
    }
    {
        std::lock_guard<std::mutex> g(g_pipe_mu);
        for (auto& kv : g_pipes) {
            HostPipe* h = kv.second;
            std::lock_guard<std::mutex> lk(h->mu);
            if (h->buf) cudaFree(h->buf);
            h->buf = nullptr;
            h->bytes = 0;
            h->layout = 0;
            for (int i = 0; i < 3; i++) h->used[i] = false;
        }
    }
    MM_CUDA_TRY(cudaDeviceSynchronize());
    trim_pool();
    return MM_OK;
}

static Crt3S crt3s_consts() {
    static const uint32_t PR[3] = {998244353u, 985661441u, 943718401u};
    Crt3S K;
    K.p1 = PR[0]; K.p2 = PR[1]; K.p3 = PR[2];
    K.i12 = (uint32_t)hpowmod(PR[0] % PR[1], PR[1] - 2, PR[1]);
    K.i13 = (uint32_t)hpowmod(PR[0] % PR[2], PR[2] - 2, PR[2]);
    K.i23 = (uint32_t)hpowmod(PR[1] % PR[2], PR[2] - 2, PR[2]);
    K.i12s = (uint32_t)(((uint64_t)K.i12 << 32) / K.p2);
    K.i13s = (uint32_t)(((uint64_t)K.i13 << 32) / K.p3);
    K.i23s = (uint32_t)(((uint64_t)K.i23 << 32) / K.p3);
    K.p12 = (uint64_t)PR[0] * PR[1];
    return K;
}
// Garner + carries in one launch: residue products Cp[3][stride] (entry e's
// coefficient k at e nc + k) -> nall = E nout 32-bit limbs; `scratch` holds
// the look-back status words and the ticket (nblk + 1 words of 8 bytes)
static mm_status crt_carry32(const uint32_t* Cp, long long stride, long long nc, long long nout, long long nall,
                             unsigned long long* scratch, uint32_t* out, cudaStream_t st) {
    const long long nblk = (nall + CARRY_B - 1) / CARRY_B;
    MM_CUDA_TRY(cudaMemsetAsync(scratch, 0, (size_t)nblk * 8 + 8, st));
    const size_t smem = 3 * (CARRY_B + CC_HALO + 1) * sizeof(uint32_t);   // 48 KiB + a little: opt in
    MM_CUDA_TRY(cudaFuncSetAttribute(k_crt_carry32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    {
        LaunchScope ls("crt_carry_fused", st);
        k_crt_carry32<<<(int)nblk, CARRY_T, smem, st>>>(Cp, stride, nc, nout, nall, crt3s_consts(), scratch,
                                                         (unsigned*)(scratch + nblk), out);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

// reduce -> scan -> apply over nout output digits; agg: one word per CARRY_B digits
template <class D>
static mm_status carry_run(const D& d, long long nout, uint32_t* agg, typename D::Out* out, cudaStream_t st) {
    // digit-sum lookbehind at position j: j - 1 (carry_gp) -- every policy handles j = 0
    const long long nblk = (nout + CARRY_B - 1) / CARRY_B;
    if constexpr (std::is_same<D, Dig16>::value) {   // shared-memory staged 16-bit limb path, one pass
        // agg holds 2 nblk + 2 words here: the look-back status words and the ticket
        // reduce -> scan -> apply (the coefficients read twice) measured faster
        // than the single-pass look-back once the staging loads were batched
        // (C5 2.408 -> 2.389 ms: the look-back's chain of inclusive prefixes,
        // not the second read, set the single pass's time); MMNTT_CARRY_FUSED=1
        // selects the single pass
        static const bool fused = getenv("MMNTT_CARRY_FUSED") != nullptr;
        if (!fused) {
            {
                LaunchScope ls("carry_reduce", st);
                k_carry16_reduce<<<(int)nblk, CARRY_T, 0, st>>>(d.c, d.nc, nout, agg);
            }
            {
                LaunchScope ls("carry_scan", st);
                k_carry_scan<<<1, 1024, 0, st>>>(agg, nblk);
            }
            {
                LaunchScope ls("carry_apply", st);
                k_carry16_apply<<<(int)nblk, CARRY_T, 0, st>>>(d.c, d.nc, nout, agg, out);
            }
            MM_LAUNCH_CHECK();
            return MM_OK;
        }
        unsigned long long* status = (unsigned long long*)agg;
        unsigned* ticket = (unsigned*)(status + nblk);
        MM_CUDA_TRY(cudaMemsetAsync(status, 0, (size_t)nblk * 8 + 8, st));
        {
            LaunchScope ls("carry_fused", st);
            k_carry16_fused<<<(int)nblk, CARRY_T, 0, st>>>(d.c, d.nc, nout, status, ticket, out);
        }
        MM_LAUNCH_CHECK();
        return MM_OK;
    }
    {
        LaunchScope ls("carry_reduce", st);
        k_carry_reduce<D><<<(int)nblk, CARRY_T, 0, st>>>(d, nout, agg);
    }
    MM_LAUNCH_CHECK();
    {
        LaunchScope ls("carry_scan", st);
        k_carry_scan<<<1, 1024, 0, st>>>(agg, nblk);
    }
    MM_LAUNCH_CHECK();
    {
        LaunchScope ls("carry_apply", st);
        k_carry_apply<D><<<(int)nblk, CARRY_T, 0, st>>>(d, nout, agg, out);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

extern "C" mm_status mm_int_mul_u16(const uint16_t* a, size_t na, const uint16_t* b, size_t nb, uint16_t* c,
                                    void* stream) {
    if (!a || !b || !c) return set_err(MM_E_ARG, "null argument");
    if (na == 0 || nb == 0) return set_err(MM_E_ARG, "empty operands");
    size_t nout = na + nb, lc = na + nb - 1;
    if (overlaps(a, na * 2, c, nout * 2) || overlaps(b, nb * 2, c, nout * 2))
        return set_err(MM_E_ALIAS, "c aliases a or b");
    size_t mn = na < nb ? na : nb;
    if ((u128)mn * 0xFFFE0001ull >= FpG::P) return set_err(MM_E_SIZE_OVERFLOW, "min(na,nb)(2^16-1)^2 >= p");
    int k = 0;
    while ((1ull << k) < lc) k++;
    if (k == 0) k = 1;
    if (k > 26) return set_err(MM_E_SIZE_OVERFLOW, "na + nb - 1 > 2^26");
    uint64_t p = FpG::P;
    uint64_t omega = hpowmod(7, (p - 1) >> k, p);    // 7 generates (Z/pZ)^*
    mm_ntt_plan* P = nullptr;
    mm_status s = cached_plan(64, p, k, omega, &P);
    if (s != MM_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    // coefficient buffer (lc u64) lives after the 2 n transform buffers of the workspace
    size_t n = 1ull << k;
    void* ws = nullptr;
    if ((s = stream_ws(st, (2 * n + lc) * 8 + 17 * 1024 * 8, &ws)) != MM_OK) return s;
    uint64_t* coef = (uint64_t*)ws + 2 * n;
    if ((s = product_impl<FpG, uint16_t, uint64_t>(P, a, (long long)na, b, (long long)nb, coef, (long long)lc, 1, st)) !=
        MM_OK)
        return s;
    // carry propagation (evaluation at 2^16)
    if ((long long)(nout + CARRY_B - 1) / CARRY_B > 17 * 1024 - 1) return set_err(MM_E_SIZE_OVERFLOW, "too many carry blocks");
    // coef + lc: 8-byte aligned status words of the single-pass carry (carry_run)
    return carry_run(Dig16{coef, (long long)lc}, (long long)nout, (uint32_t*)(coef + lc), c, st);
}

// Three-prime integer product: 32-bit chunks (h = 32, A(2^32) = a),
// three 32-bit NTT products mod p1, p2, p3, Garner CRT, carries.
extern "C" mm_status mm_int_mul_u32(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, uint32_t* c,
                                    void* stream) {
    if (!a || !b || !c) return set_err(MM_E_ARG, "null argument");
    if (na == 0 || nb == 0) return set_err(MM_E_ARG, "empty operands");
    const size_t nout = na + nb, lc = na + nb - 1;
    if (overlaps(a, na * 4, c, nout * 4) || overlaps(b, nb * 4, c, nout * 4))
        return set_err(MM_E_ALIAS, "c aliases a or b");
    int k = 0;
    while ((1ull << k) < lc) k++;
    if (k == 0) k = 1;
    // transform length <= 2^22 (2-adicity of p2, p3); then every coefficient
    // <= min(na, nb) (2^32 - 1)^2 < 2^85 < p1 p2 p3 (2^89.6): H < log2(p1 p2 p3)
    if (k > 22) return set_err(MM_E_SIZE_OVERFLOW, "na + nb - 1 > 2^22 (three-prime transform limit)");
    static const uint32_t PR[3] = {998244353u, 985661441u, 943718401u}, GEN[3] = {3, 3, 7};
    Crt3 K;
    K.p1 = PR[0]; K.p2 = PR[1]; K.p3 = PR[2];
    K.i12 = (uint32_t)hpowmod(PR[0] % PR[1], PR[1] - 2, PR[1]);
    K.i13 = (uint32_t)hpowmod(PR[0] % PR[2], PR[2] - 2, PR[2]);
    K.i23 = (uint32_t)hpowmod(PR[1] % PR[2], PR[2] - 2, PR[2]);
    K.p12 = (uint64_t)PR[0] * PR[1];
    cudaStream_t st = (cudaStream_t)stream;
    // workspace: residues [3][na + nb], products [3][lc], CRT words [3 lc], carry aggregates
    const size_t rs = na + nb;
    const size_t nblk = (nout + CARRY_B - 1) / CARRY_B;
    void* ws = nullptr;
    mm_status s = stream_ws2(st, (3 * rs + 3 * lc + 3 * lc + nblk + 64) * 4, &ws);
    if (s != MM_OK) return s;
    uint32_t* R = (uint32_t*)ws;          // R[i * rs + j]: a_j mod p_i (j < na), b at offset na
    uint32_t* Cp = R + 3 * rs;            // Cp[i * lc + k]: c_k mod p_i
    uint32_t* Wd = Cp + 3 * lc;           // 96-bit coefficients
    mm_ntt_plan* PL[3];
    for (int i = 0; i < 3; i++) {
        uint64_t omega = hpowmod(GEN[i], (PR[i] - 1) >> k, PR[i]);
        if ((s = cached_plan(32, PR[i], k, omega, &PL[i])) != MM_OK) return s;
    }
    // the three products modulo p1, p2, p3 in one launch per pass (Remark 6)
    if ((s = product3_impl(PL, a, b, K, R, (long long)rs, (long long)na, (long long)nb, Cp, (long long)lc, st)) != MM_OK)
        return s;
    // Garner CRT and carries in one pass (crt_carry32); Wd is its look-back scratch
    return crt_carry32(Cp, (long long)lc, (long long)lc, (long long)nout, (long long)nout,
                       (unsigned long long*)(((uintptr_t)Wd + 7) & ~(uintptr_t)7), c, st);
}

// ---- sharded integer product building blocks (dist.py ShardedIntMul) ----------------
extern "C" mm_status mm_ntt_fwd_cols_u16(const mm_ntt_plan* plan, const uint16_t* limbs, size_t nlimbs, void* out,
                                         size_t col0, size_t ncols, void* stream) {
    mm_status s = dist_check(plan, limbs, out, col0, ncols, true);
    if (s != MM_OK) return s;
    if (plan->word_bits != 64) return set_err(MM_E_ARG, "16-bit limb columns need a 64-bit (Goldilocks) plan");
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    FpG f;
    ColArgs<FpG> c{};
    c.in = limbs + col0;     // element (j2, j1) of the zero-padded limb vector at limbs[j2 n1 + j1]
    c.out = out;
    c.ncols = (long long)ncols;
    c.nbatch = 1;
    c.in_rs = 1ll << P->k1;
    c.out_rs = (long long)ncols;
    c.in_bs = c.out_bs = 0;
    c.in_len = (long long)nlimbs;
    c.out_len = 1ll << P->k;
    c.col0 = (long long)col0;
    c.n1 = 1ll << P->k1;
    c.k = P->k2;
    c.fs = 1;
    c.lvl = (const uint64_t*)P->lvl_f2;
    c.fs_lo = (const uint64_t*)P->fs_lo_f;
    c.fs_hi = (const uint64_t*)P->fs_hi_f;
    c.fs_full = (const uint64_t*)P->fs_full_f;
    c.fs_h = P->fs_h;
    return launch_cols<FpG, false, uint16_t, uint64_t>(f, c, (cudaStream_t)stream);
}

template <class F>
static mm_status pmul_rows_seg_impl(mm_ntt_plan* P, const void* a, const void* b, void* c, size_t row0, size_t nrows,
                                    int sl, long long seg_stride, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    F f = make_field<F>(P);
    PmulArgs<F> m{};
    m.a = a; m.b = b; m.c = c;
    m.nrows = (long long)nrows;
    m.a_rs = m.b_rs = m.c_rs = 1ll << sl;
    m.la = m.lb = m.lc = 1ll << P->k1;
    m.k = P->k1;
    m.fs = 1; m.k2 = P->k2; m.row0 = (long long)row0;
    m.in_seg_log = m.out_seg_log = sl;
    m.in_seg_stride = m.out_seg_stride = seg_stride;
    // unscaled product (mm_ntt_inv_cols applies n^-1): 1, or 2^32 to undo the 32-bit REDC
    m.sc = host_w<W>(sizeof(T) == 4 ? (uint64_t)(((u128)1 << 32) % P->p) : 1, P->p);
    m.lvl_f = (const W*)P->lvl_f1;
    m.lvl_i = (const W*)P->lvl_i1;
    m.fs_lo = (const W*)P->fs_lo_i;
    m.fs_hi = (const W*)P->fs_hi_i;
    m.fs_full = (const W*)P->fs_full_i;
    m.fs_h = P->fs_h;
    return launch_pmul<F, T, T>(f, m, st);
}
extern "C" mm_status mm_ntt_pmul_rows_seg(const mm_ntt_plan* plan, const void* a, const void* b, void* c, size_t row0,
                                          size_t nrows, size_t seg_len, size_t seg_stride, void* stream) {
    mm_status s = dist_check(plan, a, c, row0, nrows, false);
    if (s != MM_OK) return s;
    if (!b) return set_err(MM_E_ARG, "null argument");
    int sl = 0;
    if ((s = seg_check(plan, seg_len, seg_stride, nrows, &sl)) != MM_OK) return s;
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    cudaStream_t st = (cudaStream_t)stream;
    return P->word_bits == 32 ? pmul_rows_seg_impl<Fp32>(P, a, b, c, row0, nrows, sl, (long long)seg_stride, st)
                              : pmul_rows_seg_impl<FpG>(P, a, b, c, row0, nrows, sl, (long long)seg_stride, st);
}

static mm_status chunk_args(const uint64_t* coef, const uint64_t* halo, size_t nrows, size_t c1, size_t n1, size_t col0,
                            size_t nc, size_t nout, int shift, ChunkRef* R) {
    if (!coef || (!halo && nrows > 0)) return set_err(MM_E_ARG, "null argument");
    if (c1 < 4 || c1 > n1 || col0 + c1 > n1) return set_err(MM_E_ARG, "chunk [%zu, %zu) not inside a row of %zu", col0, col0 + c1, n1);
    R->coef = coef; R->halo = halo;
    R->c1 = (long long)c1; R->n1 = (long long)n1; R->col0 = (long long)col0;
    R->nc = (long long)nc; R->nout = (long long)nout; R->shift = shift;
    return MM_OK;
}
extern "C" mm_status mm_carry_chunks_halo(const uint64_t* coef, size_t nrows, size_t c1, uint64_t* halo_out, void* stream) {
    if (!coef || !halo_out || c1 < 4) return set_err(MM_E_ARG, "bad halo arguments");
    cudaStream_t st = (cudaStream_t)stream;
    {
        LaunchScope ls("carry_halo", st);
        k_chunk_halo<<<(int)((nrows * 4 + 255) / 256), 256, 0, st>>>(coef, (long long)nrows, (long long)c1, halo_out);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
extern "C" mm_status mm_carry_chunks_reduce(const uint64_t* coef, const uint64_t* halo_in, size_t nrows, size_t c1,
                                            size_t n1, size_t col0, size_t nc, size_t nout, int shift, uint32_t* agg,
                                            void* stream) {
    ChunkRef R;
    mm_status s = chunk_args(coef, halo_in, nrows, c1, n1, col0, nc, nout, shift, &R);
    if (s != MM_OK) return s;
    if (!agg) return set_err(MM_E_ARG, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    {
        LaunchScope ls("carry_reduce", st);
        k_chunk_reduce<<<(int)nrows, 256, 0, st>>>(R, agg);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
extern "C" mm_status mm_carry_chunks_scan(uint32_t* agg_all, size_t G, size_t nrows, void* stream) {
    if (!agg_all || G == 0) return set_err(MM_E_ARG, "bad scan arguments");
    cudaStream_t st = (cudaStream_t)stream;
    {
        LaunchScope ls("carry_scan", st);
        k_chunk_scan<<<1, 1024, 0, st>>>(agg_all, (long long)G, (long long)nrows);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
extern "C" mm_status mm_carry_chunks_apply(const uint64_t* coef, const uint64_t* halo_in, size_t nrows, size_t c1,
                                           size_t n1, size_t col0, size_t nc, size_t nout, int shift,
                                           const uint32_t* cin, uint16_t* out, void* stream) {
    ChunkRef R;
    mm_status s = chunk_args(coef, halo_in, nrows, c1, n1, col0, nc, nout, shift, &R);
    if (s != MM_OK) return s;
    if (!cin || !out) return set_err(MM_E_ARG, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    {
        LaunchScope ls("carry_apply", st);
        k_chunk_apply<<<(int)nrows, 256, 0, st>>>(R, cin, out);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

// Polynomial matrix product: C = A B for an m x kk matrix A and a
// kk x n matrix B of polynomials over Z/pZ (entries of A: da coefficients,
// of B: db), C entries have da + db - 1 coefficients.  Every entry is
// transformed once (length L = 2^ceil(log2(da + db - 1)), zero padded), the
// L pointwise matrix products run over Z/pZ, the m n entries of C are
// transformed back.  32-bit p < 2^30 with 2^log2(L) | p - 1.
extern "C" mm_status mm_poly_matmul(uint64_t p, uint64_t g, const uint32_t* A, const uint32_t* B, uint32_t* C,
                                    size_t m, size_t kk, size_t n, size_t da, size_t db, void* stream) {
    if (!A || !B || !C) return set_err(MM_E_ARG, "null argument");
    if (m == 0 || kk == 0 || n == 0 || da == 0 || db == 0) return set_err(MM_E_ARG, "empty operands");
    const size_t lc = da + db - 1;
    int k = 0;
    while ((1ull << k) < lc) k++;
    if (k == 0) k = 1;
    mm_status s = check_modulus(32, p, k);
    if (s != MM_OK) return s;
    const long long L = 1ll << k;
    const size_t words = (size_t)(m * kk + kk * n) * 1;   // per evaluation point in shared memory
    const size_t smem_cap = 200 * 1024 / 4;
    if (words > smem_cap) return set_err(MM_E_UNSUPPORTED_SIZE, "m kk + kk n = %zu exceeds %zu", words, smem_cap);
    // points per CTA: a power of two, >= 8 (32-byte row segments in the staging
    // loads) when the slices fit ~64 KiB, >= 256 / (4 x 4 blocks per point)
    const size_t blocks_per_point = ((m + 3) / 4) * ((n + 3) / 4);
    int FB = 1, lgF = 0;
    const size_t cap_words = (m % 4 == 0 && n % 4 == 0) ? 8 * 1024 : 16 * 1024;   // per buffer (x2 when vectorised)
    while (FB < 256 && ((size_t)FB * blocks_per_point < 256 || FB < 8) && (size_t)(2 * FB) * words <= cap_words) {
        FB *= 2;
        lgF++;
    }
    uint64_t omega = hpowmod(g % p, (p - 1) >> k, p);
    mm_ntt_plan* P = nullptr;
    if ((s = cached_plan(32, p, k, omega, &P)) != MM_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if (debug_checks()) {
        if ((s = check_rows(A, 32, m * kk, da, da, p, st)) != MM_OK) return s;
        if ((s = check_rows(B, 32, kk * n, db, db, p, st)) != MM_OK) return s;
    }
    void* ws = nullptr;
    if ((s = stream_ws2(st, (size_t)(m * kk + kk * n + m * n) * L * 4, &ws)) != MM_OK) return s;
    uint32_t* Ah = (uint32_t*)ws;
    uint32_t* Bh = Ah + m * kk * L;
    uint32_t* Ch = Bh + kk * n * L;
    if ((s = fwd_pad_impl<Fp32>(P, A, (long long)(m * kk), (long long)da, (long long)da, Ah, st)) != MM_OK) return s;
    if ((s = fwd_pad_impl<Fp32>(P, B, (long long)(kk * n), (long long)db, (long long)db, Bh, st)) != MM_OK) return s;
    const size_t smem = (size_t)FB * words * 4;
    const long long tiles = (L + FB - 1) / FB;
    const bool v4 = m % 4 == 0 && n % 4 == 0;
    const uint64_t mu = (uint64_t)(((u128)1 << 64) / p);
    if (v4) {
        // point-major operands: transpose [entries][L] -> [L][entries] (coalesced
        // slices per point), products, transpose back for the inverse transforms
        void* ws3 = nullptr;
        if ((s = stream_ws_slot(st, 3, (size_t)(m * kk + kk * n + m * n) * L * 4, &ws3)) != MM_OK) return s;
        uint32_t* At = (uint32_t*)ws3;
        uint32_t* Bt = At + m * kk * L;
        uint32_t* Ct = Bt + kk * n * L;
        const int tg = num_sms() * 8;
        {
            LaunchScope ls("transpose", st);
            k_transpose32<<<tg, 256, 0, st>>>(Ah, At, (long long)(m * kk), L);
            k_transpose32<<<tg, 256, 0, st>>>(Bh, Bt, (long long)(kk * n), L);
        }
        MM_LAUNCH_CHECK();
        int FBp = 1;
        while (FBp < 64 && (size_t)(2 * FBp) * words <= 12 * 1024 && (size_t)FBp * ((m / 4) * (n / 4)) < 256) FBp *= 2;
        const size_t smem_p = (size_t)FBp * words * 4;
        MM_CUDA_TRY(cudaFuncSetAttribute(k_point_matmul_pm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_point_matmul_pm, 256, smem_p);
        if (per < 1) per = 1;
        const long long tl = (L + FBp - 1) / FBp;
        const int gp = (int)(tl < (long long)num_sms() * per ? tl : (long long)num_sms() * per);
        {
            LaunchScope ls("point_matmul", st);
            k_point_matmul_pm<<<gp, 256, smem_p, st>>>(At, Bt, Ct, (int)m, (int)kk, (int)n, L, FBp, (uint32_t)p, mu);
        }
        MM_LAUNCH_CHECK();
        {
            LaunchScope ls("transpose", st);
            k_transpose32<<<tg, 256, 0, st>>>(Ct, Ch, L, (long long)(m * n));
        }
        MM_LAUNCH_CHECK();
        return inv_trunc_impl<Fp32>(P, Ch, (long long)(m * n), C, (long long)lc, (long long)lc, st);
    }
    auto pm_kern = (void*)k_point_matmul_any;
    MM_CUDA_TRY(cudaFuncSetAttribute(pm_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pm_kern, 256, smem);
    if (per_sm < 1) per_sm = 1;
    const int grid = (int)(tiles < (long long)num_sms() * per_sm ? tiles : (long long)num_sms() * per_sm);
    const uint64_t r64 = (uint64_t)(((u128)1 << 64) % p);
    {
        LaunchScope ls("point_matmul", st);
        k_point_matmul_any<<<grid, 256, smem, st>>>(Ah, Bh, Ch, (int)m, (int)kk, (int)n, L, FB, (uint32_t)p, r64);
    }
    MM_LAUNCH_CHECK();
    return inv_trunc_impl<Fp32>(P, Ch, (long long)(m * n), C, (long long)lc, (long long)lc, st);
}

// Integer matrix product (Table 17): C = A B
// for matrices of integers given as 32-bit limbs (entries of A: na limbs,
// of B: nb limbs; C entries na + nb limbs) -- the three-prime FFT product of
// mm_int_mul_u32 with the pointwise stage a matrix product (mm_poly_matmul
// per prime), then Garner CRT and one batched carry chain.  C entries have
// na + nb + 1 limbs (a sum of kk <= 2^32 products).
extern "C" mm_status mm_int_matmul_u32(const uint32_t* A, const uint32_t* B, uint32_t* C, size_t m, size_t kk, size_t n,
                                       size_t na, size_t nb, void* stream) {
    if (!A || !B || !C) return set_err(MM_E_ARG, "null argument");
    if (m == 0 || kk == 0 || n == 0 || na == 0 || nb == 0) return set_err(MM_E_ARG, "empty operands");
    // an entry is a sum of kk products, < kk 2^(32 (na + nb)): one more limb than a product
    const size_t lc = na + nb - 1, nout = na + nb + 1;
    int k = 0;
    while ((1ull << k) < lc) k++;
    if (k > 22) return set_err(MM_E_SIZE_OVERFLOW, "na + nb - 1 > 2^22 (three-prime transform limit)");
    // every coefficient of an entry <= kk min(na, nb) (2^32 - 1)^2 < p1 p2 p3
    if ((double)kk * (double)(na < nb ? na : nb) >= 3.3e7)
        return set_err(MM_E_SIZE_OVERFLOW, "kk min(na, nb) too large for three 30-bit primes");
    static const uint32_t PR[3] = {998244353u, 985661441u, 943718401u}, GEN[3] = {3, 3, 7};
    Crt3 K;
    K.p1 = PR[0]; K.p2 = PR[1]; K.p3 = PR[2];
    K.i12 = (uint32_t)hpowmod(PR[0] % PR[1], PR[1] - 2, PR[1]);
    K.i13 = (uint32_t)hpowmod(PR[0] % PR[2], PR[2] - 2, PR[2]);
    K.i23 = (uint32_t)hpowmod(PR[1] % PR[2], PR[2] - 2, PR[2]);
    K.p12 = (uint64_t)PR[0] * PR[1];
    cudaStream_t st = (cudaStream_t)stream;
    const size_t sa = m * kk * na, sb = kk * n * nb, sc = m * n * lc;
    const size_t nall = m * n * nout, nblk = (nall + CARRY_B - 1) / CARRY_B;
    void* ws = nullptr;
    mm_status s = stream_ws_slot(st, 2, (3 * (sa + sb) + 3 * sc + 3 * sc + nblk + 64) * 4, &ws);
    if (s != MM_OK) return s;
    uint32_t* RA = (uint32_t*)ws;           // [3][sa]
    uint32_t* RB = RA + 3 * sa;             // [3][sb]
    uint32_t* RC = RB + 3 * sb;             // [3][sc]
    uint32_t* Wd = RC + 3 * sc;             // [sc][3]
    const int grid = num_sms() * 8;
    {
        LaunchScope ls("crt_residues", st);
        k_residues3<<<grid, 256, 0, st>>>(A, (long long)sa, RA, (long long)sa, K);
        k_residues3<<<grid, 256, 0, st>>>(B, (long long)sb, RB, (long long)sb, K);
    }
    MM_LAUNCH_CHECK();
    for (int i = 0; i < 3; i++)
        if ((s = mm_poly_matmul(PR[i], GEN[i], RA + i * sa, RB + i * sb, RC + i * sc, m, kk, n, na, nb, stream)) != MM_OK)
            return s;
    return crt_carry32(RC, (long long)sc, (long long)lc, (long long)nout, (long long)nall,
                       (unsigned long long*)(((uintptr_t)Wd + 7) & ~(uintptr_t)7), C, st);
}

// ---- fused column pass + transpose over peer memory ---------------------------------
// Rank g's column pass (Algorithm 1 steps 1-2 on columns [col0, col0 + ncols))
// stores row t of its block straight into the receive buffer of the rank that
// owns row block h = t / (n2 / G), at segment g: peer_recv[h] + g r2 ncols +
// (t - h r2) ncols + c -- the layout NCCL's all-to-all would deliver, so the
// row pass (mm_ntt_fwd_rows_seg) reads it unchanged.  peer_recv[h] are device
// pointers valid in this process (cudaIpcOpenMemHandle'd peer buffers on one
// node, or local buffers for one-GPU tests); the caller orders the writes
// before the row pass (stream / cross-rank barrier).
extern "C" mm_status mm_ntt_fwd_cols_p2p(const mm_ntt_plan* plan, const void* in, void* const* peer_recv, int G,
                                         int rank, size_t col0, size_t ncols, void* stream) {
    mm_status s = dist_check(plan, in, peer_recv ? peer_recv[0] : nullptr, col0, ncols, true);
    if (s != MM_OK) return s;
    if (G < 1 || G > 8 || rank < 0 || rank >= G) return set_err(MM_E_ARG, "G must be in [1, 8], rank in [0, G)");
    mm_ntt_plan* P = const_cast<mm_ntt_plan*>(plan);
    const long long n2 = 1ll << P->k2, r2 = n2 / G;
    if (r2 * G != n2 || (r2 & (r2 - 1))) return set_err(MM_E_ARG, "n2 = %lld not split into powers of two by %d", n2, G);
    int sh = 0;
    while ((1ll << sh) < r2) sh++;
    cudaStream_t st = (cudaStream_t)stream;
    auto run = [&](auto fld) -> mm_status {
        typedef decltype(fld) F;
        typedef typename F::T T;
        typedef typename F::W W;
        F f = make_field<F>(P);
        ColArgs<F> c{};
        c.in = in; c.out = peer_recv[0];
        c.ncols = (long long)ncols;
        c.nbatch = 1;
        c.in_rs = c.out_rs = (long long)ncols;
        c.in_bs = c.out_bs = 0;
        c.in_len = c.out_len = 1ll << P->k;
        c.col0 = (long long)col0;
        c.n1 = 1ll << P->k1;
        c.k = P->k2;
        c.fs = 1;
        c.lvl = (const W*)P->lvl_f2;
        c.fs_lo = (const W*)P->fs_lo_f;
        c.fs_hi = (const W*)P->fs_hi_f;
        c.fs_full = (const W*)P->fs_full_f;
        c.fs_h = P->fs_h;
        c.npeers = G;
        c.peer_shift = sh;
        for (int h = 0; h < G; h++) {
            if (!peer_recv[h] || ((uintptr_t)peer_recv[h] & 15)) return set_err(MM_E_ARG, "peer buffer %d null or unaligned", h);
            // segment `rank` of rank h's buffer, re-based so that row t lands at t ncols
            c.peer_out[h] = (void*)((T*)peer_recv[h] + (long long)rank * r2 * (long long)ncols - (long long)h * r2 * (long long)ncols);
        }
        return launch_cols<F, false, T, T>(f, c, st);
    };
    return P->word_bits == 32 ? run(Fp32{}) : run(FpG{});
}

// CUDA IPC plumbing for the peer-scatter path (one node, one process per GPU).
// An IPC handle names a whole cudaMalloc allocation; a caching allocator
// (torch) places tensors at offsets inside its blocks, so the handle travels
// with the pointer's offset from the allocation base (cuMemGetAddressRange)
// and the opener adds it back.
typedef CUresult (*PFN_addr_range)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_addr_range addr_range_fn() {
    static PFN_addr_range fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (PFN_addr_range)p;
    }();
    return fn;
}
extern "C" mm_status mm_ipc_get_handle(const void* dev_ptr, void* handle_out /* 64 bytes */, uint64_t* offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return set_err(MM_E_ARG, "null argument");
    auto rng = addr_range_fn();
    if (!rng) return set_err(MM_E_CUDA, "cuMemGetAddressRange is not available");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (rng(&base, &size, (CUdeviceptr)(uintptr_t)dev_ptr) != CUDA_SUCCESS)
        return set_err(MM_E_CUDA, "cuMemGetAddressRange failed (not a device allocation?)");
    cudaIpcMemHandle_t h;
    MM_CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    return MM_OK;
}
extern "C" mm_status mm_ipc_open_handle(const void* handle /* 64 bytes */, void** dev_ptr) {
    if (!handle || !dev_ptr) return set_err(MM_E_ARG, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    MM_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return MM_OK;
}
extern "C" mm_status mm_ipc_close(void* dev_ptr) {
    MM_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return MM_OK;
}

// ---- truncated products (Algorithm 1 with l < n) ----
// c = a b mod p for `batch` pairs, computing only lambda = ceil(lc / n1) of the
// n2 rows of the four-step layout: the column pass keeps rows t < lambda of
// each column TFFT (step 1 restricted to the first lambda outputs), the row
// passes run on those lambda rows only (steps 3-4, pointwise product, inverse
// rows + twiddle), and the inverse column TFT recovers the lambda
// coefficients of every column from its lambda values (tft.cu).  Same
// result as mm_poly_mul, with ~lambda / n2 of its row work.
extern "C" mm_status mm_poly_mul_tft(uint64_t p, uint64_t g, const uint32_t* a, size_t la, const uint32_t* b, size_t lb,
                                     uint32_t* c, size_t batch, void* stream) {
    if (!a || !b || !c) return set_err(MM_E_ARG, "null argument");
    if (la == 0 || lb == 0 || batch == 0) return set_err(MM_E_ARG, "empty operands");
    const size_t lc = la + lb - 1;
    int k = 0;
    while ((1ull << k) < lc) k++;
    if (k <= onepass_log(32)) return mm_poly_mul(32, p, g, a, la, b, lb, c, batch, stream);   // one pass: nothing to truncate
    mm_status s = check_modulus(32, p, k);
    if (s != MM_OK) return s;
    uint64_t omega = hpowmod(g % p, (p - 1) >> k, p);
    mm_ntt_plan* P = nullptr;
    if ((s = cached_plan(32, p, k, omega, &P)) != MM_OK) return s;
    // the inverse column TFT takes columns of <= 2^10 points; the 2^11-point
    // columns of a 2^24 plan (R9) go through the padded product, which returns
    // the same c (checked before any launch)
    if (P->k2 > 10) return mm_poly_mul(32, p, g, a, la, b, lb, c, batch, stream);
    const long long n1 = 1ll << P->k1, lam = ((long long)lc + n1 - 1) / n1;
    cudaStream_t st = (cudaStream_t)stream;
    if (debug_checks()) {
        if ((s = check_rows(a, 32, batch, la, la, p, st)) != MM_OK) return s;
        if ((s = check_rows(b, 32, batch, lb, lb, p, st)) != MM_OK) return s;
    }
    void* ws = nullptr;
    if ((s = stream_ws(st, (size_t)(2 * lam * n1 * (long long)batch) * 4, &ws)) != MM_OK) return s;
    uint32_t* WA = (uint32_t*)ws;
    uint32_t* WB = WA + lam * n1 * (long long)batch;
    Fp32 f = make_field<Fp32>(P);
    for (int op = 0; op < 2; op++) {
        ColArgs<Fp32> cc{};
        cc.in = op == 0 ? (const void*)a : (const void*)b;
        cc.out = op == 0 ? WA : WB;
        cc.ncols = n1;
        cc.nbatch = (long long)batch;
        cc.in_rs = n1; cc.out_rs = n1;
        cc.in_bs = op == 0 ? (long long)la : (long long)lb;
        cc.out_bs = lam * n1;
        cc.in_len = cc.in_bs;
        cc.out_len = lam * n1;                 // rows t < lambda only (the TFFT of size lambda)
        cc.n1 = n1;
        cc.k = P->k2;
        cc.fs = 1;
        cc.lvl = (const uint2*)P->lvl_f2;
        cc.fs_lo = (const uint2*)P->fs_lo_f;
        cc.fs_hi = (const uint2*)P->fs_hi_f;
        cc.fs_full = (const uint2*)P->fs_full_f;
        cc.fs_h = P->fs_h;
        if ((s = launch_cols<Fp32, false, uint32_t, uint32_t>(f, cc, st)) != MM_OK) return s;
    }
    PmulArgs<Fp32> m{};
    m.a = WA; m.b = WB; m.c = WA;
    m.nrows = (long long)batch * lam;
    m.a_rs = m.b_rs = m.c_rs = n1;
    m.la = m.lb = m.lc = n1;
    m.k = P->k1;
    m.fs = 1; m.k2 = P->k2; m.row0 = 0;
    m.rows_per = lam;
    // the row DIT is unscaled and the column TFT normalises itself: n1^-1 2^32 (REDC)
    const uint64_t n1inv = hpowmod((uint64_t)n1 % p, p - 2, p);
    m.sc = mkw32(hmulmod(n1inv, ((u128)1 << 32) % p, p), p);
    m.lvl_f = (const uint2*)P->lvl_f1;
    m.lvl_i = (const uint2*)P->lvl_i1;
    m.fs_lo = (const uint2*)P->fs_lo_i;
    m.fs_hi = (const uint2*)P->fs_hi_i;
    m.fs_full = (const uint2*)P->fs_full_i;
    m.fs_h = P->fs_h;
    if ((s = launch_pmul<Fp32, uint32_t, uint32_t>(f, m, st)) != MM_OK) return s;
    tft::ItftArgs it{};
    it.in = WA; it.out = c;
    it.nbatch = (long long)batch;
    it.in_bs = lam * n1;
    it.out_bs = it.out_len = (long long)lc;
    it.n1 = n1;
    it.k2 = P->k2;
    it.lam = (int)lam;
    it.p = (uint32_t)p;
    it.lvl_f = (const uint2*)P->lvl_f2;
    it.lvl_i = (const uint2*)P->lvl_i2;
    it.inv2 = mkw32((p + 1) / 2, p);
    for (int j = 0; j <= P->k2 && j < 11; j++) it.inv_pow2[j] = mkw32(hpowmod((p + 1) / 2, (uint64_t)j, p), p);
    return tft::launch_col_itft(it, st);
}

// ---- many small problems in one launch (jobs.cu) ----------------------------------
// Validates every job and resolves its plan before anything launches: a bad
// job fails the whole call with nothing queued.
extern "C" mm_status mm_run_jobs(const mm_job* jobs, int njobs, void* stream) {
    if (njobs < 0 || (njobs > 0 && !jobs)) return set_err(MM_E_ARG, "null or negative job table");
    if (njobs == 0) return MM_OK;
    std::vector<DevJob> dj((size_t)njobs);
    for (int i = 0; i < njobs; i++) {
        const mm_job& J = jobs[i];
        DevJob& d = dj[(size_t)i];
        memset(&d, 0, sizeof(d));
        d.kind = J.kind;
        d.order = J.order;
        const mm_ntt_plan* P = nullptr;
        if (J.kind == MM_JOB_POLY_MUL) {
            if (!J.in || !J.in2 || !J.out) return set_err(MM_E_ARG, "job %d: null product buffer", i);
            if (J.la == 0 || J.lb == 0) return set_err(MM_E_ARG, "job %d: empty operand", i);
            const size_t lc = J.la + J.lb - 1;
            int k = 0;
            while ((1ull << k) < lc) k++;
            if (k == 0) k = 1;
            if (k > MAX_BLOCK_LOG)
                return set_err(MM_E_UNSUPPORTED_SIZE, "job %d: product length %zu > 2^%d", i, lc, MAX_BLOCK_LOG);
            mm_status s = check_modulus(32, J.p, k);
            if (s != MM_OK) return s;
            mm_ntt_plan* Q = nullptr;
            if ((s = cached_plan(32, J.p, k, hpowmod(J.g % J.p, (J.p - 1) >> k, J.p), &Q)) != MM_OK) return s;
            P = Q;
            d.sc = mkw32(P->ninv_r, P->p);   // n^-1 2^32: the REDC product's 2^-32 folded in
            d.la = (long long)J.la;
            d.lb = (long long)J.lb;
            d.in2 = (const uint32_t*)J.in2;
        } else if (J.kind == MM_JOB_FORWARD || J.kind == MM_JOB_INVERSE || J.kind == MM_JOB_ROUNDTRIP) {
            P = J.plan;
            if (!P) return set_err(MM_E_ARG, "job %d: null plan", i);
            if (P->word_bits != 32 || P->k2 != 0 || P->k > MAX_BLOCK_LOG)
                return set_err(MM_E_UNSUPPORTED_SIZE, "job %d: jobs take 32-bit single-pass plans (log2n <= %d)", i,
                               MAX_BLOCK_LOG);
            if (!J.in || (J.kind != MM_JOB_ROUNDTRIP && !J.out) || (J.kind == MM_JOB_ROUNDTRIP && !J.out2))
                return set_err(MM_E_ARG, "job %d: null buffer", i);
            if (J.order != MM_ORDER_NATURAL && J.order != MM_ORDER_BITREV) return set_err(MM_E_ARG, "job %d: bad order", i);
            d.sc = mkw32(P->ninv, P->p);
        } else {
            return set_err(MM_E_ARG, "job %d: unknown kind %d", i, J.kind);
        }
        d.k = P->k;
        d.f = make_field<Fp32>(P);
        d.lvl_f = (const uint2*)P->lvl_f1;
        d.lvl_i = (const uint2*)P->lvl_i1;
        d.in = (const uint32_t*)J.in;
        d.out = (uint32_t*)J.out;
        d.out2 = (uint32_t*)J.out2;
    }
    return launch_jobs(dj.data(), njobs, (cudaStream_t)stream);
}
