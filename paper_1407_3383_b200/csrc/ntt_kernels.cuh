// ntt_kernels.cuh -- the tile kernels of the NTT engine and their launchers.
//
//   k_rows      : C whole rows of length L = 2^LOGL per tile (single-pass
//                 transforms for n <= 2^12, and the row pass = Algorithm 1
//                 steps 3-4 / inverse).
//   k_cols      : C adjacent columns of an n2 x n1 matrix per tile (the column
//                 pass = Algorithm 1 steps 1-2 / inverse).
//   k_rows_pmul : rows of two operands -> DIF, DIF, pointwise product, DIT
//                 ("two direct TFT and one inverse TFT ... entry-wise
//                 vector product"), fused in one pass.
//
// All sizes are template parameters (LOGL); launchers dispatch on the
// runtime log2 length.  Explicit instantiations live in ntt_inst*.cu.
#pragma once
#include "common.h"
#include "ntt_core.cuh"

namespace mm {

constexpr int NT = 256;                  // threads per CTA for tile kernels
constexpr size_t SMEM_MAX = 227 * 1024;  // max dynamic shared memory per CTA on sm_100

template <class F> struct Cfg;
template <> struct Cfg<Fp32> { enum { RL = 4, BUDGET = 8192, COLC = 32, V = 4 }; };
template <> struct Cfg<FpG> { enum { RL = 3, BUDGET = 4096, COLC = 16, V = 2 }; };

// Tiles of L <= 512 points use the interleaved layout [j][c] with C transforms
// of 128 bytes per row (lane = transform: every access of every group is
// conflict-free without padding); longer transforms use one padded row per
// transform (RowLayout, pitch = 16 banks mod 32).
template <class F, int LOGL> struct InterOK {
    enum { v = (size_t)Cfg<F>::COLC * (1u << LOGL) * sizeof(typename F::T) <= 64 * 1024 };
};
template <class F, int LOGL> struct RowsTile {
    typedef typename F::T T;
    enum { C = InterOK<F, LOGL>::v ? Cfg<F>::COLC : ((Cfg<F>::BUDGET >> LOGL) > 0 ? (Cfg<F>::BUDGET >> LOGL) : 1) };
    typedef typename std::conditional<InterOK<F, LOGL>::v, ColLayout<T, LOGL, C>, RowLayout<T, LOGL, C>>::type Lay;
};
template <class F, int LOGL> struct PmulTile {
    typedef typename F::T T;
    enum { C = InterOK<F, LOGL>::v ? Cfg<F>::COLC
                                   : (((Cfg<F>::BUDGET / 2) >> LOGL) > 0 ? ((Cfg<F>::BUDGET / 2) >> LOGL) : 1) };
    typedef typename std::conditional<InterOK<F, LOGL>::v, ColLayout<T, LOGL, C>, RowLayout<T, LOGL, C>>::type Lay;
};
// column tiles: one 128-byte line per matrix row when it fits in 64 KiB
// (ColLayout), else a 32-byte sector per row transposed into padded rows.
template <class T, int LOGL, int C_> struct RowLayoutOdd : RowLayout<T, LOGL, C_> {
    typedef RowLayout<T, LOGL, C_> B;
    static constexpr int WORDS = sizeof(T) / 4;
    static constexpr int SROW = [] {
        int s = B::PADL;
        while (((s * WORDS) & 31) != WORDS) s++;   // consecutive c -> consecutive banks
        return s;
    }();
    static constexpr int ELEMS = C_ * SROW;
    __device__ __forceinline__ static int addr(int c, int j) { return c * SROW + j + (j >> 4); }
    __device__ __forceinline__ static int chunk_base(int c, int base) { return c * SROW + base + (base >> 4); }
};
template <class F, int LOGL> struct ColsTile {
    typedef typename F::T T;
    enum { C = InterOK<F, LOGL>::v ? Cfg<F>::COLC : 32 / (int)sizeof(T) };
    typedef typename std::conditional<InterOK<F, LOGL>::v, ColLayout<T, LOGL, C>, RowLayoutOdd<T, LOGL, C>>::type Lay;
};

// ---------------------------------------------------------------- args
template <class F> struct RowArgs {
    typedef typename F::W W;
    const void* in;
    void* out;
    long long nrows, in_rs, out_rs, in_len, out_len, row0;
    int k, k2, perm, fs, scale, canon, vec_in, vec_out, tw_smem;
    W sc;
    const W* lvl;
    const W* fs_lo;
    const W* fs_hi;
    const W* fs_full;     // full step-2 table [i2][j1] when small enough, else null
    int fs_h;
};
template <class F> struct ColArgs {
    typedef typename F::W W;
    const void* in;
    void* out;
    long long ncols, nbatch, in_rs, out_rs, in_bs, out_bs, in_len, out_len, col0, n1;
    int k, fs, scale, canon, vec_in, vec_out, tw_smem;
    W sc;
    const W* lvl;
    const W* fs_lo;
    const W* fs_hi;
    const W* fs_full;
    int fs_h;
};
template <class F> struct PmulArgs {
    typedef typename F::W W;
    const void* a;
    const void* b;
    void* c;
    long long nrows, a_rs, b_rs, c_rs, la, lb, lc, row0;
    int k, k2, fs, canon, vec_in, vec_out, tw_smem;
    W sc;                 // pointwise post-multiplier (n^-1, times 2^32 for the 32-bit REDC)
    const W* lvl_f;
    const W* lvl_i;
    const W* fs_lo;       // inverse step-2 twiddles
    const W* fs_hi;
    const W* fs_full;
    int fs_h;
};

// ---------------------------------------------------------------- helpers
template <class TIn, class T> __device__ __forceinline__ T ld_conv(const TIn* p) { return (T)__ldg(p); }

template <class W> __device__ __forceinline__ void stage_twiddles(W* dst, const W* src, int L) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) dst[i] = src[i];
}

// step-2 twiddle w^(j1 [i2]) (sign folded in the tables): full table or two-level split
template <class F>
__device__ __forceinline__ typename F::T fs_apply(const F& f, typename F::T v, const typename F::W* full,
                                                  const typename F::W* lo, const typename F::W* hi, int h,
                                                  long long i2, int k2, long long j1, long long n1) {
    if (full) return f.mulw(v, __ldg(full + i2 * n1 + j1));
    uint64_t e = (uint64_t)j1 * (uint64_t)brev((int)i2, k2);
    v = f.mulw(v, __ldg(lo + (e & ((1ull << h) - 1))));
    return f.mulw(v, __ldg(hi + (e >> h)));
}

template <class T> struct Vec;
template <> struct Vec<uint32_t> { typedef uint4 type; enum { N = 4 }; };
template <> struct Vec<uint64_t> { typedef ulonglong2 type; enum { N = 2 }; };

template <class T> __device__ __forceinline__ void vget(const typename Vec<T>::type& v, T* out);
template <> __device__ __forceinline__ void vget<uint32_t>(const uint4& v, uint32_t* o) {
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <> __device__ __forceinline__ void vget<uint64_t>(const ulonglong2& v, uint64_t* o) {
    o[0] = v.x; o[1] = v.y;
}
template <class T> __device__ __forceinline__ typename Vec<T>::type vmake(const T* i);
template <> __device__ __forceinline__ uint4 vmake<uint32_t>(const uint32_t* i) { return make_uint4(i[0], i[1], i[2], i[3]); }
template <> __device__ __forceinline__ ulonglong2 vmake<uint64_t>(const uint64_t* i) { return make_ulonglong2(i[0], i[1]); }

// ---------------------------------------------------------------- row-tile I/O
// Rows [r0, r0 + C) of a row-major array (row stride rs, valid prefix len per
// row, zeros beyond) <-> a tile.  For the interleaved layout the lane index
// runs over rows (one 16-byte vector per lane; the sector's other half is the
// same lane's next vector, an L1 hit), so shared accesses are conflict-free;
// for the padded row layout consecutive lanes take consecutive vectors of a
// row.  Loads of a thread are issued in batches of up to 8 vectors before any
// shared store (memory-level parallelism).
template <class Lay, int LOGL, int NTH> struct RowIO {
    static constexpr int L = 1 << LOGL;
    static constexpr int C = Lay::C;
    template <int V> __device__ __forceinline__ static void map(int e, int& c, int& j) {
        if (Lay::COL) { c = e % C; j = (e / C) * V; }
        else { c = (e * V) >> LOGL; j = (e * V) & (L - 1); }
    }
};

template <class F, class Lay, int LOGL, class TIn>
__device__ __forceinline__ void load_rows(typename F::T* s, const TIn* in, long long r0, long long nrows, long long rs,
                                          long long len, bool vec, bool perm) {
    typedef typename F::T T;
    typedef typename Vec<T>::type TV;
    constexpr int L = 1 << LOGL, C = Lay::C, V = Vec<T>::N;
    typedef RowIO<Lay, LOGL, NT> IO;
    if (L >= V && sizeof(TIn) == sizeof(T) && vec && !perm) {
        constexpr int TOT = C * L / V;                       // vectors in the tile
        constexpr int NV = (TOT + NT - 1) / NT;              // per thread
        constexpr int B = NV < 4 ? NV : 4;
#pragma unroll
        for (int u0 = 0; u0 < NV; u0 += B) {
            TV buf[B];
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e = threadIdx.x + (u0 + u) * NT;
                int c, j;
                IO::template map<V>(e, c, j);
                const bool ok = e < TOT && r0 + c < nrows;
                const TV* src = (const TV*)(ok ? (const T*)in + (r0 + c) * rs + j : (const T*)in);
                buf[u] = __ldg(src);
                if (!ok) buf[u] = TV{};
            }
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e = threadIdx.x + (u0 + u) * NT;
                if (e >= TOT) continue;
                int c, j;
                IO::template map<V>(e, c, j);
                T v[V];
                vget<T>(buf[u], v);
#pragma unroll
                for (int i = 0; i < V; i++) s[Lay::addr(c, j + i)] = v[i];
            }
        }
    } else {
        for (int e = threadIdx.x; e < C * L; e += NT) {
            int c, j;
            IO::template map<1>(e, c, j);
            const long long r = r0 + c;
            T v = 0;
            if (r < nrows && j < len) v = ld_conv<TIn, T>(in + r * rs + j);
            s[Lay::addr(c, perm ? brev(j, LOGL) : j)] = v;
        }
    }
}

// epilogue of a row tile: optional step-2 twiddle w^(+-j [i2]) (full table
// rows are contiguous: one 8- or 16-byte vector per element group), n^-1
// scaling and canonicalisation, then vector stores.
template <class F, class Lay, int LOGL, class TOut>
__device__ __forceinline__ void store_rows(const F& f, const typename F::T* s, TOut* out, long long r0, long long nrows,
                                           long long rs, long long len, bool vec, bool perm, int fs,
                                           const typename F::W* fs_full, const typename F::W* fs_lo,
                                           const typename F::W* fs_hi, int fs_h, long long row0, int k2, int scale,
                                           typename F::W sc, int canon) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename Vec<T>::type TV;
    constexpr int L = 1 << LOGL, C = Lay::C, V = Vec<T>::N;
    typedef RowIO<Lay, LOGL, NT> IO;
    if (L >= V && sizeof(TOut) == sizeof(T) && vec && !perm) {
        constexpr int TOT = C * L / V;
        constexpr int NV = (TOT + NT - 1) / NT;
        constexpr int B = NV < 2 ? NV : 2;
#pragma unroll
        for (int u0 = 0; u0 < NV; u0 += B) {
            T v[B][V];
            W w[B][V];
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e = threadIdx.x + (u0 + u) * NT;
                int c, j;
                IO::template map<V>(e < TOT ? e : 0, c, j);      // idle lanes read a valid slot
#pragma unroll
                for (int i = 0; i < V; i++) v[u][i] = s[Lay::addr(c, j + i)];
                if (fs && fs_full) {
                    const long long i2 = (row0 + r0 + (e < TOT ? c : 0)) & ((1ll << k2) - 1);
#pragma unroll
                    for (int i = 0; i < V; i++) w[u][i] = __ldg(fs_full + i2 * L + j + i);
                }
            }
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e = threadIdx.x + (u0 + u) * NT;
                int c, j;
                IO::template map<V>(e, c, j);
                const long long r = r0 + c;
                if (e >= TOT || r >= nrows) continue;
#pragma unroll
                for (int i = 0; i < V; i++) {
                    T x = v[u][i];
                    if (fs) {
                        if (fs_full) x = f.mulw(x, w[u][i]);
                        else x = fs_apply(f, x, nullptr, fs_lo, fs_hi, fs_h, (row0 + r) & ((1ll << k2) - 1), k2, j + i, L);
                    }
                    if (scale) x = f.mulw(x, sc);
                    if (canon) x = f.canon(x);
                    v[u][i] = x;
                }
                *(TV*)((T*)out + r * rs + j) = vmake<T>(v[u]);
            }
        }
    } else {
        for (int e = threadIdx.x; e < C * L; e += NT) {
            int c, j;
            IO::template map<1>(e, c, j);
            const long long r = r0 + c;
            if (r >= nrows || j >= len) continue;
            T x = s[Lay::addr(c, perm ? brev(j, LOGL) : j)];
            if (fs) x = fs_apply(f, x, fs_full, fs_lo, fs_hi, fs_h, (row0 + r) & ((1ll << k2) - 1), k2, j, L);
            if (scale) x = f.mulw(x, sc);
            if (canon) x = f.canon(x);
            out[r * rs + j] = (TOut)x;
        }
    }
}

// ---------------------------------------------------------------- row pass
template <class F, int LOGL, bool INV, class TIn, class TOut>
__global__ void __launch_bounds__(NT, 4) k_rows(F f, RowArgs<F> a) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename RowsTile<F, LOGL>::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int C = Lay::C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* tws = (W*)smem_raw;
    T* s = (T*)(tws + (a.tw_smem ? L : 0));
    if (a.tw_smem) stage_twiddles(tws, a.lvl, L);
    const W* tw = a.tw_smem ? tws : a.lvl;
    const long long ntiles = (a.nrows + C - 1) / C;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long r0 = tile * C;
        load_rows<F, Lay, LOGL, TIn>(s, (const TIn*)a.in, r0, a.nrows, a.in_rs, a.in_len, a.vec_in, INV && a.perm);
        __syncthreads();
        if (INV) tile_dit<F, Lay, LOGL, Cfg<F>::RL, NT>(f, s, tw);
        else tile_dif<F, Lay, LOGL, Cfg<F>::RL, NT>(f, s, tw);
        store_rows<F, Lay, LOGL, TOut>(f, s, (TOut*)a.out, r0, a.nrows, a.out_rs, a.out_len, a.vec_out,
                                       !INV && a.perm, INV ? a.fs : 0, a.fs_full, a.fs_lo, a.fs_hi, a.fs_h, a.row0,
                                       a.k2, a.scale, a.sc, a.canon);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- column pass
template <class F, int LOGL, bool INV, class TIn, class TOut>
__global__ void __launch_bounds__(NT, 4) k_cols(F f, ColArgs<F> a) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename Vec<T>::type TV;
    typedef typename ColsTile<F, LOGL>::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int C = Lay::C;
    constexpr int V = Vec<T>::N;
    constexpr int CV = C / V;        // vectors per tile row
    constexpr int TOT = L * CV;
    constexpr int NV = (TOT + NT - 1) / NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* tws = (W*)smem_raw;
    T* s = (T*)(tws + (a.tw_smem ? L : 0));
    if (a.tw_smem) stage_twiddles(tws, a.lvl, L);
    const W* tw = a.tw_smem ? tws : a.lvl;
    const TIn* in = (const TIn*)a.in;
    TOut* out = (TOut*)a.out;
    const long long cgroups = (a.ncols + C - 1) / C;
    const long long ntiles = cgroups * a.nbatch;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long b = tile / cgroups;
        const long long cl0 = (tile - b * cgroups) * C;
        const TIn* inb = in + b * a.in_bs + cl0;
        const long long lin0 = a.col0 + cl0;        // logical column of c = 0
        if (a.vec_in) {
            constexpr int B = NV < 4 ? NV : 4;
#pragma unroll
            for (int u0 = 0; u0 < NV; u0 += B) {
                TV buf[B];
                int nval[B];
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e = threadIdx.x + (u0 + u) * NT;
                    const int t = e / CV, c = (e % CV) * V;
                    const long long lin = (long long)t * a.n1 + lin0 + c;
                    long long lim = a.in_len - lin;
                    if (a.ncols - cl0 - c < lim) lim = a.ncols - cl0 - c;
                    nval[u] = e >= TOT ? 0 : (lim >= V ? V : (lim > 0 ? (int)lim : 0));
                    const TV* src = (const TV*)(nval[u] == V ? (const T*)inb + (long long)t * a.in_rs + c : (const T*)in);
                    buf[u] = __ldg(src);
                }
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e = threadIdx.x + (u0 + u) * NT;
                    if (e >= TOT) continue;
                    const int t = e / CV, c = (e % CV) * V;
                    T v[V];
                    vget<T>(buf[u], v);
                    if (nval[u] < V) {
#pragma unroll
                        for (int i = 0; i < V; i++)
                            v[i] = i < nval[u] ? ld_conv<TIn, T>(inb + (long long)t * a.in_rs + c + i) : (T)0;
                    }
                    if (Lay::COL) {
                        *(TV*)(s + Lay::addr(c, t)) = vmake<T>(v);
                    } else {
#pragma unroll
                        for (int i = 0; i < V; i++) s[Lay::addr(c + i, t)] = v[i];
                    }
                }
            }
        } else {
            for (int e = threadIdx.x; e < L * C; e += NT) {
                const int t = e / C, c = e % C;
                T v = 0;
                if (cl0 + c < a.ncols && (long long)t * a.n1 + lin0 + c < a.in_len)
                    v = ld_conv<TIn, T>(inb + (long long)t * a.in_rs + c);
                s[Lay::addr(c, t)] = v;
            }
        }
        __syncthreads();
        if (INV) tile_dit<F, Lay, LOGL, Cfg<F>::RL, NT>(f, s, tw);
        else tile_dif<F, Lay, LOGL, Cfg<F>::RL, NT>(f, s, tw);
        TOut* outb = out + b * a.out_bs + cl0;
        const int fs = INV ? 0 : a.fs;
        if (a.vec_out) {
            constexpr int B = NV < 2 ? NV : 2;
#pragma unroll
            for (int u0 = 0; u0 < NV; u0 += B) {
                T v[B][V];
                W w[B][V];
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e = threadIdx.x + (u0 + u) * NT;
                    const int t = (e < TOT ? e : 0) / CV, c = (e % CV) * V;
                    if (Lay::COL) vget<T>(*(const TV*)(s + Lay::addr(c, t)), v[u]);
                    else {
#pragma unroll
                        for (int i = 0; i < V; i++) v[u][i] = s[Lay::addr(c + i, t)];
                    }
                    if (fs && a.fs_full) {
                        long long j1 = lin0 + c;
                        if (j1 + V > a.n1) j1 = a.n1 - V;               // ragged column tail: any valid entry
#pragma unroll
                        for (int i = 0; i < V; i++) w[u][i] = __ldg(a.fs_full + (long long)t * a.n1 + j1 + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e = threadIdx.x + (u0 + u) * NT;
                    if (e >= TOT) continue;
                    const int t = e / CV, c = (e % CV) * V;
                    const long long lin = (long long)t * a.n1 + lin0 + c;
#pragma unroll
                    for (int i = 0; i < V; i++) {
                        T x = v[u][i];
                        if (fs) {
                            if (a.fs_full) x = f.mulw(x, w[u][i]);
                            else x = fs_apply(f, x, nullptr, a.fs_lo, a.fs_hi, a.fs_h, t, LOGL, lin0 + c + i, a.n1);
                        }
                        if (a.scale) x = f.mulw(x, a.sc);
                        if (a.canon) x = f.canon(x);
                        v[u][i] = x;
                    }
                    if (cl0 + c + V <= a.ncols && lin + V <= a.out_len) {
                        *(TV*)((T*)outb + (long long)t * a.out_rs + c) = vmake<T>(v[u]);
                    } else {
#pragma unroll
                        for (int i = 0; i < V; i++)
                            if (cl0 + c + i < a.ncols && lin + i < a.out_len)
                                outb[(long long)t * a.out_rs + c + i] = (TOut)v[u][i];
                    }
                }
            }
        } else {
            for (int e = threadIdx.x; e < L * C; e += NT) {
                const int t = e / C, c = e % C;
                if (cl0 + c >= a.ncols || (long long)t * a.n1 + lin0 + c >= a.out_len) continue;
                T x = s[Lay::addr(c, t)];
                if (fs) x = fs_apply(f, x, a.fs_full, a.fs_lo, a.fs_hi, a.fs_h, t, LOGL, lin0 + c, a.n1);
                if (a.scale) x = f.mulw(x, a.sc);
                if (a.canon) x = f.canon(x);
                outb[(long long)t * a.out_rs + c] = (TOut)x;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- fused product rows
template <class F, int LOGL, class TIn, class TOut>
__global__ void __launch_bounds__(NT, 3) k_rows_pmul(F f, PmulArgs<F> a) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename PmulTile<F, LOGL>::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int C = Lay::C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* twfs = (W*)smem_raw;
    W* twis = twfs + (a.tw_smem ? L : 0);
    T* sa = (T*)(twis + (a.tw_smem ? L : 0));
    T* sb = sa + Lay::ELEMS;
    if (a.tw_smem) {
        stage_twiddles(twfs, a.lvl_f, L);
        stage_twiddles(twis, a.lvl_i, L);
    }
    const W* twf = a.tw_smem ? twfs : a.lvl_f;
    const W* twi = a.tw_smem ? twis : a.lvl_i;
    const long long ntiles = (a.nrows + C - 1) / C;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long r0 = tile * C;
        load_rows<F, Lay, LOGL, TIn>(sa, (const TIn*)a.a, r0, a.nrows, a.a_rs, a.la, a.vec_in, false);
        load_rows<F, Lay, LOGL, TIn>(sb, (const TIn*)a.b, r0, a.nrows, a.b_rs, a.lb, a.vec_in, false);
        __syncthreads();
        tile_dif<F, Lay, LOGL, Cfg<F>::RL, NT>(f, sa, twf);
        tile_dif<F, Lay, LOGL, Cfg<F>::RL, NT>(f, sb, twf);
        for (int e = threadIdx.x; e < C * L; e += NT) {
            const int ix = Lay::COL ? e : Lay::addr(e >> LOGL, e & (L - 1));   // the interleaved tile is dense
            sa[ix] = f.mulw(f.mul_redc(sa[ix], sb[ix]), a.sc);
        }
        __syncthreads();
        tile_dit<F, Lay, LOGL, Cfg<F>::RL, NT>(f, sa, twi);
        store_rows<F, Lay, LOGL, TOut>(f, sa, (TOut*)a.c, r0, a.nrows, a.c_rs, a.lc, a.vec_out, false, a.fs, a.fs_full,
                                       a.fs_lo, a.fs_hi, a.fs_h, a.row0, a.k2, 0, a.sc, a.canon);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launchers
template <class K> static mm_status set_smem(K kern, size_t bytes) {
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return MM_OK;
}
template <class K> static int grid_for(K kern, size_t smem, long long tiles) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    if (per_sm < 1) per_sm = 1;
    long long cap = (long long)num_sms() * per_sm;
    return (int)(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
}
// twiddles go to shared memory unless they would push the CTA past ~100 KiB
static inline bool tw_in_smem(size_t data, size_t tw) {
    return data + tw <= 100 * 1024 || (data > 100 * 1024 && data + tw <= SMEM_MAX && tw <= 8 * 1024);
}
static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <class F, int LOGL, bool INV, class TIn, class TOut>
static mm_status launch_rows_k(const F& f, RowArgs<F> a, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename RowsTile<F, LOGL>::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int V = Vec<T>::N;
    size_t data = (size_t)Lay::ELEMS * sizeof(T), twb = (size_t)L * sizeof(W);
    a.tw_smem = tw_in_smem(data, twb);
    size_t smem = data + (a.tw_smem ? twb : 0);
    a.vec_in = sizeof(TIn) == sizeof(T) && !(INV && a.perm) && a.in_len >= L && a.in_rs % V == 0 && aligned16(a.in);
    a.vec_out = sizeof(TOut) == sizeof(T) && !(!INV && a.perm) && a.out_len >= L && a.out_rs % V == 0 &&
                aligned16(a.out) && !(INV && a.fs && !a.fs_full && false);
    auto kern = k_rows<F, LOGL, INV, TIn, TOut>;
    mm_status s = set_smem(kern, smem);
    if (s != MM_OK) return s;
    long long tiles = (a.nrows + Lay::C - 1) / Lay::C;
    {
        LaunchScope ls(INV ? "ntt_rows_inv" : "ntt_rows_fwd", st);
        kern<<<grid_for(kern, smem, tiles), NT, smem, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

template <class F, int LOGL, bool INV, class TIn, class TOut>
static mm_status launch_cols_k(const F& f, ColArgs<F> a, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename ColsTile<F, LOGL>::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int V = Vec<T>::N;
    size_t data = (size_t)Lay::ELEMS * sizeof(T), twb = (size_t)L * sizeof(W);
    a.tw_smem = tw_in_smem(data, twb);
    size_t smem = data + (a.tw_smem ? twb : 0);
    a.vec_in = sizeof(TIn) == sizeof(T) && a.in_rs % V == 0 && (a.in_bs % V == 0 || a.nbatch == 1) && aligned16(a.in);
    a.vec_out = sizeof(TOut) == sizeof(T) && a.out_rs % V == 0 && (a.out_bs % V == 0 || a.nbatch == 1) &&
                aligned16(a.out);
    auto kern = k_cols<F, LOGL, INV, TIn, TOut>;
    mm_status s = set_smem(kern, smem);
    if (s != MM_OK) return s;
    long long tiles = (a.ncols + Lay::C - 1) / Lay::C * a.nbatch;
    {
        LaunchScope ls(INV ? "ntt_cols_inv" : "ntt_cols_fwd", st);
        kern<<<grid_for(kern, smem, tiles), NT, smem, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

template <class F, int LOGL, class TIn, class TOut>
static mm_status launch_pmul_k(const F& f, PmulArgs<F> a, cudaStream_t st) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename PmulTile<F, LOGL>::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int V = Vec<T>::N;
    size_t data = 2 * (size_t)Lay::ELEMS * sizeof(T), twb = 2 * (size_t)L * sizeof(W);
    a.tw_smem = tw_in_smem(data, twb);
    size_t smem = data + (a.tw_smem ? twb : 0);
    a.vec_in = sizeof(TIn) == sizeof(T) && a.la >= L && a.lb >= L && a.a_rs % V == 0 && a.b_rs % V == 0 &&
               aligned16(a.a) && aligned16(a.b);
    a.vec_out = sizeof(TOut) == sizeof(T) && a.lc >= L && a.c_rs % V == 0 && aligned16(a.c);
    auto kern = k_rows_pmul<F, LOGL, TIn, TOut>;
    mm_status s = set_smem(kern, smem);
    if (s != MM_OK) return s;
    long long tiles = (a.nrows + Lay::C - 1) / Lay::C;
    {
        LaunchScope ls(a.fs ? "pmul_rows_fourstep" : "pmul_rows_single", st);
        kern<<<grid_for(kern, smem, tiles), NT, smem, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

// runtime log2 length -> compile-time kernel (cases outside [LO, HI] are not instantiated)
#define MM_CASE(K, LO, HI, CALL) \
    case K:                      \
        if constexpr (K >= LO && K <= HI) return CALL(K); else break;
#define MM_DISPATCH_K(k, LO, HI, CALL)                                                            \
    switch (k) {                                                                                  \
        MM_CASE(1, LO, HI, CALL) MM_CASE(2, LO, HI, CALL) MM_CASE(3, LO, HI, CALL)                \
        MM_CASE(4, LO, HI, CALL) MM_CASE(5, LO, HI, CALL) MM_CASE(6, LO, HI, CALL)                \
        MM_CASE(7, LO, HI, CALL) MM_CASE(8, LO, HI, CALL) MM_CASE(9, LO, HI, CALL)                \
        MM_CASE(10, LO, HI, CALL) MM_CASE(11, LO, HI, CALL) MM_CASE(12, LO, HI, CALL)             \
        MM_CASE(13, LO, HI, CALL)                                                                 \
        default: break;                                                                           \
    }                                                                                             \
    return set_err(MM_E_UNSUPPORTED_SIZE, "no kernel for sub-transform log2 length %d", (int)(k));

// entry points with runtime log2 length (explicitly instantiated in ntt_inst*.cu)
template <class F, bool INV, class TIn, class TOut>
mm_status launch_rows(const F& f, const RowArgs<F>& a, cudaStream_t st) {
#define MM_CALLR(K) launch_rows_k<F, K, INV, TIn, TOut>(f, a, st)
    MM_DISPATCH_K(a.k, 1, 13, MM_CALLR)
#undef MM_CALLR
}
template <class F, bool INV, class TIn, class TOut>
mm_status launch_cols(const F& f, const ColArgs<F>& a, cudaStream_t st) {
#define MM_CALLC(K) launch_cols_k<F, K, INV, TIn, TOut>(f, a, st)
    MM_DISPATCH_K(a.k, 3, 13, MM_CALLC)
#undef MM_CALLC
}
template <class F, class TIn, class TOut>
mm_status launch_pmul(const F& f, const PmulArgs<F>& a, cudaStream_t st) {
#define MM_CALLP(K) launch_pmul_k<F, K, TIn, TOut>(f, a, st)
    MM_DISPATCH_K(a.k, 1, 13, MM_CALLP)
#undef MM_CALLP
}

}  // namespace mm
