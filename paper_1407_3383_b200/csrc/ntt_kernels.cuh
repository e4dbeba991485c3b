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
//   k_cols_tma  : k_cols for 32-bit / FP64 one-row-per-column tiles with the
//                 input staged by TMA box copies.
// The Goldilocks C4 / C5 passes with TMA / bulk-copy staging live in
// gold_cols.cu and gold_rows.cu; the launchers below route to them.
//
// All sizes are template parameters (LOGL); launchers dispatch on the
// runtime log2 length.  Explicit instantiations live in ntt_inst*.cu.
#pragma once
#include <type_traits>
#include "common.h"
#include "ntt_core.cuh"
#include "gold.cuh"
#include "tma.cuh"

namespace mm {

constexpr int NT = 256;                  // threads per CTA for tile kernels
constexpr size_t SMEM_MAX = 227 * 1024;  // max dynamic shared memory per CTA on sm_100

// Goldilocks tiles of 2^11..2^13 points run gold.cuh's 8-point split with
// delayed reduction (shared-memory layout: one pad word per 64 elements)
template <class F, int LOGL> struct GoldT {
    enum { v = std::is_same<F, FpG>::value && LOGL >= 10 && LOGL <= 13 };
};
template <class T, int LOGL, int C_> struct RowLayoutG {
    static constexpr int L = 1 << LOGL;
    static constexpr int C = C_;
    static constexpr int SROW = [] {
        int s = L + (L >> 6);
        while ((s & 15) != 1) s++;      // consecutive c -> consecutive 8-byte bank pairs
        return s;
    }();
    static constexpr int ELEMS = C * SROW;
    static constexpr bool COL = false;
    __device__ __forceinline__ static int addr(int c, int j) { return c * SROW + j + (j >> 6); }
    template <int PER> __device__ __forceinline__ static void split(int ch, int& c, int& b) {
        c = ch / PER;
        b = ch % PER;
    }
    __device__ __forceinline__ static int chunk_base(int c, int base) { return c * SROW + base + (base >> 6); }
    __host__ __device__ static constexpr int off(int x) { return x + (x >> 6); }
};

// threads per CTA of the row kernels: 2^13-point Goldilocks rows fill 66 KiB of
// shared memory per row, so their CTAs take 512 threads (two per SM, 32 warps)
template <class F, int LOGL> struct NTr {
    enum { v = (GoldT<F, LOGL>::v && LOGL == 13) ? 512 : NT };
};

// column kernels: 512 threads for 2^11- and 2^12-point Goldilocks columns (66 KiB tiles)
template <class F, int LOGL> struct NTc {
    enum { v = (GoldT<F, LOGL>::v && LOGL >= 11) ? 512 : NT };
};

template <class F> struct Cfg;
template <> struct Cfg<Fp32> { enum { RL = 4, BUDGET = 8192, ROWB = 2048, COLC = 32, V = 4 }; };
template <> struct Cfg<FpG> { enum { RL = 3, BUDGET = 4096, ROWB = 4096, COLC = 16, V = 2 }; };
template <> struct Cfg<FpD> { enum { RL = 3, BUDGET = 4096, ROWB = 4096, COLC = 16, V = 2 }; };

// Column tiles of L <= 512 points use the interleaved layout [j][c] with C
// transforms of 128 bytes per row (the global row-major order of the column
// block; lane = transform: every access of every group is conflict-free
// without padding); longer columns use one padded row per transform.
template <class F, int LOGL> struct InterOK {
    enum { v = (size_t)Cfg<F>::COLC * (1u << LOGL) * sizeof(typename F::T) <= 64 * 1024 };
};
// Row tiles keep one padded row per transform: global accesses stay fully
// coalesced (the interleaved layout made every warp access touch 32 lines).
template <class F, int LOGL> struct RowsTile {
    typedef typename F::T T;
    // ROWB: elements per row tile (32-bit: 8 KiB, so that small batches -- C1's
    // 16 rows of 2^10 -- spread over more CTAs; the product tiles keep BUDGET)
    enum { C = (Cfg<F>::ROWB >> LOGL) > 0 ? (Cfg<F>::ROWB >> LOGL) : 1 };
    typedef typename std::conditional<GoldT<F, LOGL>::v, RowLayoutG<T, LOGL, C>, RowLayout<T, LOGL, C>>::type Lay;
};
template <class F, int LOGL> struct PmulTile {
    typedef typename F::T T;
    enum { C = ((Cfg<F>::BUDGET / 2) >> LOGL) > 0 ? ((Cfg<F>::BUDGET / 2) >> LOGL) : 1 };
    typedef typename std::conditional<GoldT<F, LOGL>::v, RowLayoutG<T, LOGL, C>, RowLayout<T, LOGL, C>>::type Lay;
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
    // Goldilocks columns (latency-bound passes, sized for resident warps):
    // four of 2^11 points (66 KiB, full 32-byte row segments) and two of 2^12
    // (66 KiB) with 512-thread CTAs (NTc); two of 2^10 (16 KiB, 256 threads)
    enum { C = GoldT<F, LOGL>::v ? (LOGL == 11 ? 4 : 2) : InterOK<F, LOGL>::v ? Cfg<F>::COLC : 32 / (int)sizeof(T) };
    typedef typename std::conditional<
        InterOK<F, LOGL>::v, ColLayout<T, LOGL, C>,
        typename std::conditional<GoldT<F, LOGL>::v, RowLayoutG<T, LOGL, C>, RowLayoutOdd<T, LOGL, C>>::type>::type Lay;
};

// ---------------------------------------------------------------- args
template <class F> struct RowArgs {
    typedef typename F::W W;
    const void* in;
    void* out;
    long long nrows, in_rs, out_rs, in_len, out_len, row0;
    int k, k2, perm, fs, scale, canon, vec_in, vec_out;
    int in_seg_log, out_seg_log;           // segmented rows: element j of row r at
    long long in_seg_stride, out_seg_stride; // (j >> log) * stride + r * rs + (j mod 2^log); log 0 = plain
    W sc;
    const W* lvl;
    const W* fs_lo;
    const W* fs_hi;
    const W* fs_full;     // full step-2 table [i2][j1] when small enough, else null
    int fs_h;
    long long rows_per;   // > 0: truncated transforms of rows_per rows each (TFT), i2 = row mod rows_per
};
template <class F> struct ColArgs {
    typedef typename F::W W;
    const void* in;
    void* out;
    long long ncols, nbatch, in_rs, out_rs, in_bs, out_bs, in_len, out_len, col0, n1;
    int k, fs, scale, canon, vec_in, vec_out;
    int reduce_in;        // 32-bit fields: input words are raw (any u32), reduced on load (Fp32::reduce_raw)
    W sc;
    const W* lvl;
    const W* fs_lo;
    const W* fs_hi;
    const W* fs_full;
    int fs_h;
    // peer scatter (sharded transforms): row t of the output block goes to
    // peer_out[t >> peer_shift] + t out_rs + c -- the all-to-all receive
    // buffers of the other ranks written in place (npeers = 0: plain out)
    int npeers, peer_shift;
    void* peer_out[8];
    // Remark 6: nmod > 1 moduli in one launch -- batch rows
    // [q mod_span, (q+1) mod_span) run over field fm[q] with plan q's tables
    int nmod;
    long long mod_span;
    F fm[3];
    W scm[3];
    const W* lvlm[3];
    const W* fslom[3];
    const W* fshim[3];
    const W* fsfullm[3];
};
// Goldilocks forward column pass of 2^11-point columns with TMA-staged tiles
// and step-2 twiddles (gold_cols.cu); taken by launch_cols_e when
// gold_cols_tma_ok (full-length input, one modulus; peer scatter included)
bool gold_tma_enabled();   // MMNTT_GOLD_TMA not 0 and the tensor-map encoder available
bool gold_cols_tma_ok(const ColArgs<FpG>& a);
mm_status launch_gold_cols_tma(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st);
// the same for 2^12-point columns of zero-padded 16-bit limbs (C5, gold_cols.cu)
bool gold_cols16_tma_ok(const ColArgs<FpG>& a);
// Goldilocks forward row pass of 2^13 points with bulk-copied rows (gold_rows.cu)
bool gold_rows_tma_ok(const RowArgs<FpG>& a);
mm_status launch_gold_rows_tma(const FpG& f, const RowArgs<FpG>& a, cudaStream_t st);
bool gold_rows_inv_tma_ok(const RowArgs<FpG>& a);
mm_status launch_gold_rows_inv_tma(const FpG& f, const RowArgs<FpG>& a, cudaStream_t st);
// inverse Goldilocks column passes of 2^11 / 2^12 points with TMA-staged tiles (gold_cols.cu)
bool gold_cols_inv_tma_ok(const ColArgs<FpG>& a, int logl);
mm_status launch_gold_cols_inv_tma(const FpG& f, const ColArgs<FpG>& a, int logl, int epiv, cudaStream_t st);
mm_status launch_gold_cols16_tma(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st);

template <class F> struct PmulArgs {
    typedef typename F::W W;
    const void* a;
    const void* b;
    void* c;
    long long nrows, a_rs, b_rs, c_rs, la, lb, lc, row0;
    int k, k2, fs, canon, vec_in, vec_out;
    int in_seg_log, out_seg_log;           // segmented rows for a, b (in) and c (out), as RowArgs
    long long in_seg_stride, out_seg_stride;
    W sc;                 // pointwise post-multiplier (n^-1, times 2^32 for the 32-bit REDC)
    const W* lvl_f;
    const W* lvl_i;
    const W* fs_lo;       // inverse step-2 twiddles
    const W* fs_hi;
    const W* fs_full;
    int fs_h;
    long long rows_per;   // > 0: truncated transforms of rows_per rows each (TFT), i2 = row mod rows_per
    void* scratch;        // single-buffer tiles (PmulK::SB): L words per CTA for the first spectrum
    // Remark 6: nmod > 1 moduli in one launch -- rows [q mod_span,
    // (q+1) mod_span) run over field fm[q] with plan q's tables and scale
    int nmod;
    long long mod_span;
    F fm[3];
    W scm[3];
    const W* lvlfm[3];
    const W* lvlim[3];
    const W* fslom[3];
    const W* fshim[3];
    const W* fsfullm[3];
};

// Goldilocks fused product rows of 2^13 points with bulk-copied rows (gold_rows.cu)
bool gold_pmul_rows_tma_ok(const PmulArgs<FpG>& a);
mm_status launch_gold_pmul_rows_tma(const FpG& f, const PmulArgs<FpG>& a, cudaStream_t st);

// Epilogue selector (compile time): bits 0-1 = step-2 twiddle (0 none, 1 full
// table, 2 two-level split table), bit 2 = multiply by a constant (n^-1),
// bit 3 = canonicalise to [0, p).
enum { EPI_FS_FULL = 1, EPI_FS_SPLIT = 2, EPI_SCALE = 4, EPI_CANON = 8 };

// ---------------------------------------------------------------- helpers
template <class TIn, class T> __device__ __forceinline__ T ld_conv(const TIn* p) { return (T)__ldg(p); }

template <class W> __device__ __forceinline__ void stage_twiddles(W* dst, const W* src, int L) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) dst[i] = src[i];
}

template <class T> struct Vec;
template <> struct Vec<uint32_t> { typedef uint4 type; enum { N = 4 }; };
template <> struct Vec<uint64_t> { typedef ulonglong2 type; enum { N = 2 }; };
template <> struct Vec<double> { typedef double2 type; enum { N = 2 }; };

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
template <> __device__ __forceinline__ void vget<double>(const double2& v, double* o) {
    o[0] = v.x; o[1] = v.y;
}
template <> __device__ __forceinline__ double2 vmake<double>(const double* i) { return make_double2(i[0], i[1]); }

// V consecutive twiddles (8 bytes each) with 16-byte loads
template <class W, int V> __device__ __forceinline__ void ld_wvec(const W* p, W* w) {
    static_assert(sizeof(W) == 8, "twiddles are 8 bytes");
#pragma unroll
    for (int i = 0; i < V; i += 2) {
        uint4 u = __ldg((const uint4*)(p + i));
        w[i] = *reinterpret_cast<const W*>(&u.x);
        w[i + 1] = *reinterpret_cast<const W*>(&u.z);
    }
}

template <class F, int EPIV> struct Epi {
    typedef typename F::T T;
    typedef typename F::W W;
    static constexpr int FS = EPIV & 3;
    static constexpr bool SC = (EPIV & EPI_SCALE) != 0, CN = (EPIV & EPI_CANON) != 0;
    __device__ __forceinline__ static T apply(const F& f, T x, W wf, const W* lo, const W* hi, int h, uint32_t e,
                                              const W& sc) {
        if (FS == 1) x = f.mulw(x, wf);
        if (FS == 2) {
            x = f.mulw(x, __ldg(lo + (e & ((1u << h) - 1))));
            x = f.mulw(x, __ldg(hi + (e >> h)));
        }
        if (SC) x = f.mulw(x, sc);
        if (CN) x = f.canon(x);
        return x;
    }
};

// twiddles in shared memory when the CTA stays under ~100 KiB
template <class F, int LOGL, int ELEMS, int NTAB> struct TwPlace {
    enum { SMEM = !GoldT<F, LOGL>::v &&
                  (size_t)ELEMS * sizeof(typename F::T) + (size_t)NTAB * (1u << LOGL) * sizeof(typename F::W) <= 100 * 1024 };
};

// The tile transform of a pass: Goldilocks tiles take gold.cuh's path when the
// plan's w_64 is the one it is compiled for (full = gtab + L holds w_L^e), the
// radix-2^RL groups of ntt_core.cuh otherwise.
template <class F, class Lay, int LOGL, bool INV, int NTH = NT>
__device__ __forceinline__ void run_tile(const F& f, typename F::T* s, const typename F::W* tw, const typename F::W* gtab) {
    if constexpr (GoldT<F, LOGL>::v) {
        const uint64_t* full = (const uint64_t*)gtab + (1 << LOGL);
        constexpr uint64_t W64 = INV ? gold::Pow2Val<gold::S_INV>::v : gold::Pow2Val<gold::S_FWD>::v;
        if (__ldg(full + ((1 << LOGL) >> 6)) == W64) {
            if (INV) gold::tile_dit<Lay, LOGL, NTH>((uint64_t*)s, full);
            else gold::tile_dif<Lay, LOGL, NTH>((uint64_t*)s, full);
            return;
        }
    }
    if (INV) tile_dit<F, Lay, LOGL, Cfg<F>::RL, NTH>(f, s, tw);
    else tile_dif<F, Lay, LOGL, Cfg<F>::RL, NTH>(f, s, tw);
}

// ---------------------------------------------------------------- row-tile I/O
// Vector index e -> (row c, first element j) of a row tile.  For 32-bit rows of
// >= 64 points and an even number of rows, a warp takes 16 vectors of row c
// and 16 of row c+1: with the j + (j >> 4) padding and a row pitch of 16 banks
// mod 32 every 4-byte shared access of the warp then hits a distinct bank
// (the plain mapping gave 2-way conflicts).  Global accesses stay 256-byte
// contiguous per half-warp.
template <class T, class Lay, int LOGL> struct RowVecMap {
    static constexpr int L = 1 << LOGL, V = Vec<T>::N, VR = L / V, C = Lay::C;
    static constexpr bool PAIRED = sizeof(T) == 4 && VR >= 16 && (C % 2) == 0;
    __device__ __forceinline__ static void map(int e, int& c, int& j) {
        if constexpr (PAIRED) {
            constexpr int NCH = VR / 16;
            const int hl = e & 15, hw = (e >> 4) & 1, rest = e >> 5;
            const int rp = rest / NCH, k = rest % NCH;
            c = 2 * rp + hw;
            j = (16 * k + hl) * V;
        } else {
            c = (e * V) >> LOGL;
            j = (e * V) & (L - 1);
        }
    }
};

// offset of element j within a (possibly segmented) row
__device__ __forceinline__ long long seg_j(int j, int seglog, long long segstride) {
    return seglog ? (long long)(j >> seglog) * segstride + (j & ((1 << seglog) - 1)) : (long long)j;
}

// cp.async (LDGSTS) helpers: 16-byte copies global -> shared, zero-filling the
// bytes beyond src_bytes (0 -> the destination is zeroed, nothing is read)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// Rows [r0, r0 + C) of a row-major array (row stride rs, valid prefix len per
// row, zeros beyond) -> padded row tile; consecutive lanes take consecutive
// 16-byte vectors of a row (fully coalesced).  A thread issues up to 4
// vector loads before its shared stores.
template <class F, class Lay, int LOGL, class TIn, int NTH = NT>
__device__ __forceinline__ void load_rows(typename F::T* s, const TIn* in, long long r0, long long nrows, long long rs,
                                          long long len64, bool vec, bool perm, int seglog = 0, long long segstride = 0) {
    typedef typename F::T T;
    typedef typename Vec<T>::type TV;
    constexpr int L = 1 << LOGL, C = Lay::C, V = Vec<T>::N;
    // rows of this tile that exist and the valid prefix, clamped to the tile
    // (32-bit compares in the per-vector tests below)
    const int rlim = nrows - r0 < C ? (int)(nrows - r0) : C;
    const int len = len64 < L ? (int)len64 : L;
    if (L >= V && sizeof(TIn) == sizeof(T) && vec && !perm) {
        constexpr int TOT = C * L / V;
        constexpr int NV = (TOT + NTH - 1) / NTH;
        constexpr int B = NV < 4 ? NV : 4;
        const T* tb = (const T*)in + r0 * rs;
#pragma unroll
        for (int u0 = 0; u0 < NV; u0 += B) {
            TV buf[B];
            int mode[B];                                      // 0 zero, 1 full, 2 partial
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e = threadIdx.x + (u0 + u) * NTH;
                int c, j;
                RowVecMap<T, Lay, LOGL>::map(e, c, j);
                const bool rowok = e < TOT && c < rlim;
                mode[u] = !rowok || j >= len ? 0 : (j + V <= len ? 1 : 2);
                buf[u] = __ldg((const TV*)(mode[u] == 1 ? tb + (unsigned)c * (unsigned)rs + seg_j(j, seglog, segstride)
                                                        : (const T*)in));
            }
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e = threadIdx.x + (u0 + u) * NTH;
                if (e >= TOT) continue;
                int c, j;
                RowVecMap<T, Lay, LOGL>::map(e, c, j);
                T v[V];
                vget<T>(buf[u], v);
                if (mode[u] != 1) {
#pragma unroll
                    for (int i = 0; i < V; i++)
                        v[i] = (mode[u] == 2 && j + i < len)
                                   ? __ldg(tb + (unsigned)c * (unsigned)rs + seg_j(j + i, seglog, segstride)) : (T)0;
                }
#pragma unroll
                for (int i = 0; i < V; i++) s[Lay::addr(c, j + i)] = v[i];
            }
        }
    } else {
        for (int e = threadIdx.x; e < C * L; e += NTH) {
            const int c = e >> LOGL, j = e & (L - 1);
            T v = 0;
            if (c < rlim && j < len) v = ld_conv<TIn, T>(in + (r0 + c) * rs + seg_j(j, seglog, segstride));
            s[Lay::addr(c, perm ? brev(j, LOGL) : j)] = v;
        }
    }
}

// epilogue + stores of a row tile (step-2 twiddle rows are contiguous in the
// full table: one or two 16-byte loads per vector)
template <class F, class Lay, int LOGL, class TOut, int EPIV, int NTH = NT>
__device__ __forceinline__ void store_rows(const F& f, const typename F::T* s, TOut* out, long long r0, long long nrows,
                                           long long rs, long long len64, bool vec, bool perm, const typename F::W* fs_full,
                                           const typename F::W* fs_lo, const typename F::W* fs_hi, int fs_h,
                                           long long row0, int k2, const typename F::W& sc, int seglog = 0,
                                           long long segstride = 0, long long rows_per = 0) {
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename Vec<T>::type TV;
    typedef Epi<F, EPIV> E;
    constexpr int L = 1 << LOGL, C = Lay::C, V = Vec<T>::N;
    const int rlim = nrows - r0 < C ? (int)(nrows - r0) : C;
    const int len = len64 < L ? (int)len64 : L;
    const unsigned i2mask = (1u << k2) - 1;
    const unsigned i2b = (unsigned)((row0 + r0) & i2mask);
    // frequency row of tile row c (a truncated transform keeps rows_per rows per transform)
    auto i2_of = [&](int c) -> unsigned {
        return rows_per ? (unsigned)((row0 + r0 + c) % rows_per) : ((i2b + (unsigned)c) & i2mask);
    };
    if (L >= V && sizeof(TOut) == sizeof(T) && vec && !perm) {
        constexpr int TOT = C * L / V;
        constexpr int NV = (TOT + NTH - 1) / NTH;
        constexpr int B = NV < 2 ? NV : 2;
        T* ob = (T*)out + r0 * rs;
#pragma unroll
        for (int u0 = 0; u0 < NV; u0 += B) {
            T v[B][V];
            W w[B][V];
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e0 = threadIdx.x + (u0 + u) * NTH;
                const int e = e0 < TOT ? e0 : 0;                  // idle lanes read a valid slot
                int c, j;
                RowVecMap<T, Lay, LOGL>::map(e, c, j);
#pragma unroll
                for (int i = 0; i < V; i++) v[u][i] = s[Lay::addr(c, j + i)];
                if (E::FS == 1) ld_wvec<W, V>(fs_full + i2_of(c) * L + j, w[u]);
            }
#pragma unroll
            for (int u = 0; u < B; u++) {
                const int e = threadIdx.x + (u0 + u) * NTH;
                int c, j;
                RowVecMap<T, Lay, LOGL>::map(e < TOT ? e : 0, c, j);
                if (e >= TOT || c >= rlim || j >= len) continue;
                const unsigned i2r = brev((int)i2_of(c), k2);
#pragma unroll
                for (int i = 0; i < V; i++) v[u][i] = E::apply(f, v[u][i], w[u][i], fs_lo, fs_hi, fs_h, (unsigned)(j + i) * i2r, sc);
                if (j + V <= len) {
                    *(TV*)(ob + (unsigned)c * (unsigned)rs + seg_j(j, seglog, segstride)) = vmake<T>(v[u]);
                } else {
#pragma unroll
                    for (int i = 0; i < V; i++)
                        if (j + i < len) ob[(unsigned)c * (unsigned)rs + seg_j(j + i, seglog, segstride)] = v[u][i];
                }
            }
        }
    } else {
        for (int e = threadIdx.x; e < C * L; e += NTH) {
            const int c = e >> LOGL, j = e & (L - 1);
            if (c >= rlim || j >= len) continue;
            const unsigned i2 = i2_of(c);
            W wf{};
            if (E::FS == 1) wf = __ldg(fs_full + i2 * L + j);
            T x = E::apply(f, s[Lay::addr(c, perm ? brev(j, LOGL) : j)], wf, fs_lo, fs_hi, fs_h,
                           (unsigned)j * (unsigned)brev((int)i2, k2), sc);
            out[(r0 + c) * rs + seg_j(j, seglog, segstride)] = (TOut)x;
        }
    }
}

// ---------------------------------------------------------------- row pass
template <class F, int LOGL> struct RowsK {
    typedef typename RowsTile<F, LOGL>::Lay Lay;
    enum { TWS = TwPlace<F, LOGL, Lay::ELEMS, 1>::SMEM };
    static constexpr size_t smem() {
        return (size_t)Lay::ELEMS * sizeof(typename F::T) + (TWS ? (size_t)(1u << LOGL) * sizeof(typename F::W) : 0);
    }
};

template <class F, int LOGL, bool INV, class TIn, class TOut, int EPIV>
__global__ void __launch_bounds__(NTr<F, LOGL>::v, 1024 / NTr<F, LOGL>::v) k_rows(F f, RowArgs<F> a) {
    constexpr int NTH = NTr<F, LOGL>::v;
    typedef typename F::T T;
    typedef typename F::W W;
    typedef RowsK<F, LOGL> K;
    typedef typename K::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int C = Lay::C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* tws = (W*)smem_raw;
    T* s = (T*)(tws + (K::TWS ? L : 0));
    if (K::TWS) stage_twiddles(tws, a.lvl, L);
    const W* tw = K::TWS ? (const W*)tws : a.lvl;
    const long long ntiles = (a.nrows + C - 1) / C;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long r0 = tile * C;
        load_rows<F, Lay, LOGL, TIn, NTH>(s, (const TIn*)a.in, r0, a.nrows, a.in_rs, a.in_len, a.vec_in, INV && a.perm,
                                     a.in_seg_log, a.in_seg_stride);
        __syncthreads();
        run_tile<F, Lay, LOGL, INV, NTH>(f, s, tw, a.lvl);
        store_rows<F, Lay, LOGL, TOut, EPIV, NTH>(f, s, (TOut*)a.out, r0, a.nrows, a.out_rs, a.out_len, a.vec_out,
                                             !INV && a.perm, a.fs_full, a.fs_lo, a.fs_hi, a.fs_h, a.row0, a.k2, a.sc,
                                             a.out_seg_log, a.out_seg_stride, a.rows_per);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- column pass
template <class F, int LOGL> struct ColsK {
    typedef typename ColsTile<F, LOGL>::Lay Lay;
    // interleaved column tiles are double-buffered with cp.async (the next
    // tile streams in while the current one is transformed)
    enum { PIPE = Lay::COL ? 1 : 0 };
    enum { TWS = TwPlace<F, LOGL, (PIPE ? 2 : 1) * Lay::ELEMS, 1>::SMEM };
    // Goldilocks forward columns of 2^12 points (C5): the step-2 twiddle
    // w^(j1 k) of frequency k = k_lo + 2^LO k_hi is formed on chip as
    // T_lo[k_lo] T_hi[k_hi] from 2^LO + 2^HI table entries per column, loaded
    // with the tile; the full-table loads at the store are 16-byte segments per
    // row whose latency the tile waits for (C5 column passes 1.09 -> 1.00 ms).
    // For C4's 2^11-point tiles of four columns the extra product costs more
    // than the wait (1.70 -> 1.77 ms): they keep the table.
    enum { LO = LOGL / 2, NLO = 1 << LO, NHI = 1 << (LOGL - LO), NOTF = NLO + NHI };
    enum { OTF = GoldT<F, LOGL>::v && LOGL == 12 };
    static constexpr size_t smem() {
        return (PIPE ? 2 : 1) * (size_t)Lay::ELEMS * sizeof(typename F::T) +
               (TWS ? (size_t)(1u << LOGL) * sizeof(typename F::W) : 0) +
               (OTF ? (size_t)Lay::C * NOTF * sizeof(typename F::W) : 0);
    }
};

// rows t of a column tile with linear index t n1 + lin0 + [0, C): fully valid for
// t < *full, fully beyond the valid prefix for t >= *zero
__device__ __forceinline__ void col_rows_valid(long long len, long long lin0, long long n1, int C, int L, int* full,
                                               int* zero) {
    long long f = len - lin0 - C;
    long long fr = f < 0 ? 0 : f / n1 + 1;
    long long z = len - lin0;
    long long zr = z <= 0 ? 0 : (z + n1 - 1) / n1;
    *full = (int)(fr < L ? fr : L);
    *zero = (int)(zr < L ? zr : L);
}

template <class F, int LOGL, bool INV, class TIn, class TOut, int EPIV>
__global__ void __launch_bounds__(NTc<F, LOGL>::v, 1024 / NTc<F, LOGL>::v) k_cols(F f, ColArgs<F> a) {
    constexpr int NTH = NTc<F, LOGL>::v;
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename Vec<T>::type TV;
    typedef ColsK<F, LOGL> K;
    typedef typename K::Lay Lay;
    typedef Epi<F, EPIV> E;
    constexpr int L = 1 << LOGL;
    constexpr int C = Lay::C;
    constexpr int V = Vec<T>::N;
    constexpr int CV = C / V;        // vectors per tile row
    constexpr int TOT = L * CV;
    constexpr int NV = (TOT + NTH - 1) / NTH;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* tws = (W*)smem_raw;
    T* s = (T*)(tws + (K::TWS ? L : 0));
    constexpr bool OTF = K::OTF && !INV && E::FS == 1;
    W* otf = (W*)(s + (K::PIPE ? 2 : 1) * Lay::ELEMS);       // [c][T_lo (NLO) | T_hi (NHI)]
    if (K::TWS) stage_twiddles(tws, a.lvl, L);
    const W* tw = K::TWS ? (const W*)tws : a.lvl;
    const long long cgroups = a.ncols / C;                 // host guarantees ncols % C == 0
    const long long ntiles = cgroups * a.nbatch;
    // the modulus of the current tile (Remark 6): field, tables, scale
    F ff = f;
    const W* lvl = a.lvl;
    const W* fsf = a.fs_full;
    const W* fslo = a.fs_lo;
    const W* fshi = a.fs_hi;
    W sc = a.sc;
    int curq = 0;
    const unsigned irs = (unsigned)a.in_rs, ors = (unsigned)a.out_rs, n1 = (unsigned)a.n1;
    constexpr bool PIPE = K::PIPE && sizeof(TIn) == sizeof(T);
    const bool pipe = PIPE && a.vec_in && !a.reduce_in;   // cp.async lands words unseen: no reduction on load
    // cp.async the whole column tile `tile` into dst (zero-fill beyond in_len)
    // tiles run column-group-major (tile = cg nbatch + b): the nbatch tiles of one
    // column group are in flight together and share their step-2 table segment
    // (w^(j1 [i2]) does not depend on the batch row) through L2.  Several
    // moduli (different tables per batch row): batch-major, so a CTA restages
    // its twiddles only when its tiles cross into the next modulus.
    const bool bmajor = a.nmod > 1;
    auto issue = [&](long long tile, T* dst) {
        const long long b = bmajor ? tile / cgroups : tile % a.nbatch;
        const long long cl0 = (bmajor ? tile % cgroups : tile / a.nbatch) * C;
        const long long lin0 = a.col0 + cl0;
        const T* tb = (const T*)a.in + b * a.in_bs + cl0;
        int tfull, tzero;
        col_rows_valid(a.in_len, lin0, a.n1, C, L, &tfull, &tzero);
#pragma unroll
        for (int u = 0; u < NV; u++) {
            const int e = threadIdx.x + u * NTH;
            if (e >= TOT) continue;
            const int t = e / CV, c = (e % CV) * V;
            int nb = 16;
            if (t >= tfull) {
                long long rem = t < tzero ? a.in_len - ((long long)t * a.n1 + lin0 + c) : 0;
                nb = rem <= 0 ? 0 : (rem >= V ? 16 : (int)rem * (int)sizeof(T));
            }
            cp_async16(dst + Lay::addr(c, t), nb ? (const void*)(tb + (unsigned)t * irs + c) : a.in, nb);
        }
    };
    int it = 0;
    if (pipe) {
        if ((long long)blockIdx.x < ntiles) issue(blockIdx.x, s);
        cp_async_commit();
    }
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        const long long b = bmajor ? tile / cgroups : tile % a.nbatch;
        const long long cl0 = (bmajor ? tile % cgroups : tile / a.nbatch) * C;
        const long long lin0 = a.col0 + cl0;        // logical column of c = 0
        if (bmajor) {
            const int q = (int)(b / a.mod_span);
            if (q != curq || tile == blockIdx.x) {
                curq = q;
                ff = a.fm[q];
                lvl = a.lvlm[q];
                fsf = a.fsfullm[q];
                fslo = a.fslom[q];
                fshi = a.fshim[q];
                sc = a.scm[q];
                if (K::TWS) {
                    __syncthreads();
                    stage_twiddles(tws, lvl, L);
                    __syncthreads();
                } else {
                    tw = lvl;
                }
            }
        }
        const TIn* inb = (const TIn*)a.in + b * a.in_bs + cl0;
        int tfull, tzero;
        T* cur = s;
        // this tile's step-2 bases T_lo[c][m] = w^(j1 m), T_hi[c][h] = w^(j1 2^LO h):
        // entries of the full table at rows brev(m), brev(2^LO h); in flight with
        // the tile's loads, stored before the barrier that precedes the transform
        W otf_v{};
        if constexpr (OTF) {
            static_assert(C * K::NOTF <= NTH, "one step-2 base per thread");
            if (threadIdx.x < C * K::NOTF) {
                const int c = threadIdx.x / K::NOTF, r = threadIdx.x % K::NOTF;
                const int row = r < K::NLO ? r : (r - K::NLO) << K::LO;
                otf_v = __ldg(fsf + (unsigned)brev(row, LOGL) * n1 + (unsigned)lin0 + c);
            }
        }
        if (pipe) {
            cur = s + (it & 1) * Lay::ELEMS;
            const long long nxt = tile + gridDim.x;
            if (nxt < ntiles) issue(nxt, s + ((it + 1) & 1) * Lay::ELEMS);
            cp_async_commit();
            cp_async_wait<1>();
        } else if (a.vec_in && sizeof(TIn) == sizeof(T)) {
            col_rows_valid(a.in_len, lin0, a.n1, C, L, &tfull, &tzero);
            constexpr int B = NV < 4 ? NV : 4;
            const T* tb = (const T*)inb;
#pragma unroll
            for (int u0 = 0; u0 < NV; u0 += B) {
                TV buf[B];
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e = threadIdx.x + (u0 + u) * NTH;
                    const int t = e / CV, c = (e % CV) * V;
                    buf[u] = __ldg((const TV*)(e < TOT && t < tfull ? tb + (unsigned)t * irs + c : (const T*)a.in));
                }
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e = threadIdx.x + (u0 + u) * NTH;
                    if (e >= TOT) continue;
                    const int t = e / CV, c = (e % CV) * V;
                    T v[V];
                    vget<T>(buf[u], v);
                    if (t >= tfull) {
#pragma unroll
                        for (int i = 0; i < V; i++)
                            v[i] = (t < tzero && (long long)t * a.n1 + lin0 + c + i < a.in_len)
                                       ? __ldg(tb + (unsigned)t * irs + c + i) : (T)0;
                    }
                    if constexpr (std::is_same<F, Fp32>::value)
                        if (a.reduce_in) {
#pragma unroll
                            for (int i = 0; i < V; i++) v[i] = ff.reduce_raw(v[i]);
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
            // element loads (narrow or unaligned input, e.g. 16-bit limbs): up
            // to eight in flight per thread before the shared stores
            col_rows_valid(a.in_len, lin0, a.n1, C, L, &tfull, &tzero);
            constexpr int TOTE = L * C, NE = (TOTE + NTH - 1) / NTH, BE = NE < 8 ? NE : 8;
            for (int u0 = 0; u0 < NE; u0 += BE) {
                T v[BE];
#pragma unroll
                for (int u = 0; u < BE; u++) {
                    const int e = threadIdx.x + (u0 + u) * NTH;
                    const int t = e / C, c = e % C;
                    v[u] = 0;
                    if (e < TOTE && (t < tfull || (t < tzero && (long long)t * a.n1 + lin0 + c < a.in_len)))
                        v[u] = ld_conv<TIn, T>(inb + (unsigned)t * irs + c);
                    if constexpr (std::is_same<F, Fp32>::value)
                        if (a.reduce_in) v[u] = ff.reduce_raw(v[u]);
                }
#pragma unroll
                for (int u = 0; u < BE; u++) {
                    const int e = threadIdx.x + (u0 + u) * NTH;
                    if (e < TOTE) s[Lay::addr(e % C, e / C)] = v[u];
                }
            }
        }
        if constexpr (OTF)
            if (threadIdx.x < C * K::NOTF) otf[threadIdx.x] = otf_v;
        __syncthreads();
        run_tile<F, Lay, LOGL, INV, NTH>(ff, cur, tw, lvl);
        col_rows_valid(a.out_len, lin0, a.n1, C, L, &tfull, &tzero);
        TOut* outb = (TOut*)a.out + b * a.out_bs + cl0;
        if (a.vec_out && sizeof(TOut) == sizeof(T)) {
            constexpr int B = NV < 2 ? NV : 2;
            T* ob = (T*)outb;
#pragma unroll
            for (int u0 = 0; u0 < NV; u0 += B) {
                T v[B][V];
                W w[B][V];
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e0 = threadIdx.x + (u0 + u) * NTH;
                    const int e = e0 < TOT ? e0 : 0;
                    const int t = e / CV, c = (e % CV) * V;
                    if (Lay::COL) vget<T>(*(const TV*)(cur + Lay::addr(c, t)), v[u]);
                    else {
#pragma unroll
                        for (int i = 0; i < V; i++) v[u][i] = cur[Lay::addr(c + i, t)];
                    }
                    if constexpr (OTF) {
                        const unsigned k = (unsigned)brev(t, LOGL);
#pragma unroll
                        for (int i = 0; i < V; i++)
                            w[u][i] = FpG::mul(otf[(c + i) * K::NOTF + (k & (K::NLO - 1))],
                                               otf[(c + i) * K::NOTF + K::NLO + (k >> K::LO)]);
                    } else if (E::FS == 1) {
                        ld_wvec<W, V>(fsf + (unsigned)t * n1 + (unsigned)lin0 + c, w[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < B; u++) {
                    const int e = threadIdx.x + (u0 + u) * NTH;
                    if (e >= TOT) continue;
                    const int t = e / CV, c = (e % CV) * V;
                    if (t >= tzero) continue;
                    const unsigned bt = (unsigned)brev(t, LOGL);
#pragma unroll
                    for (int i = 0; i < V; i++)
                        v[u][i] = E::apply(ff, v[u][i], w[u][i], fslo, fshi, a.fs_h,
                                           ((unsigned)lin0 + c + i) * bt, sc);
                    if (a.npeers) {         // fused transpose: store into the owning rank's receive buffer
                        T* pb = (T*)a.peer_out[t >> a.peer_shift] + cl0;
                        *(TV*)(pb + (unsigned)t * ors + c) = vmake<T>(v[u]);
                    } else if (t < tfull) {
                        *(TV*)(ob + (unsigned)t * ors + c) = vmake<T>(v[u]);
                    } else {
#pragma unroll
                        for (int i = 0; i < V; i++)
                            if ((long long)t * a.n1 + lin0 + c + i < a.out_len) ob[(unsigned)t * ors + c + i] = v[u][i];
                    }
                }
            }
        } else {
            for (int e = threadIdx.x; e < L * C; e += NTH) {
                const int t = e / C, c = e % C;
                if (t >= tzero || (t >= tfull && (long long)t * a.n1 + lin0 + c >= a.out_len)) continue;
                W wf{};
                if constexpr (OTF) {
                    const unsigned k = (unsigned)brev(t, LOGL);
                    wf = FpG::mul(otf[c * K::NOTF + (k & (K::NLO - 1))], otf[c * K::NOTF + K::NLO + (k >> K::LO)]);
                } else if (E::FS == 1) {
                    wf = __ldg(fsf + (unsigned)t * n1 + (unsigned)lin0 + c);
                }
                T x = E::apply(ff, cur[Lay::addr(c, t)], wf, fslo, fshi, a.fs_h,
                               ((unsigned)lin0 + c) * (unsigned)brev(t, LOGL), sc);
                outb[(unsigned)t * ors + c] = (TOut)x;
            }
        }
        __syncthreads();
    }
    // fused transpose: order this thread's peer stores system-wide before the
    // stream's next kernel raises the ready flags (dist.cu k_dist_signal)
    if (a.npeers) __threadfence_system();
}

// ---------------------------------------------------------------- column pass, TMA-staged (32-bit / FP64)
// The generic column pass for tiles of C columns stored as one padded row
// per column (RowLayoutOdd: 2^10-point 32-bit columns, 2^10 / 2^11-point
// FP64 columns -- the 32-bit n >= 2^20 and FP64 n >= 2^20 plans) with its
// input staged by TMA instead of per-thread loads: L / 256 box copies {C
// columns, 256 rows} land the tile ([row][C], 32 / 64-byte row segments,
// rows beyond the valid prefix zero-filled) a tile ahead, the landing buffer
// is copied into the padded tile (lanes: columns fastest; raw 32-bit words
// reduced on the way for the three-prime product) and the next tile streams
// in under the transform.  Same tiles, layouts, twiddles and epilogues as
// k_cols (a per-tile modulus for Remark 6 batches).
template <class F, int LOGL> struct ColsTmaK {
    typedef typename ColsTile<F, LOGL>::Lay Lay;
    typedef typename F::T T;
    static constexpr int L = 1 << LOGL, C = Lay::C, BOXR = 256, NB = L / BOXR;
    static constexpr unsigned LAND_BYTES = (unsigned)L * C * sizeof(T);
    enum { OK = !Lay::COL && !GoldT<F, LOGL>::v && LOGL >= 8 && (C * sizeof(T)) % 16 == 0 };
    enum { TWS = ColsK<F, LOGL>::TWS };
    static constexpr size_t smem() {
        return LAND_BYTES + (size_t)Lay::ELEMS * sizeof(T) + (TWS ? (size_t)L * sizeof(typename F::W) : 0) + 16;
    }
};

template <class F, int LOGL, bool INV, int EPIV>
__global__ void __launch_bounds__(NT, 3) k_cols_tma(const __grid_constant__ CUtensorMap tm, F f, ColArgs<F> a) {
    typedef ColsTmaK<F, LOGL> K;
    typedef typename K::Lay Lay;
    typedef typename F::T T;
    typedef typename F::W W;
    typedef typename Vec<T>::type TV;
    typedef Epi<F, EPIV> E;
    constexpr int L = K::L, C = K::C, V = Vec<T>::N, CV = C / V, TOT = L * CV;
    extern __shared__ __align__(1024) unsigned char smem_tma[];   // own name: the 16-byte smem_raw of the other kernels would override the alignment
    T* land = (T*)smem_tma;
    T* s = land + L * C;
    W* tws = (W*)(s + Lay::ELEMS);
    uint64_t* bar = (uint64_t*)(tws + (K::TWS ? L : 0));
    const long long cgroups = a.ncols / C, ntiles = cgroups * a.nbatch;
    const bool bmajor = a.nmod > 1;
    const bool bsel = a.in_bs != 0;            // 0: every batch row reads the same input (three-prime raw limbs)
    auto coords = [&](long long tile, long long& b, long long& cl0) {
        b = bmajor ? tile / cgroups : tile % a.nbatch;
        cl0 = (bmajor ? tile % cgroups : tile / a.nbatch) * C;
    };
    auto issue = [&](long long tile) {
        long long b, cl0;
        coords(tile, b, cl0);
        mbar_arrive_tx(&bar[0], K::LAND_BYTES);
        for (int i = 0; i < K::NB; i++)
            tma_load_box3(land + i * K::BOXR * C, &tm, (int)cl0, i * K::BOXR, bsel ? (int)b : 0, &bar[0]);
    };
    F ff = f;
    const W* lvl = a.lvl;
    const W* fsf = a.fs_full;
    const W* fslo = a.fs_lo;
    const W* fshi = a.fs_hi;
    W sc = a.sc;
    int curq = -1;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_fence_init();
        if ((long long)blockIdx.x < ntiles) issue(blockIdx.x);
    }
    if (K::TWS && !bmajor) stage_twiddles(tws, lvl, L);
    __syncthreads();
    const W* tw = K::TWS ? (const W*)tws : lvl;
    const unsigned ors = (unsigned)a.out_rs;
    int it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        long long b, cl0;
        coords(tile, b, cl0);
        const long long lin0 = a.col0 + cl0;
        if (bmajor) {   // the modulus of this tile (Remark 6)
            const int q = (int)(b / a.mod_span);
            if (q != curq) {
                curq = q;
                ff = a.fm[q];
                lvl = a.lvlm[q];
                fsf = a.fsfullm[q];
                fslo = a.fslom[q];
                fshi = a.fshim[q];
                sc = a.scm[q];
                if (K::TWS) {
                    __syncthreads();
                    stage_twiddles(tws, lvl, L);
                    __syncthreads();
                } else {
                    tw = lvl;
                }
            }
        }
        mbar_wait(&bar[0], it & 1);
        for (int e = threadIdx.x; e < L * C; e += NT) {
            T v = land[e];
            if constexpr (std::is_same<F, Fp32>::value)
                if (a.reduce_in) v = ff.reduce_raw(v);
            s[Lay::addr(e % C, e / C)] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x);
        run_tile<F, Lay, LOGL, INV, NT>(ff, s, tw, lvl);
        int tfull, tzero;
        col_rows_valid(a.out_len, lin0, a.n1, C, L, &tfull, &tzero);
        T* ob = (T*)a.out + b * a.out_bs + cl0;
        for (int e = threadIdx.x; e < TOT; e += NT) {
            const int t = e / CV, c = (e % CV) * V;
            if (t >= tzero) continue;
            T v[V];
            W w[V];
#pragma unroll
            for (int i = 0; i < V; i++) v[i] = s[Lay::addr(c + i, t)];
            if (E::FS == 1) ld_wvec<W, V>(fsf + (unsigned)t * (unsigned)a.n1 + (unsigned)lin0 + c, w);
            const unsigned bt = (unsigned)brev(t, LOGL);
#pragma unroll
            for (int i = 0; i < V; i++) v[i] = E::apply(ff, v[i], w[i], fslo, fshi, a.fs_h, ((unsigned)lin0 + c + i) * bt, sc);
            if (t < tfull) {
                *(TV*)(ob + (unsigned)t * ors + c) = vmake<T>(v);
            } else {
#pragma unroll
                for (int i = 0; i < V; i++)
                    if ((long long)t * a.n1 + lin0 + c + i < a.out_len) ob[(unsigned)t * ors + c + i] = v[i];
            }
        }
        __syncthreads();
    }
}

// TMA view of the column input: {ncols (block), valid rows, batch rows}; the
// valid prefix must end on a row boundary (rows past it are zero-filled)
static inline bool cols_tma_on() {
    static const bool on = [] {
        const char* e = getenv("MMNTT_TMA_COLS");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <class F, int LOGL> static bool cols_tma_ok(const ColArgs<F>& a) {
    typedef typename F::T T;
    return cols_tma_on() && tma_encoder() != nullptr && a.npeers == 0 && a.vec_in && a.vec_out && a.n1 > 0 &&
           a.in_len % a.n1 == 0 && a.in_len > 0 && (a.in_rs * (long long)sizeof(T)) % 16 == 0 &&
           ((a.in_bs * (long long)sizeof(T)) % 16 == 0) && a.in_rs >= a.ncols && a.nbatch < (1ll << 31) &&
           a.ncols < (1ll << 31) && (a.in_bs == 0 || a.in_bs >= (a.in_len / a.n1) * a.in_rs);
}
template <class F, int LOGL, bool INV, int EPIV>
static mm_status launch_cols_tma(const F& f, const ColArgs<F>& a, cudaStream_t st) {
    typedef ColsTmaK<F, LOGL> K;
    typedef typename F::T T;
    auto enc = tma_encoder();
    const long long rows = a.in_len / a.n1 < K::L ? a.in_len / a.n1 : K::L;
    const long long nb = a.in_bs ? a.nbatch : 1;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    cuuint64_t dims[3] = {(cuuint64_t)a.ncols, (cuuint64_t)rows, (cuuint64_t)nb};
    cuuint64_t strides[2] = {(cuuint64_t)a.in_rs * sizeof(T), (cuuint64_t)(a.in_bs ? a.in_bs : a.in_rs * rows) * sizeof(T)};
    cuuint32_t box[3] = {(cuuint32_t)K::C, (cuuint32_t)K::BOXR, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 3,
                     const_cast<void*>(a.in), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(MM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    auto kern = k_cols_tma<F, LOGL, INV, EPIV>;
    const size_t smem = K::smem();
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long tiles = a.ncols / K::C * a.nbatch;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    if (per_sm < 1) per_sm = 1;
    const long long cap = (long long)num_sms() * per_sm;
    {
        LaunchScope ls(INV ? "ntt_cols_inv" : "ntt_cols_fwd", st);
        kern<<<(int)(tiles < cap ? tiles : cap), NT, smem, st>>>(tm, f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

// ---------------------------------------------------------------- fused product rows
template <class F, int LOGL> struct PmulK {
    typedef typename PmulTile<F, LOGL>::Lay Lay;
    // SB: one 2^13-point Goldilocks row in shared memory at a time (66 KiB, three
    // CTAs per SM instead of one): the first operand's spectrum waits in a
    // per-CTA L2-resident scratch row while the second is transformed
    enum { SB = GoldT<F, LOGL>::v && LOGL == 13 };
    enum { TWS = TwPlace<F, LOGL, (SB ? 1 : 2) * Lay::ELEMS, 2>::SMEM };
    static constexpr size_t smem() {
        return (SB ? 1 : 2) * (size_t)Lay::ELEMS * sizeof(typename F::T) +
               (TWS ? 2 * (size_t)(1u << LOGL) * sizeof(typename F::W) : 0);
    }
};

template <class F, int LOGL, class TIn, class TOut, int EPIV>
__global__ void __launch_bounds__(NTr<F, LOGL>::v, NTr<F, LOGL>::v == 512 ? 2 : 3) k_rows_pmul(F f, PmulArgs<F> a) {
    constexpr int NTH = NTr<F, LOGL>::v;
    typedef typename F::T T;
    typedef typename F::W W;
    typedef PmulK<F, LOGL> K;
    typedef typename K::Lay Lay;
    constexpr int L = 1 << LOGL;
    constexpr int C = Lay::C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* twfs = (W*)smem_raw;
    W* twis = twfs + (K::TWS ? L : 0);
    T* sa = (T*)(twis + (K::TWS ? L : 0));
    T* sb = sa + Lay::ELEMS;
    if (K::TWS) {
        stage_twiddles(twfs, a.lvl_f, L);
        stage_twiddles(twis, a.lvl_i, L);
    }
    const W* twf = K::TWS ? (const W*)twfs : a.lvl_f;
    const W* twi = K::TWS ? (const W*)twis : a.lvl_i;
    if (K::SB && a.nmod > 1) return;   // host never combines them (Goldilocks 2^13 rows: one modulus)
    const long long ntiles = (a.nrows + C - 1) / C;
    if constexpr (K::SB) {
        static_assert(C == 1, "single-buffer product tiles hold one row");
        // spectrum of a -> scratch row (same thread writes and reads element j:
        // plain loads, program order, no fence)
        T* scr = (T*)a.scratch + (size_t)blockIdx.x * L;
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const long long r0 = tile;
            // both operands through ONE copy of the forward tile code (a loop,
            // not two inlined calls: the 2^13-point tile is large enough that
            // two copies plus the inverse missed in the instruction cache)
#pragma unroll 1
            for (int op = 0; op < 2; op++) {
                load_rows<F, Lay, LOGL, TIn, NTH>(sa, (const TIn*)(op ? a.b : a.a), r0, a.nrows, op ? a.b_rs : a.a_rs,
                                             op ? a.lb : a.la, a.vec_in, false, a.in_seg_log, a.in_seg_stride);
                __syncthreads();
                run_tile<F, Lay, LOGL, false, NTH>(f, sa, twf, a.lvl_f);
                for (int j = 2 * threadIdx.x; j < L; j += 2 * NTH) {
                    const int ix = Lay::addr(0, j);            // j even: j, j + 1 share a 64-block
                    if (op == 0) {
                        *(ulonglong2*)(scr + j) = make_ulonglong2(sa[ix], sa[ix + 1]);
                    } else {
                        const ulonglong2 u = *(const ulonglong2*)(scr + j);
                        sa[ix] = f.mulw(f.mul_redc((T)u.x, sa[ix]), a.sc);
                        sa[ix + 1] = f.mulw(f.mul_redc((T)u.y, sa[ix + 1]), a.sc);
                    }
                }
                __syncthreads();
            }
            run_tile<F, Lay, LOGL, true, NTH>(f, sa, twi, a.lvl_i);
            store_rows<F, Lay, LOGL, TOut, EPIV, NTH>(f, sa, (TOut*)a.c, r0, a.nrows, a.c_rs, a.lc, a.vec_out, false,
                                                 a.fs_full, a.fs_lo, a.fs_hi, a.fs_h, a.row0, a.k2, a.sc,
                                                 a.out_seg_log, a.out_seg_stride, a.rows_per);
            __syncthreads();
        }
        return;
    }
    // the modulus of the current tile (Remark 6): rows of one tile never
    // straddle two moduli (host: mod_span % C == 0)
    F ff = f;
    const W* lvlf = a.lvl_f;
    const W* lvli = a.lvl_i;
    const W* fsf = a.fs_full;
    const W* fslo = a.fs_lo;
    const W* fshi = a.fs_hi;
    W sc = a.sc;
    int curq = -1;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long r0 = tile * C;
        if (a.nmod > 1) {
            const int q = (int)(r0 / a.mod_span);
            if (q != curq) {
                curq = q;
                ff = a.fm[q];
                lvlf = a.lvlfm[q];
                lvli = a.lvlim[q];
                fsf = a.fsfullm[q];
                fslo = a.fslom[q];
                fshi = a.fshim[q];
                sc = a.scm[q];
                if (K::TWS) {
                    __syncthreads();
                    stage_twiddles(twfs, lvlf, L);
                    stage_twiddles(twis, lvli, L);
                    __syncthreads();
                } else {
                    twf = lvlf;
                    twi = lvli;
                }
            }
        }
        load_rows<F, Lay, LOGL, TIn, NTH>(sa, (const TIn*)a.a, r0, a.nrows, a.a_rs, a.la, a.vec_in, false, a.in_seg_log,
                                     a.in_seg_stride);
        load_rows<F, Lay, LOGL, TIn, NTH>(sb, (const TIn*)a.b, r0, a.nrows, a.b_rs, a.lb, a.vec_in, false, a.in_seg_log,
                                     a.in_seg_stride);
        __syncthreads();
        run_tile<F, Lay, LOGL, false, NTH>(ff, sa, twf, lvlf);
        run_tile<F, Lay, LOGL, false, NTH>(ff, sb, twf, lvlf);
        {
            constexpr int R = L < 16 ? L : 16;
            constexpr int PER = L / R;
            for (int ch = threadIdx.x; ch < C * PER; ch += NTH) {
                const int c = ch / PER, b = ch % PER;
                const int base = Lay::chunk_base(c, b * R);
#pragma unroll
                for (int t = 0; t < R; t++) {
                    const int ix = base + t;          // R consecutive elements never cross a pad
                    sa[ix] = ff.mulw(ff.mul_redc(sa[ix], sb[ix]), sc);
                }
            }
        }
        __syncthreads();
        run_tile<F, Lay, LOGL, true, NTH>(ff, sa, twi, lvli);
        store_rows<F, Lay, LOGL, TOut, EPIV, NTH>(ff, sa, (TOut*)a.c, r0, a.nrows, a.c_rs, a.lc, a.vec_out, false, fsf,
                                             fslo, fshi, a.fs_h, a.row0, a.k2, sc, a.out_seg_log,
                                             a.out_seg_stride, a.rows_per);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launchers
template <class K> static mm_status set_smem(K kern, size_t bytes) {
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return MM_OK;
}
template <class K> static int grid_for(K kern, size_t smem, long long tiles, int threads = NT) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    long long cap = (long long)num_sms() * per_sm;
    return (int)(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
}
static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <class F, int LOGL, bool INV, class TIn, class TOut, int EPIV>
static mm_status launch_rows_e(const F& f, RowArgs<F> a, cudaStream_t st) {
    typedef typename F::T T;
    typedef RowsK<F, LOGL> K;
    constexpr int L = 1 << LOGL;
    constexpr int V = Vec<T>::N;
    const size_t smem = K::smem();
    a.vec_in = sizeof(TIn) == sizeof(T) && !(INV && a.perm) && a.in_rs % V == 0 && a.in_seg_stride % V == 0 &&
               (!a.in_seg_log || (1 << a.in_seg_log) >= V) && aligned16(a.in);
    a.vec_out = sizeof(TOut) == sizeof(T) && !(!INV && a.perm) && a.out_rs % V == 0 && a.out_seg_stride % V == 0 &&
                (!a.out_seg_log || (1 << a.out_seg_log) >= V) && aligned16(a.out);
    if constexpr (std::is_same<F, FpG>::value && LOGL == 13 && !INV && EPIV == EPI_CANON && sizeof(TIn) == 8 &&
                  sizeof(TOut) == 8)
        if (gold_rows_tma_ok(a)) return launch_gold_rows_tma(f, a, st);
    if constexpr (std::is_same<F, FpG>::value && LOGL == 13 && INV && EPIV == EPI_FS_FULL && sizeof(TIn) == 8 &&
                  sizeof(TOut) == 8)
        if (gold_rows_inv_tma_ok(a)) return launch_gold_rows_inv_tma(f, a, st);
    auto kern = k_rows<F, LOGL, INV, TIn, TOut, EPIV>;
    mm_status s = set_smem(kern, smem);
    if (s != MM_OK) return s;
    long long tiles = (a.nrows + K::Lay::C - 1) / K::Lay::C;
    {
        LaunchScope ls(INV ? "ntt_rows_inv" : "ntt_rows_fwd", st);
        kern<<<grid_for(kern, smem, tiles, NTr<F, LOGL>::v), NTr<F, LOGL>::v, smem, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    (void)L;
    return MM_OK;
}

template <class F, int LOGL, bool INV, class TIn, class TOut, int EPIV>
static mm_status launch_cols_e(const F& f, ColArgs<F> a, cudaStream_t st) {
    typedef typename F::T T;
    typedef ColsK<F, LOGL> K;
    constexpr int V = Vec<T>::N;
    const size_t smem = K::smem();
    if (a.ncols % K::Lay::C != 0)
        return set_err(MM_E_UNSUPPORTED_SIZE, "column block of %lld columns is not a multiple of the tile width %d",
                       a.ncols, (int)K::Lay::C);
    a.vec_in = sizeof(TIn) == sizeof(T) && a.in_rs % V == 0 && (a.in_bs % V == 0 || a.nbatch == 1) && aligned16(a.in);
    a.vec_out = sizeof(TOut) == sizeof(T) && a.out_rs % V == 0 && (a.out_bs % V == 0 || a.nbatch == 1) &&
                aligned16(a.out);
    if (a.npeers && !a.vec_out) return set_err(MM_E_ARG, "peer scatter needs 16-byte aligned rows");
    if constexpr (std::is_same<F, FpG>::value && LOGL == 11 && !INV && EPIV == EPI_FS_FULL && sizeof(TIn) == 8 &&
                  sizeof(TOut) == 8)
        if (gold_cols_tma_ok(a)) return launch_gold_cols_tma(f, a, st);
    if constexpr (std::is_same<F, FpG>::value && LOGL == 12 && !INV && EPIV == EPI_FS_FULL && sizeof(TIn) == 2 &&
                  sizeof(TOut) == 8)
        if (gold_cols16_tma_ok(a)) return launch_gold_cols16_tma(f, a, st);
    if constexpr (std::is_same<F, FpG>::value && (LOGL == 11 || LOGL == 12) && INV &&
                  (EPIV == EPI_CANON || EPIV == (EPI_SCALE | EPI_CANON)) && sizeof(TIn) == 8 && sizeof(TOut) == 8)
        if (gold_cols_inv_tma_ok(a, LOGL)) return launch_gold_cols_inv_tma(f, a, LOGL, EPIV, st);
    if constexpr ((std::is_same<F, Fp32>::value || std::is_same<F, FpD>::value) && ColsTmaK<F, LOGL>::OK &&
                  sizeof(TIn) == sizeof(T) && sizeof(TOut) == sizeof(T))
        if (cols_tma_ok<F, LOGL>(a)) return launch_cols_tma<F, LOGL, INV, EPIV>(f, a, st);
    auto kern = k_cols<F, LOGL, INV, TIn, TOut, EPIV>;
    mm_status s = set_smem(kern, smem);
    if (s != MM_OK) return s;
    long long tiles = a.ncols / K::Lay::C * a.nbatch;
    {
        LaunchScope ls(INV ? "ntt_cols_inv" : "ntt_cols_fwd", st);
        kern<<<grid_for(kern, smem, tiles, NTc<F, LOGL>::v), NTc<F, LOGL>::v, smem, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

template <class F, int LOGL, class TIn, class TOut, int EPIV>
static mm_status launch_pmul_e(const F& f, PmulArgs<F> a, cudaStream_t st) {
    typedef typename F::T T;
    typedef PmulK<F, LOGL> K;
    constexpr int V = Vec<T>::N;
    const size_t smem = K::smem();
    a.vec_in = sizeof(TIn) == sizeof(T) && a.a_rs % V == 0 && a.b_rs % V == 0 && a.in_seg_stride % V == 0 &&
               (!a.in_seg_log || (1 << a.in_seg_log) >= V) && aligned16(a.a) && aligned16(a.b);
    a.vec_out = sizeof(TOut) == sizeof(T) && a.c_rs % V == 0 && a.out_seg_stride % V == 0 &&
                (!a.out_seg_log || (1 << a.out_seg_log) >= V) && aligned16(a.c);
    if constexpr (std::is_same<F, FpG>::value && LOGL == 13 && EPIV == EPI_FS_FULL && sizeof(TIn) == 8 &&
                  sizeof(TOut) == 8)
        if (gold_pmul_rows_tma_ok(a)) return launch_gold_pmul_rows_tma(f, a, st);
    auto kern = k_rows_pmul<F, LOGL, TIn, TOut, EPIV>;
    mm_status s = set_smem(kern, smem);
    if (s != MM_OK) return s;
    long long tiles = (a.nrows + K::Lay::C - 1) / K::Lay::C;
    const int grid = grid_for(kern, smem, tiles, NTr<F, LOGL>::v);
    if (K::SB) MM_CUDA_TRY(alloc_async(&a.scratch, (size_t)grid * (1u << LOGL) * sizeof(T), st));
    {
        LaunchScope ls(a.fs ? "pmul_rows_fourstep" : "pmul_rows_single", st);
        kern<<<grid, NTr<F, LOGL>::v, smem, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    if (K::SB) MM_CUDA_TRY(cudaFreeAsync(a.scratch, st));
    return MM_OK;
}

static inline int epi_code(int fs, bool full, int scale, int canon) {
    return (fs ? (full ? EPI_FS_FULL : EPI_FS_SPLIT) : 0) | (scale ? EPI_SCALE : 0) | (canon ? EPI_CANON : 0);
}

// epilogue variants actually used by the drivers (others return an error)
template <class F, int LOGL, bool INV, class TIn, class TOut>
static mm_status launch_rows_k(const F& f, const RowArgs<F>& a, cudaStream_t st) {
    const int e = epi_code(INV ? a.fs : 0, a.fs_full != nullptr, a.scale, a.canon);
    if (!INV) {
        if (e == EPI_CANON) return launch_rows_e<F, LOGL, INV, TIn, TOut, EPI_CANON>(f, a, st);
    } else {
        if (e == (EPI_SCALE | EPI_CANON)) return launch_rows_e<F, LOGL, INV, TIn, TOut, EPI_SCALE | EPI_CANON>(f, a, st);
        if (e == EPI_FS_FULL) return launch_rows_e<F, LOGL, INV, TIn, TOut, EPI_FS_FULL>(f, a, st);
        if (e == EPI_FS_SPLIT) return launch_rows_e<F, LOGL, INV, TIn, TOut, EPI_FS_SPLIT>(f, a, st);
    }
    return set_err(MM_E_ARG, "unsupported row-pass epilogue %d", e);
}
template <class F, int LOGL, bool INV, class TIn, class TOut>
static mm_status launch_cols_k(const F& f, const ColArgs<F>& a, cudaStream_t st) {
    const int e = epi_code(INV ? 0 : a.fs, a.fs_full != nullptr, a.scale, a.canon);
    if (!INV) {
        if (e == EPI_FS_FULL) return launch_cols_e<F, LOGL, INV, TIn, TOut, EPI_FS_FULL>(f, a, st);
        if (e == EPI_FS_SPLIT) return launch_cols_e<F, LOGL, INV, TIn, TOut, EPI_FS_SPLIT>(f, a, st);
    } else {
        if (e == EPI_CANON) return launch_cols_e<F, LOGL, INV, TIn, TOut, EPI_CANON>(f, a, st);
        if (e == (EPI_SCALE | EPI_CANON)) return launch_cols_e<F, LOGL, INV, TIn, TOut, EPI_SCALE | EPI_CANON>(f, a, st);
    }
    return set_err(MM_E_ARG, "unsupported column-pass epilogue %d", e);
}
template <class F, int LOGL, class TIn, class TOut>
static mm_status launch_pmul_k(const F& f, const PmulArgs<F>& a, cudaStream_t st) {
    const int e = epi_code(a.fs, a.fs_full != nullptr, 0, a.canon);
    if (e == EPI_CANON) return launch_pmul_e<F, LOGL, TIn, TOut, EPI_CANON>(f, a, st);
    if (e == EPI_FS_FULL) return launch_pmul_e<F, LOGL, TIn, TOut, EPI_FS_FULL>(f, a, st);
    if (e == EPI_FS_SPLIT) return launch_pmul_e<F, LOGL, TIn, TOut, EPI_FS_SPLIT>(f, a, st);
    return set_err(MM_E_ARG, "unsupported product epilogue %d", e);
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
    MM_DISPATCH_K(a.k, 5, 12, MM_CALLC)
#undef MM_CALLC
}
template <class F, class TIn, class TOut>
mm_status launch_pmul(const F& f, const PmulArgs<F>& a, cudaStream_t st) {
#define MM_CALLP(K) launch_pmul_k<F, K, TIn, TOut>(f, a, st)
    MM_DISPATCH_K(a.k, 1, 13, MM_CALLP)
#undef MM_CALLP
}

}  // namespace mm
