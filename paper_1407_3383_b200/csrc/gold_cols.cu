// gold_cols.cu -- Goldilocks column passes (Algorithm 1 steps 1-2 and their
// inverse) with their tiles staged by TMA:
//   k_gcols_fwd    2^11-point forward columns with step-2 twiddles (C4)
//   k_gcols_inv    2^11 / 2^12-point inverse columns (C4 inverse, C5)
//   k_gcols16_fwd  2^12-point forward columns of zero-padded 16-bit limbs (C5)
// The forward C4 kernel, in detail:
//
// k_cols (ntt_kernels.cuh) loads a tile of four columns with per-thread
// 16-byte loads and the step-2 twiddles at its store with per-thread table
// loads: both wait on HBM latency inside the transform (ncu r05: long
// scoreboard the top stall, issue active 51 %).  Here one thread moves each
// 64 KiB tile (4 columns x 2048 rows, 32-byte row segments) with ONE 3-D box
// copy into a landing buffer, and the tile's step-2 twiddles (the same
// [row][4 columns] box of the plan's full table) into a second one:
//
//   wait data(i) -> stage A reads the landing buffer (radix-4 DFTs over the
//   top digit, lanes = 4 columns x 8 rows: 256 contiguous bytes per warp
//   access) and writes the padded compute tile -> barrier -> TMA data(i+1)
//   -> stages B-D (gold.cuh) -> wait twiddles(i) -> step-2 product, 16-byte
//   stores -> barrier -> TMA twiddles(i+1)
//
// so the next tile streams in under stages B-D and the twiddles under the
// whole transform.  Shared memory per CTA: two landing tiles + the padded
// compute tile (64 + 64 + 65 KiB, one CTA per SM).
#include <string.h>
#include <stdlib.h>
#include "ntt_kernels.cuh"
#include "tma.cuh"

namespace mm {
namespace gcols {

constexpr int LOGL = 11, L = 1 << LOGL;
constexpr int BOXR = 256, NBOX = L / BOXR;             // box {C, 256, 8}: the whole tile
// RowLayoutG with a column pitch of 16 / C mod 16 words (8-byte bank pairs):
// stage A's stores (lanes = C columns x 16 / C rows per half-warp) and the
// step-2 loop's loads hit 16 distinct bank pairs; stages B-D (lanes along one
// column, stride 1 or 65 words) are unaffected
template <int C> struct LayC : RowLayoutG<uint64_t, LOGL, C> {
    static constexpr int SROW = [] {
        int s = L + (L >> 6);
        while ((s & 15) != 16 / C) s++;
        return s;
    }();
    static constexpr int ELEMS = C * SROW;
    __device__ __forceinline__ static int addr(int c, int j) { return c * SROW + j + (j >> 6); }
    __device__ __forceinline__ static int chunk_base(int c, int base) { return c * SROW + base + (base >> 6); }
};
// C columns per tile: 4 (32-byte row segments, 64 KiB tiles, one 1024-thread
// CTA per SM).  C = 2 (16-byte segments, two 512-thread CTAs per SM) measured
// 3.34 ms against 1.34 for C4's column pass: box copies of 16-byte rows are
// slow, so only C = 4 is launched.
template <int C> struct TileCfg {
    static constexpr unsigned TILE_BYTES = L * C * 8;
    static constexpr size_t SMEM = 2 * (size_t)TILE_BYTES + (size_t)LayC<C>::ELEMS * 8 + 16;
    static constexpr int NTH = C == 4 ? 1024 : 512;
};

template <int C>
__global__ void __launch_bounds__(TileCfg<C>::NTH, C == 4 ? 1 : 2) k_gcols_fwd(const __grid_constant__ CUtensorMap tmx,
                                                              const __grid_constant__ CUtensorMap tmw, FpG f,
                                                              ColArgs<FpG> a) {
    typedef LayC<C> Lay;
    constexpr int NTH = TileCfg<C>::NTH;
    constexpr unsigned TILE_BYTES = TileCfg<C>::TILE_BYTES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* land = (uint64_t*)smem_raw;                 // [row][C] input tile (TMA)
    uint64_t* twl = land + L * C;                          // [row][C] step-2 twiddles (TMA)
    uint64_t* s = twl + L * C;                             // padded compute tile [c][j]
    uint64_t* bar = s + Lay::ELEMS;                        // 0: data, 1: twiddles
    const uint64_t* full = (const uint64_t*)a.lvl + L;     // w_L^e, e < L
    const bool fast = __ldg(full + (L >> 6)) == gold::Pow2Val<gold::S_FWD>::v;
    const long long ntiles = a.ncols / C * a.nbatch;
    const unsigned ors = (unsigned)a.out_rs;
    // tile -> (batch row, first column): column-group-major, as k_cols
    auto coords = [&](long long tile, long long& b, long long& cl0) {
        b = tile % a.nbatch;
        cl0 = tile / a.nbatch * C;
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
        if ((long long)blockIdx.x < ntiles) {
            long long b, cl0;
            coords(blockIdx.x, b, cl0);
            tma_load_tile(land, &tmx, (int)cl0, 0, (int)(b * NBOX), &bar[0], TILE_BYTES);
            tma_load_tile(twl, &tmw, (int)(a.col0 + cl0), 0, 0, &bar[1], TILE_BYTES);
        }
    }
    __syncthreads();
    int it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        long long b, cl0;
        coords(tile, b, cl0);
        const long long nxt = tile + gridDim.x;
        mbar_wait(&bar[0], it & 1);
        if (fast) {
            // stage A (gold::dif_ln with NA = 32): radix-4 DFTs over ah of
            // j = 512 ah + 64 al + b6, then w_32^(al r); lanes: c fastest
            for (int q = threadIdx.x; q < C * 512; q += NTH) {
                const int c = q % C, b6 = (q / C) & 63, al = q / (64 * C);
                const int j0 = 64 * al + b6;
                uint64_t v[8];
#pragma unroll
                for (int t = 0; t < 4; t++) v[t] = land[(j0 + 512 * t) * C + c];
                gold::dif_a<4, gold::S_FWD>(v, al);
#pragma unroll
                for (int t = 0; t < 4; t++) s[Lay::addr(c, j0 + 512 * t)] = v[t];
            }
        } else {
            for (int e = threadIdx.x; e < L * C; e += NTH) s[Lay::addr(e % C, e / C)] = land[e];
        }
        __syncthreads();
        // the landing buffer is free: the next tile streams in under stages B-D
        if (threadIdx.x == 0 && nxt < ntiles) {
            long long nb, ncl0;
            coords(nxt, nb, ncl0);
            tma_load_tile(land, &tmx, (int)ncl0, 0, (int)(nb * NBOX), &bar[0], TILE_BYTES);
        }
        if (fast) gold::dif_ln_bcd<Lay, L, 1, NTH, gold::S_FWD>(s, full, 1, L / 64);
        else run_tile<FpG, Lay, LOGL, false, NTH>(f, s, a.lvl, a.lvl);
        // step 2: x_{t, c} w^(j1 [t]) from the twiddle tile, 16-byte stores
        mbar_wait(&bar[1], it & 1);
        uint64_t* ob = (uint64_t*)a.out + b * a.out_bs + cl0;
        for (int e = threadIdx.x; e < L * C / 2; e += NTH) {
            const int t = e / (C / 2), c = (e % (C / 2)) * 2;
            const ulonglong2 w = *(const ulonglong2*)(twl + t * C + c);
            const uint64_t v0 = f.mulw(s[Lay::addr(c, t)], w.x);
            const uint64_t v1 = f.mulw(s[Lay::addr(c + 1, t)], w.y);
            // fused transpose (sharded transform): row t goes to its owner's receive buffer
            uint64_t* dst = a.npeers ? (uint64_t*)a.peer_out[t >> a.peer_shift] + cl0 : ob;
            *(ulonglong2*)(dst + (unsigned)t * ors + c) = make_ulonglong2(v0, v1);
        }
        __syncthreads();
        if (threadIdx.x == 0 && nxt < ntiles) {
            long long nb, ncl0;
            coords(nxt, nb, ncl0);
            tma_load_tile(twl, &tmw, (int)(a.col0 + ncl0), 0, 0, &bar[1], TILE_BYTES);
        }
    }
    // peer stores ordered system-wide before the stream's next kernel raises the ready flags
    if (a.npeers) __threadfence_system();
}

// 3-D view {cols, 256 rows, groups of 256 rows} of a row-major u64 matrix with
// row stride rs words; box {C, 256, 8} = one whole tile
static mm_status make_map(CUtensorMap* tm, const void* base, long long cols, long long rs, long long groups, int C) {
    auto enc = tma_encoder();
    if (!enc) return set_err(MM_E_CUDA, "cuTensorMapEncodeTiled is not available");
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)BOXR, (cuuint64_t)groups};
    cuuint64_t strides[2] = {(cuuint64_t)rs * 8, (cuuint64_t)rs * 8 * BOXR};
    cuuint32_t box[3] = {(cuuint32_t)C, (cuuint32_t)BOXR, (cuuint32_t)NBOX};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(MM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return MM_OK;
}

template <int C> static mm_status launch(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st) {
    CUtensorMap tmx, tmw;
    memset(&tmx, 0, sizeof(tmx));
    memset(&tmw, 0, sizeof(tmw));
    mm_status s = make_map(&tmx, a.in, a.ncols, a.in_rs, a.nbatch * NBOX, C);
    if (s == MM_OK) s = make_map(&tmw, a.fs_full, a.n1, a.n1, NBOX, C);
    if (s != MM_OK) return s;
    auto kern = k_gcols_fwd<C>;
    constexpr size_t SMEM = TileCfg<C>::SMEM;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TileCfg<C>::NTH, SMEM);
    if (per_sm < 1) per_sm = 1;
    const long long tiles = a.ncols / C * a.nbatch, cap = (long long)num_sms() * per_sm;
    const int grid = (int)(tiles < cap ? tiles : cap);
    {
        LaunchScope ls("ntt_cols_fwd", st);
        kern<<<grid, TileCfg<C>::NTH, SMEM, st>>>(tmx, tmw, f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}


// ---------------------------------------------------------------- inverse columns
// Inverse column pass (the last step of an inverse transform or product,
// P:923) of 2^11- or 2^12-point columns, 4 columns per tile: the tile arrives
// by box copies into a 64 KiB landing buffer -- the whole 2^11-point tile, or
// a 2^12-point tile in two halves -- and is copied into the padded compute
// tile (lanes: c fastest, conflict-free with the 4 mod 16 pitch); the next
// tile's (first half) streams in under the whole DIT.  A 2^12-point tile's
// first half runs its half-local DIT stages while the second is in flight.
template <int LOGL> struct Inv {
    static constexpr int L = 1 << LOGL, C = 4, HALVES = LOGL == 12 ? 2 : 1, LR = L / HALVES;
    static constexpr unsigned LAND_BYTES = LR * C * 8;       // 64 KiB
    struct Lay : RowLayoutG<uint64_t, LOGL, C> {
        static constexpr int SROW = [] {
            int s = L + (L >> 6);
            while ((s & 15) != 4) s++;
            return s;
        }();
        static constexpr int ELEMS = C * SROW;
        __device__ __forceinline__ static int addr(int c, int j) { return c * SROW + j + (j >> 6); }
        __device__ __forceinline__ static int chunk_base(int c, int base) { return c * SROW + base + (base >> 6); }
    };
    static constexpr size_t SMEM = LAND_BYTES + (size_t)Lay::ELEMS * 8 + 16;
};

template <int LOGL, int EPIV>
__global__ void __launch_bounds__(1024, 1) k_gcols_inv(const __grid_constant__ CUtensorMap tmx, FpG f,
                                                       ColArgs<FpG> a) {
    typedef Inv<LOGL> K;
    typedef typename K::Lay Lay;
    typedef Epi<FpG, EPIV> E;
    constexpr int NTH = 1024, C = K::C, L = K::L, LR = K::LR, HALVES = K::HALVES, GPH = LR / BOXR;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* land = (uint64_t*)smem_raw;
    uint64_t* s = land + LR * C;
    uint64_t* bar = s + Lay::ELEMS;
    const uint64_t* full = (const uint64_t*)a.lvl + L;     // inverse powers w_L^-e, e < L
    const bool fast = __ldg(full + (L >> 6)) == gold::Pow2Val<gold::S_INV>::v;
    const long long ntiles = a.ncols / C * a.nbatch;
    const unsigned ors = (unsigned)a.out_rs;
    auto coords = [&](long long tile, long long& b, long long& cl0) {
        b = tile % a.nbatch;
        cl0 = tile / a.nbatch * C;
    };
    auto issue = [&](long long tile, int h) {
        long long b, cl0;
        coords(tile, b, cl0);
        tma_load_tile(land, &tmx, (int)cl0, 0, (int)(b * (L / BOXR) + h * GPH), &bar[0], K::LAND_BYTES);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_fence_init();
        if ((long long)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    }
    __syncthreads();
    unsigned ph = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        long long b, cl0;
        coords(tile, b, cl0);
        const long long nxt = tile + gridDim.x;
        for (int h = 0; h < HALVES; h++) {
            mbar_wait(&bar[0], ph & 1);
            ph++;
            for (int e = threadIdx.x; e < LR * C; e += NTH) s[Lay::addr(e % C, h * LR + e / C)] = land[e];
            __syncthreads();
            if (threadIdx.x == 0) {
                if (h + 1 < HALVES) issue(tile, h + 1);
                else if (nxt < ntiles) issue(nxt, 0);
            }
            // 2^12 points: the stages that stay inside one half run while the
            // other half is in flight
            if constexpr (HALVES == 2)
                if (fast) gold::dit4096_half<Lay, NTH, gold::S_INV>(s, full, h);
        }
        if (HALVES == 2 && fast) gold::dit4096_a<Lay, NTH, gold::S_INV>(s);
        else run_tile<FpG, Lay, LOGL, true, NTH>(f, s, a.lvl, a.lvl);
        // canonical (and n^-1 for a standalone inverse), truncated to out_len
        const long long lin0 = a.col0 + cl0;
        uint64_t* ob = (uint64_t*)a.out + b * a.out_bs + cl0;
        for (int e = threadIdx.x; e < L * C / 2; e += NTH) {
            const int t = e >> 1, c = (e & 1) * 2;
            const long long lin = (long long)t * a.n1 + lin0 + c;
            if (lin >= a.out_len) continue;
            const uint64_t v0 = E::apply(f, s[Lay::addr(c, t)], 0, nullptr, nullptr, 0, 0u, a.sc);
            const uint64_t v1 = E::apply(f, s[Lay::addr(c + 1, t)], 0, nullptr, nullptr, 0, 0u, a.sc);
            if (lin + 1 < a.out_len) *(ulonglong2*)(ob + (unsigned)t * ors + c) = make_ulonglong2(v0, v1);
            else ob[(unsigned)t * ors + c] = v0;
        }
        __syncthreads();
    }
}

template <int LOGL, int EPIV> static mm_status launch_inv(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st) {
    typedef Inv<LOGL> K;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    mm_status s = make_map(&tm, a.in, a.ncols, a.in_rs, a.nbatch * (K::L / BOXR), K::C);
    if (s != MM_OK) return s;
    auto kern = k_gcols_inv<LOGL, EPIV>;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM));
    const long long tiles = a.ncols / K::C * a.nbatch;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    {
        LaunchScope ls("ntt_cols_inv", st);
        kern<<<grid, 1024, K::SMEM, st>>>(tm, f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

// ---------------------------------------------------------------- 16-bit limbs (C5)
// The forward column pass of a zero-padded 16-bit limb vector (C5: 2^25 =
// 2^12 columns x 2^13 rows, limbs in rows t < R <= 2^11).  A tile holds four
// 2^12-point columns (130 KiB, one 1024-thread CTA per SM; its 32-byte output
// row segments are whole sectors -- two-column tiles processed one after the
// other by the same CTA wrote half sectors twice as many bytes to DRAM),
// whose rows are 8 bytes of limbs: one TMA box {8 columns, 256 rows} per 256
// rows lands the limbs of TWO tiles at once ([R][8] x 2 B = 32 KiB), the CTA
// transforms them one after the other and the next super-tile's limbs stream
// in under the last tile's stages B-D.  The step-2 twiddle is formed on chip
// from per-column bases T_lo, T_hi (k_cols' OTF path, C5: faster than the
// table loads); T_hi is stored at bit-reversed positions so that the store
// loop's lanes read consecutive words.
namespace g16 {
constexpr int LOGL = 12, L = 1 << LOGL, C = 4, SUPER = 8, NSUB = SUPER / C, RMAX = L / 2;
constexpr int LO = LOGL / 2, NLO = 1 << LO, NHI = 1 << (LOGL - LO), NOTF = NLO + NHI;
constexpr int NTH = 1024, BOXR = 256;
struct Lay : RowLayoutG<uint64_t, LOGL, C> {
    static constexpr int SROW = [] {
        int s = L + (L >> 6);
        while ((s & 15) != 16 / C) s++;     // stage A's stores: 4 columns x 4 rows per half-warp
        return s;
    }();
    static constexpr int ELEMS = C * SROW;
    __device__ __forceinline__ static int addr(int c, int j) { return c * SROW + j + (j >> 6); }
    __device__ __forceinline__ static int chunk_base(int c, int base) { return c * SROW + base + (base >> 6); }
};
constexpr unsigned LAND_BYTES = RMAX * SUPER * 2;                 // 32 KiB
constexpr size_t SMEM = LAND_BYTES + (size_t)Lay::ELEMS * 8 + (size_t)C * NOTF * 8 + 16;

__global__ void __launch_bounds__(NTH, 1) k_gcols16_fwd(const __grid_constant__ CUtensorMap tmx, FpG f,
                                                       ColArgs<FpG> a, int nrows) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint16_t* land = (uint16_t*)smem_raw;                 // [row][8] limbs (TMA)
    uint64_t* s = (uint64_t*)(smem_raw + LAND_BYTES);      // padded compute tile [c][j]
    uint64_t* otf = s + Lay::ELEMS;                        // [c][T_lo | T_hi]
    uint64_t* bar = otf + C * NOTF;
    const uint64_t* full = (const uint64_t*)a.lvl + L;
    const bool fast = __ldg(full + (L >> 6)) == gold::Pow2Val<gold::S_FWD>::v;
    const uint64_t* fsf = a.fs_full;
    const long long nsuper = a.ncols / SUPER;
    const unsigned ors = (unsigned)a.out_rs, n1 = (unsigned)a.n1;
    const int nbox = (nrows + BOXR - 1) / BOXR;
    const unsigned bytes = (unsigned)nbox * BOXR * SUPER * 2;
    auto issue = [&](long long st) {
        mbar_arrive_tx(&bar[0], bytes);
        for (int i = 0; i < nbox; i++)
            tma_load_box2(land + i * BOXR * SUPER, &tmx, (int)(st * SUPER), i * BOXR, &bar[0]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_fence_init();
        if ((long long)blockIdx.x < nsuper) issue(blockIdx.x);
    }
    __syncthreads();
    int it = 0;
    for (long long st = blockIdx.x; st < nsuper; st += gridDim.x, it++) {
        mbar_wait(&bar[0], it & 1);
        for (int sub = 0; sub < NSUB; sub++) {
            const long long cl0 = st * SUPER + sub * C;
            const long long lin0 = a.col0 + cl0;
            // this tile's step-2 bases (in flight with stage A)
            uint64_t otf_v = 0;
            int otf_slot = 0;
            if (threadIdx.x < C * NOTF) {
                const int c = threadIdx.x / NOTF, r = threadIdx.x % NOTF;
                const int row = r < NLO ? r : (r - NLO) << LO;
                otf_v = __ldg(fsf + (unsigned)brev(row, LOGL) * n1 + (unsigned)lin0 + c);
                otf_slot = c * NOTF + (r < NLO ? r : NLO + brev(r - NLO, LOGL - LO));
            }
            if (fast) {
                // stage A (NA = 64): 8-point DFTs over ah of j = 512 ah + 64 al + b6,
                // rows >= nrows zero; lanes: c fastest
                for (int q = threadIdx.x; q < C * 512; q += NTH) {
                    const int c = q % C, b6 = (q / C) & 63, al = q / (64 * C);
                    const int j0 = 64 * al + b6;
                    static_assert(RMAX / 512 == 4, "rows >= 2048 (t >= 4) are zero padding");
                    uint64_t v[8];
#pragma unroll
                    for (int t = 0; t < 8; t++) {
                        const int row = j0 + 512 * t;
                        v[t] = (t < 4 && row < nrows) ? land[row * SUPER + sub * C + c] : 0ull;
                    }
                    gold::dif8_zh<gold::S_FWD>(v);      // the zero upper half skips the span-4 level
                    gold::rot<gold::S_FWD, 1, 8>(v, al);
#pragma unroll
                    for (int t = 0; t < 8; t++) s[Lay::addr(c, j0 + 512 * t)] = v[t];
                }
            } else {
                for (int e = threadIdx.x; e < L * C; e += NTH) {
                    const int row = e / C, c = e % C;
                    s[Lay::addr(c, row)] = row < nrows ? land[row * SUPER + sub * C + c] : 0ull;
                }
            }
            if (threadIdx.x < C * NOTF) otf[otf_slot] = otf_v;
            __syncthreads();
            // the last tile of the super-tile has read its limbs: the next super-tile streams in
            if (sub == NSUB - 1 && threadIdx.x == 0 && st + gridDim.x < nsuper) issue(st + gridDim.x);
            if (fast) gold::dif_ln_bcd<Lay, L, 1, NTH, gold::S_FWD>(s, full, 1, L / 64);
            else run_tile<FpG, Lay, LOGL, false, NTH>(f, s, a.lvl, a.lvl);
            uint64_t* ob = (uint64_t*)a.out + cl0;
            // w^(j1 k), k = [t]: T_lo[k mod 2^LO] (warp-uniform) T_hi[k >> LO]
            // (stored at [t mod 2^LO]); lanes: 2 per row, 32-byte row segments
            for (int e = threadIdx.x; e < L * C / 2; e += NTH) {
                const int t = e / (C / 2), c = (e % (C / 2)) * 2;
                const unsigned lo = (unsigned)brev(t, LOGL) & (NLO - 1), hi = (unsigned)t & (NHI - 1);
                const uint64_t w0 = FpG::mul(otf[c * NOTF + lo], otf[c * NOTF + NLO + hi]);
                const uint64_t w1 = FpG::mul(otf[(c + 1) * NOTF + lo], otf[(c + 1) * NOTF + NLO + hi]);
                const uint64_t v0 = f.mulw(s[Lay::addr(c, t)], w0);
                const uint64_t v1 = f.mulw(s[Lay::addr(c + 1, t)], w1);
                *(ulonglong2*)(ob + (unsigned)t * ors + c) = make_ulonglong2(v0, v1);
            }
            __syncthreads();
        }
    }
}
}  // namespace g16
}  // namespace gcols

bool gold_tma_enabled() {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    return on && tma_encoder() != nullptr;
}

bool gold_cols_tma_ok(const ColArgs<FpG>& a) {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    using namespace gcols;
    return on && tma_encoder() != nullptr && a.nmod <= 1 && a.fs_full != nullptr &&
           a.vec_in && a.vec_out && a.ncols % 4 == 0 && a.in_rs % 2 == 0 && a.n1 % 2 == 0 &&
           (a.nbatch == 1 || a.in_bs == (long long)L * a.in_rs) && a.in_len >= (long long)L * a.n1 &&
           a.out_len >= (long long)L * a.n1 &&
           ((uintptr_t)a.fs_full & 15) == 0 && a.nbatch * NBOX < (1ll << 31) && a.n1 < (1ll << 31);
}

bool gold_cols16_tma_ok(const ColArgs<FpG>& a) {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    using namespace gcols::g16;
    // limbs in whole rows t < in_len / n1 <= 2^11 (every column of the block
    // valid exactly up to that row), one batch row, 16-byte aligned rows
    return on && tma_encoder() != nullptr && a.nbatch == 1 && a.nmod <= 1 && a.npeers == 0 && a.fs_full != nullptr &&
           a.vec_out && a.ncols % SUPER == 0 && a.in_rs == a.n1 && a.n1 % 8 == 0 && a.in_len % a.n1 == 0 &&
           a.in_len / a.n1 <= RMAX && a.in_len > 0 && a.out_len >= (long long)L * a.n1 && ((uintptr_t)a.in & 15) == 0 &&
           a.n1 < (1ll << 31);
}

mm_status launch_gold_cols16_tma(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st) {
    using namespace gcols::g16;
    auto enc = tma_encoder();
    if (!enc) return set_err(MM_E_CUDA, "cuTensorMapEncodeTiled is not available");
    const int nrows = (int)(a.in_len / a.n1);
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    cuuint64_t dims[2] = {(cuuint64_t)a.ncols, (cuuint64_t)nrows};
    cuuint64_t strides[1] = {(cuuint64_t)a.in_rs * 2};
    cuuint32_t box[2] = {(cuuint32_t)SUPER, (cuuint32_t)BOXR};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(a.in), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(MM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    auto kern = k_gcols16_fwd;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTH, SMEM);
    if (per_sm < 1) per_sm = 1;
    const long long tiles = a.ncols / SUPER, cap = (long long)num_sms() * per_sm;
    const int grid = (int)(tiles < cap ? tiles : cap);
    {
        LaunchScope ls("ntt_cols_fwd", st);
        kern<<<grid, NTH, SMEM, st>>>(tm, f, a, nrows);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

bool gold_cols_inv_tma_ok(const ColArgs<FpG>& a, int logl) {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    const long long L = 1ll << logl;
    return on && (logl == 11 || logl == 12) && tma_encoder() != nullptr && a.nmod <= 1 && a.npeers == 0 &&
           a.vec_in && a.vec_out && a.ncols % 4 == 0 && a.in_rs % 2 == 0 && (a.nbatch == 1 || a.in_bs == L * a.in_rs) &&
           a.in_len >= L * a.n1 && a.nbatch * (L / 256) < (1ll << 31) && a.n1 < (1ll << 31);
}

mm_status launch_gold_cols_inv_tma(const FpG& f, const ColArgs<FpG>& a, int logl, int epiv, cudaStream_t st) {
    using namespace gcols;
    if (logl == 11 && epiv == EPI_CANON) return launch_inv<11, EPI_CANON>(f, a, st);
    if (logl == 11 && epiv == (EPI_SCALE | EPI_CANON)) return launch_inv<11, EPI_SCALE | EPI_CANON>(f, a, st);
    if (logl == 12 && epiv == EPI_CANON) return launch_inv<12, EPI_CANON>(f, a, st);
    if (logl == 12 && epiv == (EPI_SCALE | EPI_CANON)) return launch_inv<12, EPI_SCALE | EPI_CANON>(f, a, st);
    return set_err(MM_E_ARG, "no TMA inverse column kernel for 2^%d points, epilogue %d", logl, epiv);
}

mm_status launch_gold_cols_tma(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st) {
    return gcols::launch<4>(f, a, st);
}

}  // namespace mm
