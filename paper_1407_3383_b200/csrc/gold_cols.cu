// gold_cols.cu -- the Goldilocks forward column pass of 2^11-point columns
// (C4: 2^24 = 2^11 columns x 2^13 rows, Algorithm 1 steps 1-2)
// with its tiles staged by TMA.
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
// whole transform.  Shared memory: 64 + 64 + 65 KiB, one CTA per SM.
#include <string.h>
#include <stdlib.h>
#include "ntt_kernels.cuh"
#include "tma.cuh"

namespace mm {
namespace gcols {

constexpr int LOGL = 11, L = 1 << LOGL, C = 4;
// RowLayoutG with a column pitch of 4 mod 16 words (8-byte bank pairs): stage
// A's stores (lanes = 4 columns x 4 rows per half-warp) and the step-2 loop's
// loads (8 rows x columns {c, c + 2}) hit 16 distinct bank pairs; stages B-D
// (lanes along one column, stride 1 or 65 words) are unaffected
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
constexpr int BOXR = 256, NBOX = L / BOXR;             // box {4, 256, 8}: the whole tile
constexpr unsigned TILE_BYTES = L * C * 8;               // 64 KiB
constexpr size_t SMEM = 2 * (size_t)TILE_BYTES + (size_t)Lay::ELEMS * 8 + 16;

template <int NTH>
__global__ void __launch_bounds__(NTH, 1) k_gcols_fwd(const __grid_constant__ CUtensorMap tmx,
                                                       const __grid_constant__ CUtensorMap tmw, FpG f, ColArgs<FpG> a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* land = (uint64_t*)smem_raw;                 // [row][4] input tile (TMA)
    uint64_t* twl = land + L * C;                          // [row][4] step-2 twiddles (TMA)
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
                const int c = q & 3, b6 = (q >> 2) & 63, al = q >> 8;
                const int j0 = 64 * al + b6;
                uint64_t v[8];
#pragma unroll
                for (int t = 0; t < 4; t++) v[t] = land[(j0 + 512 * t) * C + c];
                gold::dif_a<4, gold::S_FWD>(v, al);
#pragma unroll
                for (int t = 0; t < 4; t++) s[Lay::addr(c, j0 + 512 * t)] = v[t];
            }
        } else {
            for (int e = threadIdx.x; e < L * C; e += NTH) s[Lay::addr(e & 3, e >> 2)] = land[e];
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
            const int t = e >> 1, c = (e & 1) * 2;
            const ulonglong2 w = *(const ulonglong2*)(twl + t * C + c);
            const uint64_t v0 = f.mulw(s[Lay::addr(c, t)], w.x);
            const uint64_t v1 = f.mulw(s[Lay::addr(c + 1, t)], w.y);
            *(ulonglong2*)(ob + (unsigned)t * ors + c) = make_ulonglong2(v0, v1);
        }
        __syncthreads();
        if (threadIdx.x == 0 && nxt < ntiles) {
            long long nb, ncl0;
            coords(nxt, nb, ncl0);
            tma_load_tile(twl, &tmw, (int)(a.col0 + ncl0), 0, 0, &bar[1], TILE_BYTES);
        }
    }
}

// 3-D view {cols, 256 rows, groups of 256 rows} of a row-major u64 matrix with
// row stride rs words; box {4, 256, 8} = one whole tile
static mm_status make_map(CUtensorMap* tm, const void* base, long long cols, long long rs, long long groups) {
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

static int threads_cfg() {
    static int nt = [] {
        const char* e = getenv("MMNTT_GOLD_TMA_NT");
        return e && atoi(e) == 512 ? 512 : 1024;
    }();
    return nt;
}

template <int NTH> static mm_status launch(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st) {
    CUtensorMap tmx, tmw;
    memset(&tmx, 0, sizeof(tmx));
    memset(&tmw, 0, sizeof(tmw));
    mm_status s = make_map(&tmx, a.in, a.ncols, a.in_rs, a.nbatch * NBOX);
    if (s == MM_OK) s = make_map(&tmw, a.fs_full, a.n1, a.n1, NBOX);
    if (s != MM_OK) return s;
    auto kern = k_gcols_fwd<NTH>;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    const long long tiles = a.ncols / C * a.nbatch;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    {
        LaunchScope ls("ntt_cols_fwd", st);
        kern<<<grid, NTH, SMEM, st>>>(tmx, tmw, f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

}  // namespace gcols

bool gold_cols_tma_ok(const ColArgs<FpG>& a) {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    using namespace gcols;
    return on && tma_encoder() != nullptr && a.nmod <= 1 && a.npeers == 0 && a.fs_full != nullptr &&
           a.vec_in && a.vec_out && a.ncols % C == 0 && a.in_rs % 2 == 0 && a.n1 % 2 == 0 &&
           a.in_bs == (long long)L * a.in_rs && a.in_len >= (long long)L * a.n1 && a.out_len >= (long long)L * a.n1 &&
           ((uintptr_t)a.fs_full & 15) == 0 && a.nbatch * NBOX < (1ll << 31) && a.n1 < (1ll << 31);
}

mm_status launch_gold_cols_tma(const FpG& f, const ColArgs<FpG>& a, cudaStream_t st) {
    return gcols::threads_cfg() == 512 ? gcols::launch<512>(f, a, st) : gcols::launch<1024>(f, a, st);
}

}  // namespace mm
