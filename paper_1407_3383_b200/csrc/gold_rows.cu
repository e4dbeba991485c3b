// gold_rows.cu -- the Goldilocks 2^13-point row passes with their rows
// staged by bulk copies: the forward row pass (C4: Algorithm 1 steps 3-4,
// P:895-913), the inverse row pass and the fused product rows (C5).
//
// k_rows (ntt_kernels.cuh) loads a row with per-thread 16-byte loads into
// the padded tile and then runs the radix-2 level of span 4096 as a separate
// shared-memory pass.  Here one thread moves each 64 KiB row with ONE bulk
// copy (cp.async.bulk, mbarrier completion) into a landing buffer, the
// radix-2 level reads the landing buffer and writes the padded tile (that
// pass's shared-memory round trip is gone), and the next row streams in under
// the two 4096-point halves (gold.cuh) and the store.  Shared memory 64 + 65
// KiB: one 1024-thread CTA per SM.
#include <stdlib.h>
#include "ntt_kernels.cuh"
#include "tma.cuh"

namespace mm {
namespace grows {

constexpr int LOGL = 13, L = 1 << LOGL, H = L / 2, NTH = 1024;
typedef RowLayoutG<uint64_t, LOGL, 1> Lay;
constexpr unsigned ROW_BYTES = L * 8;
constexpr size_t SMEM = ROW_BYTES + (size_t)Lay::ELEMS * 8 + 16;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// row r of a (possibly segmented) row array into the landing buffer: element
// j at base + r rs + seg_j(j) -- one copy per 2^seglog-element segment (the
// sharded transform's rows are G segments in G receive buffers)
__device__ __forceinline__ void load_row(uint64_t* land, const uint64_t* base, long long r, long long rs, int seglog,
                                         long long segstride, uint64_t* bar) {
    if (!seglog) {
        bulk_load(land, base + r * rs, ROW_BYTES, bar);
        return;
    }
    mbar_arrive_tx(bar, ROW_BYTES);
    const int seg = 1 << seglog;
    for (int i = 0; i < L / seg; i++) bulk_copy(land + i * seg, base + i * segstride + r * rs, (unsigned)seg * 8, bar);
}

__global__ void __launch_bounds__(NTH, 1) k_grows_fwd(FpG f, RowArgs<FpG> a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* land = (uint64_t*)smem_raw;
    uint64_t* s = land + L;
    uint64_t* bar = s + Lay::ELEMS;
    const uint64_t* full = (const uint64_t*)a.lvl + L;    // w_L^e, e < L
    const bool fast = __ldg(full + (L >> 6)) == gold::Pow2Val<gold::S_FWD>::v;
    const uint64_t* in = (const uint64_t*)a.in;
    uint64_t* out = (uint64_t*)a.out;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_fence_init();
        if ((long long)blockIdx.x < a.nrows)
            load_row(land, in, blockIdx.x, a.in_rs, a.in_seg_log, a.in_seg_stride, &bar[0]);
    }
    __syncthreads();
    int it = 0;
    for (long long r = blockIdx.x; r < a.nrows; r += gridDim.x, it++) {
        mbar_wait(&bar[0], it & 1);
        if (fast) {
            // radix-2 level of span 4096 (twiddle w_8192^j) from the landing buffer
            for (int j = threadIdx.x; j < H; j += NTH) {
                const uint64_t x = land[j], y = land[j + H];
                s[Lay::addr(0, j)] = FpG::add(x, y);
                s[Lay::addr(0, j + H)] = FpG::mul(FpG::sub(x, y), __ldg(full + j));
            }
        } else {
            for (int j = threadIdx.x; j < L; j += NTH) s[Lay::addr(0, j)] = land[j];
        }
        __syncthreads();
        const long long nxt = r + gridDim.x;
        if (threadIdx.x == 0 && nxt < a.nrows) load_row(land, in, nxt, a.in_rs, a.in_seg_log, a.in_seg_stride, &bar[0]);
        if (fast) gold::dif_ln<Lay, 4096, 2, NTH, gold::S_FWD>(s, full, 2, L / 64);
        else run_tile<FpG, Lay, LOGL, false, NTH>(f, s, a.lvl, a.lvl);
        // canonical output, 16-byte stores (TFT order within the row)
        uint64_t* ob = out + r * a.out_rs;
        for (int e = threadIdx.x; e < L / 2; e += NTH) {
            const int j = 2 * e;
            *(ulonglong2*)(ob + j) = make_ulonglong2(f.canon(s[Lay::addr(0, j)]), f.canon(s[Lay::addr(0, j + 1)]));
        }
        __syncthreads();
    }
}


// ---------------------------------------------------------------- fused product rows (C5)
// Steps 3-4 of both operands, the entry-wise product with n^-1 and
// the inverse row transform with the inverse step-2 twiddle, per row of
// 2^13 points.  k_rows_pmul keeps one row in shared memory (two CTAs per SM)
// and parks the first spectrum in an L2 scratch row; here one 1024-thread CTA
// per SM holds both spectra (2 x 65 KiB) beside a 64 KiB landing buffer that
// the operand rows stream through by bulk copies: a_r, then b_r while a_r is
// transformed, then a_{r+1} while b_r is transformed and the product row is
// formed and transformed back.
constexpr size_t PSMEM = ROW_BYTES + 2 * (size_t)Lay::ELEMS * 8 + 16;

__global__ void __launch_bounds__(NTH, 1) k_gpmul_rows(FpG f, PmulArgs<FpG> a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* land = (uint64_t*)smem_raw;
    uint64_t* sa = land + L;
    uint64_t* sb = sa + Lay::ELEMS;
    uint64_t* bar = sb + Lay::ELEMS;
    const uint64_t* fullf = (const uint64_t*)a.lvl_f + L;
    const bool fast = __ldg(fullf + (L >> 6)) == gold::Pow2Val<gold::S_FWD>::v;
    const uint64_t* fulli = (const uint64_t*)a.lvl_i + L;
    const bool fasti = __ldg(fulli + (L >> 6)) == gold::Pow2Val<gold::S_INV>::v;
    const uint64_t* A = (const uint64_t*)a.a;
    const uint64_t* B = (const uint64_t*)a.b;
    uint64_t* Cc = (uint64_t*)a.c;
    const unsigned i2mask = (1u << a.k2) - 1;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_fence_init();
        if ((long long)blockIdx.x < a.nrows)
            load_row(land, A, blockIdx.x, a.a_rs, a.in_seg_log, a.in_seg_stride, &bar[0]);
    }
    __syncthreads();
    unsigned ph = 0;
    for (long long r = blockIdx.x; r < a.nrows; r += gridDim.x) {
        const long long nxt = r + gridDim.x;
#pragma unroll 1
        for (int op = 0; op < 2; op++) {
            uint64_t* s = op ? sb : sa;
            mbar_wait(&bar[0], ph & 1);
            ph++;
            if (fast) {
                for (int j = threadIdx.x; j < H; j += NTH) {
                    const uint64_t x = land[j], y = land[j + H];
                    s[Lay::addr(0, j)] = FpG::add(x, y);
                    s[Lay::addr(0, j + H)] = FpG::mul(FpG::sub(x, y), __ldg(fullf + j));
                }
            } else {
                for (int j = threadIdx.x; j < L; j += NTH) s[Lay::addr(0, j)] = land[j];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                if (op == 0) load_row(land, B, r, a.b_rs, a.in_seg_log, a.in_seg_stride, &bar[0]);
                else if (nxt < a.nrows) load_row(land, A, nxt, a.a_rs, a.in_seg_log, a.in_seg_stride, &bar[0]);
            }
            if (fast) gold::dif_ln<Lay, 4096, 2, NTH, gold::S_FWD>(s, fullf, 2, L / 64);
            else run_tile<FpG, Lay, LOGL, false, NTH>(f, s, a.lvl_f, a.lvl_f);
        }
        // entry-wise product with n^-1 (same positions in both bit-reversed spectra)
        for (int j = threadIdx.x; j < L; j += NTH) {
            const int ix = Lay::addr(0, j);
            sa[ix] = f.mulw(f.mul_redc(sa[ix], sb[ix]), a.sc);
        }
        __syncthreads();
        // inverse row transform and the inverse step-2 twiddle w^-(j1 [i2]) (the
        // plan's full table row); on the gold path the last DIT level (span
        // 4096, twiddle w_8192^-j) runs in the store loop
        const uint64_t* tw = a.fs_full + (size_t)((unsigned)(a.row0 + r) & i2mask) * L;
        uint64_t* ob = Cc + r * a.c_rs;        // element j at ob + seg_j(j): plain or segmented rows
        const int osl = a.out_seg_log;
        const long long oss = a.out_seg_stride;
        if (fast && fasti) {
            gold::dit_ln<Lay, 4096, 2, NTH, gold::S_INV>(sa, fulli, 2, L / 64);
            for (int j = threadIdx.x; j < H; j += NTH) {
                const uint64_t x = sa[Lay::addr(0, j)], t = FpG::mul(sa[Lay::addr(0, j + H)], __ldg(fulli + j));
                ob[seg_j(j, osl, oss)] = f.mulw(FpG::add(x, t), __ldg(tw + j));
                ob[seg_j(j + H, osl, oss)] = f.mulw(FpG::sub(x, t), __ldg(tw + j + H));
            }
        } else {
            run_tile<FpG, Lay, LOGL, true, NTH>(f, sa, a.lvl_i, a.lvl_i);
            for (int e = threadIdx.x; e < L / 2; e += NTH) {
                const int j = 2 * e;           // j, j + 1 in one segment (segments >= 2 elements)
                const ulonglong2 w = __ldg((const ulonglong2*)(tw + j));
                *(ulonglong2*)(ob + seg_j(j, osl, oss)) =
                    make_ulonglong2(f.mulw(sa[Lay::addr(0, j)], w.x), f.mulw(sa[Lay::addr(0, j + 1)], w.y));
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- inverse rows (C4 inverse)
// Inverse row transform (DIT) of 2^13-point rows with the inverse step-2
// twiddle: the row and its twiddle row (the plan's full table) arrive by bulk
// copies a row ahead; the row is copied into the padded tile (the DIT's first
// stage reads 8 consecutive words per thread), the last DIT level runs in the
// store loop.  64 + 64 + 65 KiB: one 1024-thread CTA per SM.
constexpr size_t ISMEM = 2 * (size_t)ROW_BYTES + (size_t)Lay::ELEMS * 8 + 16;

__global__ void __launch_bounds__(NTH, 1) k_grows_inv(FpG f, RowArgs<FpG> a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* land = (uint64_t*)smem_raw;
    uint64_t* twl = land + L;
    uint64_t* s = twl + L;
    uint64_t* bar = s + Lay::ELEMS;
    const uint64_t* fulli = (const uint64_t*)a.lvl + L;
    const bool fast = __ldg(fulli + (L >> 6)) == gold::Pow2Val<gold::S_INV>::v;
    const uint64_t* in = (const uint64_t*)a.in;
    uint64_t* out = (uint64_t*)a.out;
    const unsigned i2mask = (1u << a.k2) - 1;
    auto twrow = [&](long long r) { return a.fs_full + (size_t)((unsigned)(a.row0 + r) & i2mask) * L; };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
        if ((long long)blockIdx.x < a.nrows) {
            bulk_load(land, in + blockIdx.x * a.in_rs, ROW_BYTES, &bar[0]);
            bulk_load(twl, twrow(blockIdx.x), ROW_BYTES, &bar[1]);
        }
    }
    __syncthreads();
    int it = 0;
    for (long long r = blockIdx.x; r < a.nrows; r += gridDim.x, it++) {
        const long long nxt = r + gridDim.x;
        mbar_wait(&bar[0], it & 1);
        for (int j = threadIdx.x; j < L; j += NTH) s[Lay::addr(0, j)] = land[j];
        __syncthreads();
        if (threadIdx.x == 0 && nxt < a.nrows) bulk_load(land, in + nxt * a.in_rs, ROW_BYTES, &bar[0]);
        uint64_t* ob = out + r * a.out_rs;     // element j at ob + seg_j(j): plain or segmented rows
        const int osl = a.out_seg_log;
        const long long oss = a.out_seg_stride;
        if (fast) {
            gold::dit_ln<Lay, 4096, 2, NTH, gold::S_INV>(s, fulli, 2, L / 64);
            mbar_wait(&bar[1], it & 1);
            for (int j = threadIdx.x; j < H; j += NTH) {
                const uint64_t x = s[Lay::addr(0, j)], t = FpG::mul(s[Lay::addr(0, j + H)], __ldg(fulli + j));
                ob[seg_j(j, osl, oss)] = f.mulw(FpG::add(x, t), twl[j]);
                ob[seg_j(j + H, osl, oss)] = f.mulw(FpG::sub(x, t), twl[j + H]);
            }
        } else {
            run_tile<FpG, Lay, LOGL, true, NTH>(f, s, a.lvl, a.lvl);
            mbar_wait(&bar[1], it & 1);
            for (int j = threadIdx.x; j < L; j += NTH) ob[seg_j(j, osl, oss)] = f.mulw(s[Lay::addr(0, j)], twl[j]);
        }
        __syncthreads();
        if (threadIdx.x == 0 && nxt < a.nrows) bulk_load(twl, twrow(nxt), ROW_BYTES, &bar[1]);
    }
}
}  // namespace grows

bool gold_rows_tma_ok(const RowArgs<FpG>& a) {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    using namespace grows;
    return on && !a.perm && a.vec_in && a.vec_out && (a.in_seg_log == 0 || a.in_seg_log >= 8) && a.out_seg_log == 0 &&
           a.in_len == L && a.out_len == L && a.in_rs % 2 == 0 && a.rows_per == 0;
}

bool gold_pmul_rows_tma_ok(const PmulArgs<FpG>& a) {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    using namespace grows;
    return on && a.nmod <= 1 && a.fs == 1 && a.fs_full != nullptr && a.vec_in && a.vec_out &&
           (a.in_seg_log == 0 || a.in_seg_log >= 8) && a.la == L && a.lb == L && a.lc == L && a.a_rs % 2 == 0 && a.b_rs % 2 == 0 &&
           a.rows_per == 0 && ((uintptr_t)a.fs_full & 15) == 0;
}

mm_status launch_gold_pmul_rows_tma(const FpG& f, const PmulArgs<FpG>& a, cudaStream_t st) {
    using namespace grows;
    auto kern = k_gpmul_rows;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PSMEM));
    const int grid = (int)(a.nrows < num_sms() ? a.nrows : num_sms());
    {
        LaunchScope ls("pmul_rows_fourstep", st);
        kern<<<grid, NTH, PSMEM, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

bool gold_rows_inv_tma_ok(const RowArgs<FpG>& a) {
    static const bool on = [] {
        const char* e = getenv("MMNTT_GOLD_TMA");
        return !(e && e[0] == '0');
    }();
    using namespace grows;
    return on && !a.perm && a.fs == 1 && a.fs_full != nullptr && a.vec_in && a.vec_out && a.in_seg_log == 0 &&
           a.in_len == L && a.out_len == L && a.in_rs % 2 == 0 &&
           a.rows_per == 0 && ((uintptr_t)a.fs_full & 15) == 0;
}

mm_status launch_gold_rows_inv_tma(const FpG& f, const RowArgs<FpG>& a, cudaStream_t st) {
    using namespace grows;
    auto kern = k_grows_inv;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ISMEM));
    const int grid = (int)(a.nrows < num_sms() ? a.nrows : num_sms());
    {
        LaunchScope ls("ntt_rows_inv", st);
        kern<<<grid, NTH, ISMEM, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

mm_status launch_gold_rows_tma(const FpG& f, const RowArgs<FpG>& a, cudaStream_t st) {
    using namespace grows;
    auto kern = k_grows_fwd;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    const int grid = (int)(a.nrows < num_sms() ? a.nrows : num_sms());
    {
        LaunchScope ls("ntt_rows_fwd", st);
        kern<<<grid, NTH, SMEM, st>>>(f, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

}  // namespace mm
