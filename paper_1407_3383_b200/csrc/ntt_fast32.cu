// ntt_fast32.cu -- the 2^16-point four-step (n1 = n2 = 256) for p < 2^30,
// specialised for BASELINE C3 (see fast32.h for the pass structure).
//
// Every pass is two radix-16 register groups around one shared-memory
// exchange.  A "table" group (spans 128..16 of a 256-point transform) works
// on the 16 elements lo + 16 t of one transform, so its 15 twiddles
// tw[m + lo + 16 k] depend on lo only; a "constant" group (spans 8..1) works
// on 16 consecutive elements, so its 15 twiddles are the level-table entries
// 1..15, passed by value as kernel parameters (constant bank operands, no
// loads).  Global loads / stores go straight between registers and HBM in
// the table group's layout (a warp touches whole 128-byte lines).
//
// Butterflies (Harvey's lazy forms, values in [0, 2p) / [0, 4p), p < 2^30):
//   DIF (Gentleman-Sande): (x, y) -> (x + y, (x - y) w)
//   DIT (Cooley-Tukey)   : (x, y) -> (x + y w, x - y w)
// with the fixed-multiplicand product of Function 8:
// c = hi(d psi), d w - c p in [0, 2p).  The DIF sum is written as
// min(x + y, x + y - 2p) with the second term opaque to ptxas, so it becomes
// IADD3 + VIADDMNMX on the ALU pipe and the butterfly is 3 ALU + 3 FMA-pipe
// instructions (the plain form puts the sum on the FMA pipe as IMAD.IADD).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <string.h>
#include <stdlib.h>
#include "common.h"
#include "arith.cuh"
#include "fast32.h"
#include "tma.cuh"

namespace mm {
namespace f32 {

constexpr int NT = 256;

__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t add_sub(uint32_t x, uint32_t y, uint32_t c) {
    uint32_t t;
    asm("{ .reg .u32 r; add.u32 r, %1, %2; sub.u32 %0, r, %3; }" : "=r"(t) : "r"(x), "r"(y), "r"(c));
    return t;
}
__device__ __forceinline__ uint32_t sub_add(uint32_t x, uint32_t y, uint32_t c) {   // x - y + c = (x + c) - y
    return add_sub(x, c, y);
}
// Function 8 (lazy): x w mod p in [0, 2p) for any x < 2^32
__device__ __forceinline__ uint32_t mulw(uint32_t x, uint2 w, const Fld& f) {
    uint32_t c = __umulhi(x, w.y);
    return x * w.x - c * f.p;
}
__device__ __forceinline__ void dif(uint32_t& x, uint32_t& y, uint2 w, const Fld& f) {
    uint32_t t = add_sub(x, y, f.p2);
    uint32_t d = sub_add(x, y, f.p2);
    x = umin(x + y, t);
    y = mulw(d, w, f);
}
__device__ __forceinline__ void dif1(uint32_t& x, uint32_t& y, const Fld& f) {
    uint32_t t = add_sub(x, y, f.p2);
    uint32_t d = sub_add(x, y, f.p2);
    x = umin(x + y, t);
    y = umin(d, d - f.p2);
}
// DIT with the sum reduced: x' = min(xx + t, xx + t - 2p) in [0, 2p) (IADD3 +
// VIADDMNMX on the ALU pipe, so ptxas cannot move the add to the FMA pipe as
// IMAD.IADD), y' = xx - t + 2p in (0, 4p).  XR: x is already in [0, 2p).
template <bool XR>
__device__ __forceinline__ void dit(uint32_t& x, uint32_t& y, uint2 w, const Fld& f) {
    const uint32_t xx = XR ? x : umin(x, x - f.p2);
    const uint32_t t = mulw(y, w, f);
    const uint32_t s = add_sub(xx, t, f.p2);
    x = umin(xx + t, s);
    y = sub_add(xx, t, f.p2);
}
template <bool XR>
__device__ __forceinline__ void dit1(uint32_t& x, uint32_t& y, const Fld& f) {
    const uint32_t xx = XR ? x : umin(x, x - f.p2);
    const uint32_t yy = umin(y, y - f.p2);
    const uint32_t s = add_sub(xx, yy, f.p2);
    x = umin(xx + yy, s);
    y = sub_add(xx, yy, f.p2);
}
// Montgomery REDC (Function 13), subtractive form, lazy:
// x y 2^-32 mod p in (0, 2p) for x y < 2^32 p.
__device__ __forceinline__ uint32_t redc(uint32_t x, uint32_t y, const Fld& f) {
    uint32_t lo = x * y, hi = __umulhi(x, y);
    uint32_t m = lo * f.pinv;
    return hi - __umulhi(m, f.p) + f.p;
}
// [0, 4p) -> [0, p)
__device__ __forceinline__ uint32_t canon4(uint32_t x, const Fld& f) {
    x = umin(x, x - f.p2);
    return umin(x, x - f.p);
}

// ---- register groups on v[16]
// DIF, elements lo + 16 t: level half-spans 128, 64, 32, 16 (h = 8, 4, 2, 1 in t)
template <int NV>
__device__ __forceinline__ void dif_tab(uint32_t (*v)[16], int lo, const uint2* tw, const Fld& f, bool half0) {
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
        for (int t = 0; t < 16; t++) {
            if (t & h) continue;
            const uint2 w = tw[16 * h + lo + 16 * (t & (h - 1))];
#pragma unroll
            for (int u = 0; u < NV; u++) {
                if (h == 8 && half0) v[u][t + 8] = mulw(v[u][t], w, f);   // (x, 0) -> (x, x w)
                else dif(v[u][t], v[u][t + h], w, f);
            }
        }
    }
}
// DIF, 16 consecutive elements: half-spans 8, 4, 2, 1 with constant twiddles
__device__ __forceinline__ void dif_const(uint32_t* v, const Tw15& T, const Fld& f) {
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
        for (int t = 0; t < 16; t++) {
            if (t & h) continue;
            const int k = t & (h - 1);
            if (k == 0) dif1(v[t], v[t + h], f);
            else dif(v[t], v[t + h], T.w[h + k], f);
        }
    }
}
// DIT, 16 consecutive elements: half-spans 1, 2, 4, 8 with constant twiddles
__device__ __forceinline__ void dit_const(uint32_t* v, const Tw15& T, const Fld& f) {
#pragma unroll
    for (int h = 1; h <= 8; h <<= 1) {
#pragma unroll
        for (int t = 0; t < 16; t++) {
            if (t & h) continue;
            const int k = t & (h - 1);
            const bool xr = h == 1 || (t & (h >> 1)) == 0;
            if (k == 0) {
                if (xr) dit1<true>(v[t], v[t + h], f); else dit1<false>(v[t], v[t + h], f);
            } else {
                if (xr) dit<true>(v[t], v[t + h], T.w[h + k], f); else dit<false>(v[t], v[t + h], T.w[h + k], f);
            }
        }
    }
}
// DIT, elements lo + 16 t: half-spans 16, 32, 64, 128.  XR0: every input in [0, 2p).
template <bool XR0>
__device__ __forceinline__ void dit_tab(uint32_t* v, int lo, const uint2* tw, const Fld& f) {
#pragma unroll
    for (int h = 1; h <= 8; h <<= 1) {
#pragma unroll
        for (int t = 0; t < 16; t++) {
            if (t & h) continue;
            const uint2 w = tw[16 * h + lo + 16 * (t & (h - 1))];
            // level h = 1 of this group takes the previous group's outputs: x' at t with bit 3 clear
            const bool xr = h == 1 ? XR0 : (t & (h >> 1)) == 0;
            if (xr) dit<true>(v[t], v[t + h], w, f); else dit<false>(v[t], v[t + h], w, f);
        }
    }
}

// ---------------------------------------------------------------- column passes
// Tile = one batch row's 256 x 32 block (32 adjacent columns), shared layout
// [t][c] (lane = column: every shared access is conflict-free).  Warp w owns
// the table-group chunks lo in {w, w + 8} and the constant-group chunks
// (rows 16 b .. 16 b + 15) b in {w, w + 8}.  The next tile streams into
// shared memory with cp.async (LDGSTS, zero-filled beyond the valid prefix)
// while the current one is transformed.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, int src_bytes) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// rows [0, RIN) of the 32-column block `tile` -> st[row * 32 + c]; element
// (row, col) of batch row b is in[b * in_bs + row * 256 + col], valid iff
// row * 256 + col < len (zeros beyond).  VEC: 16-byte copies (in_bs % 4 == 0).
template <int RIN, bool MASK, bool VEC>
__device__ __forceinline__ void issue_cols(uint32_t* st, const uint32_t* in, long long tile, long long in_bs,
                                           long long len) {
    const long long b = tile >> 3;
    const int cg = (int)(tile & 7) << 5;
    const uint32_t* src = in + b * in_bs + cg;
    const int lim = (int)(len < (1 << 16) ? len : (1 << 16)) - cg;   // valid iff row * 256 + cc < lim
    if (VEC) {
#pragma unroll
        for (int k = 0; k < RIN * 8 / NT; k++) {
            const int e = threadIdx.x + NT * k, row = e >> 3, cc = (e & 7) * 4;
            int nb = 16;
            if (MASK) {
                const int rem = lim - row * 256 - cc;
                nb = rem <= 0 ? 0 : (rem >= 4 ? 16 : 4 * rem);
            }
            cp_async16(st + row * 32 + cc, nb ? (const void*)(src + row * 256 + cc) : (const void*)in, nb);
        }
    } else {
#pragma unroll
        for (int k = 0; k < RIN * 32 / NT; k++) {
            const int e = threadIdx.x + NT * k, row = e >> 5, cc = e & 31;
            const int nb = (!MASK || row * 256 + cc < lim) ? 4 : 0;
            cp_async4(st + row * 32 + cc, nb ? (const void*)(src + row * 256 + cc) : (const void*)in, nb);
        }
    }
}

template <bool HALF> struct ColFwdSmem {
    static constexpr int RIN = HALF ? 128 : 256;
    static constexpr size_t bytes = 256 * sizeof(uint2) + (RIN + 256) * 32 * sizeof(uint32_t) + 128;
};

// TMA: tensor-map load of the staging tile (in_len a multiple of 256), else
// cp.async with per-element zero fill (MASK, VEC as issue_cols).
template <bool HALF, bool MASK, bool VEC, bool TMA>
__global__ void __launch_bounds__(NT, HALF ? 4 : 3) k_col_fwd(const __grid_constant__ CUtensorMap tm, ColFwdArgs a) {
    constexpr int RIN = ColFwdSmem<HALF>::RIN;
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t* st = (uint32_t*)smem;            // staging: next tile's input rows (TMA destination)
    uint32_t* s = st + RIN * 32;               // working tile
    uint2* tws = (uint2*)(s + 256 * 32);
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 256; i += NT) tws[i] = a.lvl[i];
    const int c = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long ntiles = a.nbatch * 8;
    const Fld f = a.f;
    if (TMA) {
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            mbar_fence_init();
        }
        __syncthreads();
        if (threadIdx.x == 0 && (long long)blockIdx.x < ntiles)
            tma_load_tile(st, &tm, (int)(blockIdx.x & 7) * 32, 0, (int)(blockIdx.x >> 3), &bar, RIN * 128);
    } else {
        if ((long long)blockIdx.x < ntiles) issue_cols<RIN, MASK, VEC>(st, a.in, blockIdx.x, a.in_bs, a.in_len);
        cp_commit();
    }
    unsigned it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        const long long b = tile >> 3;
        const int col = ((int)(tile & 7) << 5) + c;
        if (TMA) mbar_wait(&bar, it & 1);
        else cp_wait_all();
        __syncthreads();
        uint32_t v[2][16];
#pragma unroll
        for (int u = 0; u < 2; u++)
#pragma unroll
            for (int t = 0; t < 16; t++) v[u][t] = (HALF && t >= 8) ? 0u : st[(w + 8 * u + 16 * t) * 32 + c];
        __syncthreads();
        if (TMA) {
            const long long nt = tile + gridDim.x;
            if (threadIdx.x == 0 && nt < ntiles) tma_load_tile(st, &tm, (int)(nt & 7) * 32, 0, (int)(nt >> 3), &bar, RIN * 128);
        } else {
            if (tile + gridDim.x < ntiles) issue_cols<RIN, MASK, VEC>(st, a.in, tile + gridDim.x, a.in_bs, a.in_len);
            cp_commit();
        }
        dif_tab<1>(&v[0], w, tws, f, HALF);
        dif_tab<1>(&v[1], w + 8, tws, f, HALF);
#pragma unroll
        for (int u = 0; u < 2; u++)
#pragma unroll
            for (int t = 0; t < 16; t++) s[(w + 8 * u + 16 * t) * 32 + c] = v[u][t];
        __syncthreads();
        uint32_t* dst = a.out + b * a.out_bs + col;
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int r0 = 16 * (w + 8 * u);
#pragma unroll
            for (int t = 0; t < 16; t++) v[u][t] = s[(r0 + t) * 32 + c];
            dif_const(v[u], a.tc, f);
            // step 2: row r0 + t holds frequency [r0 + t]_8; times w^(col [i2]_8)
#pragma unroll
            for (int t = 0; t < 16; t++) {
                const int row = r0 + t;
                dst[row * 256] = mulw(v[u][t], __ldg(a.fs + row * 256 + col), f);
            }
        }
    }
}

constexpr size_t COL_INV_SMEM = 256 * sizeof(uint2) + 2 * 256 * 32 * sizeof(uint32_t) + 128;

// input tiles by TMA into two alternating buffers (one mbarrier each)
template <bool MASK>
__global__ void __launch_bounds__(NT, 3) k_col_inv(const __grid_constant__ CUtensorMap tm, ColInvArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t* buf = (uint32_t*)smem;           // two 256 x 32 tiles
    uint2* tws = (uint2*)(buf + 2 * 256 * 32);
    __shared__ uint64_t bar[2];
    for (int i = threadIdx.x; i < 256; i += NT) tws[i] = a.lvl[i];
    const int c = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long ntiles = a.nbatch * 8;
    const Fld f = a.f;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && (long long)blockIdx.x < ntiles)
        tma_load_tile(buf, &tm, (int)(blockIdx.x & 7) * 32, 0, (int)(blockIdx.x >> 3), &bar[0], 256 * 128);
    unsigned it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        const long long b = tile >> 3;
        const int col = ((int)(tile & 7) << 5) + c;
        uint32_t* s = buf + (it & 1) * 256 * 32;
        mbar_wait(&bar[it & 1], (it >> 1) & 1);
        __syncthreads();
        const long long nt = tile + gridDim.x;
        if (threadIdx.x == 0 && nt < ntiles)
            tma_load_tile(buf + ((it + 1) & 1) * 256 * 32, &tm, (int)(nt & 7) * 32, 0, (int)(nt >> 3), &bar[(it + 1) & 1],
                          256 * 128);
        uint32_t v[2][16];
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int r0 = 16 * (w + 8 * u);
#pragma unroll
            for (int t = 0; t < 16; t++) v[u][t] = s[(r0 + t) * 32 + c];
            dit_const(v[u], a.tc, f);
#pragma unroll
            for (int t = 0; t < 16; t++) s[(r0 + t) * 32 + c] = v[u][t];
        }
        __syncthreads();
        uint32_t* dst = a.out + b * a.out_bs + col;
        const int lim = (int)(a.out_len - col);
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int lo = w + 8 * u;
#pragma unroll
            for (int t = 0; t < 16; t++) v[u][t] = s[(lo + 16 * t) * 32 + c];
            // phase A left x' (in [0, 2p)) at chunk positions < 8, i.e. rows with lo < 8
            if (u == 0) dit_tab<true>(v[u], lo, tws, f);
            else dit_tab<false>(v[u], lo, tws, f);
#pragma unroll
            for (int t = 0; t < 16; t++) {
                const int row = lo + 16 * t;
                if (!MASK || row * 256 < lim) dst[row * 256] = canon4(v[u][t], f);
            }
        }
    }
}

// ---------------------------------------------------------------- fused product rows
// Tile = 16 rows of 256; thread (r, lo) = (tid >> 4, tid & 15): a warp owns rows
// 2w and 2w + 1 and every shared exchange stays inside them, so the phases
// are separated by __syncwarp, not CTA barriers (warps drift freely and
// interleave their multiply- and add-heavy phases).  Shared rows
// are padded by one 16-byte chunk per 8 (chunk q at q + (q >> 3)) with a row
// pitch of 76 chunks (= 4 mod 8): the strided 4-byte accesses of the table
// groups (16 lanes x 4 chunks per row, two rows per warp) and the 16-byte
// accesses of the constant group (8 lanes per phase) are both conflict-free,
// and every address is a per-thread base plus an immediate.
constexpr int ROWP = 76 * 4;   // words per padded row
__device__ __forceinline__ int pad_word(int j) { return j + 4 * (j >> 5); }   // 4 * ((j >> 2) + (j >> 5)) + (j & 3)

__global__ void __launch_bounds__(NT, 4) k_row_pmul(RowPmulArgs a) {
    __shared__ uint2 twf[256], twi[256];
    __shared__ __align__(16) uint32_t sa[16 * ROWP];
    __shared__ __align__(16) uint32_t sb[16 * ROWP];
    for (int i = threadIdx.x; i < 256; i += NT) {
        twf[i] = a.lvl_f[i];
        twi[i] = a.lvl_i[i];
    }
    const int r = threadIdx.x >> 4, lo = threadIdx.x & 15;
    const long long ntiles = a.nrows >> 4;
    const Fld f = a.f;
    __syncthreads();
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row = tile * 16 + r;
        {   // warm L2 with the next tile's rows (one 128-byte line per thread per
            // operand) so its phase-A loads hit L2 instead of HBM
            const long long nt = tile + gridDim.x;
            if (nt < ntiles) {
                const long long off = nt * 16 * 256 + threadIdx.x * 16;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a.A + off));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a.B + off));
            }
        }
        uint32_t v[2][16];
#pragma unroll
        for (int t = 0; t < 16; t++) {
            v[0][t] = __ldg(a.A + row * 256 + lo + 16 * t);
            v[1][t] = __ldg(a.B + row * 256 + lo + 16 * t);
        }
        dif_tab<2>(v, lo, twf, f, false);
#pragma unroll
        for (int t = 0; t < 16; t++) {
            const int ix = r * ROWP + pad_word(lo + 16 * t);
            sa[ix] = v[0][t];
            sb[ix] = v[1][t];
        }
        __syncwarp();
        // constant group: 16 consecutive spectrum values of both operands
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int ix = r * ROWP + pad_word(16 * lo + 4 * i);
            const uint4 x = *(const uint4*)(sa + ix);
            const uint4 y = *(const uint4*)(sb + ix);
            v[0][4 * i] = x.x; v[0][4 * i + 1] = x.y; v[0][4 * i + 2] = x.z; v[0][4 * i + 3] = x.w;
            v[1][4 * i] = y.x; v[1][4 * i + 1] = y.y; v[1][4 * i + 2] = y.z; v[1][4 * i + 3] = y.w;
        }
        dif_const(v[0], a.tf, f);
        dif_const(v[1], a.tf, f);
#pragma unroll
        for (int t = 0; t < 16; t++) v[0][t] = redc(v[0][t], v[1][t], f);   // P:952 entry-wise product
        dit_const(v[0], a.ti, f);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int ix = r * ROWP + pad_word(16 * lo + 4 * i);
            *(uint4*)(sa + ix) = make_uint4(v[0][4 * i], v[0][4 * i + 1], v[0][4 * i + 2], v[0][4 * i + 3]);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 16; t++) v[0][t] = sa[r * ROWP + pad_word(lo + 16 * t)];
        dit_tab<false>(v[0], lo, twi, f);
        // inverse step 2 (w^-(j1 [i2]_8)) with n^-1 2^32 folded in
        const uint2* fsr = a.fsi + (row & 255) * 256 + lo;
        uint32_t* dst = a.C + row * 256 + lo;
#pragma unroll
        for (int t = 0; t < 16; t++) dst[16 * t] = mulw(v[0][t], __ldg(fsr + 16 * t), f);
        __syncwarp();
    }
}

// ---------------------------------------------------------------- plain row passes (k = 16 transforms)
// Forward: steps 3-4 of a row (DIF, table group then constant group), output
// canonical in the TFT order.  Inverse: DIT (constant group then table group)
// and the inverse step-2 twiddle with n^-1 folded in.  Warp-private rows as in
// k_row_pmul.
__global__ void __launch_bounds__(NT, 4) k_row_fwd(RowArgs32 a) {
    __shared__ uint2 tw[256];
    __shared__ __align__(16) uint32_t sa[16 * ROWP];
    for (int i = threadIdx.x; i < 256; i += NT) tw[i] = a.lvl[i];
    const int r = threadIdx.x >> 4, lo = threadIdx.x & 15;
    const long long ntiles = a.nrows >> 4;
    const Fld f = a.f;
    __syncthreads();
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row = tile * 16 + r;
        uint32_t v[1][16];
#pragma unroll
        for (int t = 0; t < 16; t++) v[0][t] = __ldg(a.in + row * 256 + lo + 16 * t);
        dif_tab<1>(v, lo, tw, f, false);
#pragma unroll
        for (int t = 0; t < 16; t++) sa[r * ROWP + pad_word(lo + 16 * t)] = v[0][t];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint4 x = *(const uint4*)(sa + r * ROWP + pad_word(16 * lo + 4 * i));
            v[0][4 * i] = x.x; v[0][4 * i + 1] = x.y; v[0][4 * i + 2] = x.z; v[0][4 * i + 3] = x.w;
        }
        dif_const(v[0], a.tc, f);
        uint4* dst = (uint4*)(a.out + row * 256 + 16 * lo);
#pragma unroll
        for (int i = 0; i < 4; i++)
            dst[i] = make_uint4(canon4(v[0][4 * i], f), canon4(v[0][4 * i + 1], f), canon4(v[0][4 * i + 2], f),
                                canon4(v[0][4 * i + 3], f));
        __syncwarp();
    }
}

__global__ void __launch_bounds__(NT, 4) k_row_inv(RowArgs32 a) {
    __shared__ uint2 tw[256];
    __shared__ __align__(16) uint32_t sa[16 * ROWP];
    for (int i = threadIdx.x; i < 256; i += NT) tw[i] = a.lvl[i];
    const int r = threadIdx.x >> 4, lo = threadIdx.x & 15;
    const long long ntiles = a.nrows >> 4;
    const Fld f = a.f;
    __syncthreads();
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row = tile * 16 + r;
        uint32_t v[16];
        const uint4* src = (const uint4*)(a.in + row * 256 + 16 * lo);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint4 x = __ldg(src + i);
            v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
        }
        dit_const(v, a.tc, f);
#pragma unroll
        for (int i = 0; i < 4; i++)
            *(uint4*)(sa + r * ROWP + pad_word(16 * lo + 4 * i)) = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 16; t++) v[t] = sa[r * ROWP + pad_word(lo + 16 * t)];
        dit_tab<false>(v, lo, tw, f);
        const uint2* fsr = a.fsi + (row & 255) * 256 + lo;
        uint32_t* dst = a.out + row * 256 + lo;
#pragma unroll
        for (int t = 0; t < 16; t++) dst[16 * t] = mulw(v[t], __ldg(fsr + 16 * t), f);
        __syncwarp();
    }
}

// ---------------------------------------------------------------- natural-order row passes
// NATURAL order without a permutation pass.  The output of Algorithm 1 at
// row i2, position i1 is frequency f1 256 + f2 with f1 = [i1]_8, f2 = [i2]_8
// ([i2 256 + i1]_16 = [i1]_8 256 + [i2]_8).  A tile takes the 16 rows
// whose frequencies f2 = 16 g + r are consecutive (row i2 = [f2]_8), so for
// every f1 it owns 16 consecutive output words (64 B): the row results are
// staged in shared memory as [f1][r] (pitch 17: conflict-free both ways) and
// leave as 128-bit stores.  The inverse reads the natural spectrum the same
// way and hands the rows to the column pass in its usual layout.
constexpr int NATP = 17;            // staging pitch (words) of one f1 row
__device__ __forceinline__ int brev8i(int x) { return (int)(__brev((unsigned)x) >> 24); }

__global__ void __launch_bounds__(NT, 4) k_row_fwd_nat(RowArgs32 a) {
    __shared__ uint2 tw[256];
    __shared__ __align__(16) uint32_t sa[16 * ROWP];   // row exchange, then the [256][NATP] staging
    for (int i = threadIdx.x; i < 256; i += NT) tw[i] = a.lvl[i];
    const int r = threadIdx.x >> 4, lo = threadIdx.x & 15;
    const long long ntiles = a.nrows >> 4;
    const Fld f = a.f;
    __syncthreads();
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long b = tile >> 4;
        const int g = (int)(tile & 15);
        const long long row = b * 256 + brev8i(16 * g + r);
        uint32_t v[1][16];
#pragma unroll
        for (int t = 0; t < 16; t++) v[0][t] = __ldg(a.in + row * 256 + lo + 16 * t);
        dif_tab<1>(v, lo, tw, f, false);
#pragma unroll
        for (int t = 0; t < 16; t++) sa[r * ROWP + pad_word(lo + 16 * t)] = v[0][t];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint4 x = *(const uint4*)(sa + r * ROWP + pad_word(16 * lo + 4 * i));
            v[0][4 * i] = x.x; v[0][4 * i + 1] = x.y; v[0][4 * i + 2] = x.z; v[0][4 * i + 3] = x.w;
        }
        dif_const(v[0], a.tc, f);
        __syncthreads();                                  // every warp is done with its exchange rows
#pragma unroll
        for (int j = 0; j < 16; j++) sa[brev8i(16 * lo + j) * NATP + r] = canon4(v[0][j], f);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; k++) {                     // four lanes per 64-byte segment: whole sectors per warp
            const int f1 = 64 * k + (threadIdx.x >> 2), q = threadIdx.x & 3;
            const uint32_t* src = sa + f1 * NATP + 4 * q;
            *(uint4*)(a.out + b * 65536 + (long long)f1 * 256 + 16 * g + 4 * q) =
                make_uint4(src[0], src[1], src[2], src[3]);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NT, 4) k_row_inv_nat(RowArgs32 a) {
    __shared__ uint2 tw[256];
    __shared__ __align__(16) uint32_t sa[16 * ROWP];
    for (int i = threadIdx.x; i < 256; i += NT) tw[i] = a.lvl[i];
    const int r = threadIdx.x >> 4, lo = threadIdx.x & 15;
    const long long ntiles = a.nrows >> 4;
    const Fld f = a.f;
    __syncthreads();
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long b = tile >> 4;
        const int g = (int)(tile & 15);
        const int i2 = brev8i(16 * g + r);
        {
            uint4 x[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {                 // four lanes per 64-byte segment
                const int f1 = 64 * k + (threadIdx.x >> 2), q = threadIdx.x & 3;
                x[k] = __ldg((const uint4*)(a.in + b * 65536 + (long long)f1 * 256 + 16 * g + 4 * q));
            }
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int f1 = 64 * k + (threadIdx.x >> 2), q = threadIdx.x & 3;
                uint32_t* d = sa + f1 * NATP + 4 * q;
                d[0] = x[k].x; d[1] = x[k].y; d[2] = x[k].z; d[3] = x[k].w;
            }
        }
        __syncthreads();
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = sa[brev8i(16 * lo + j) * NATP + r];   // position 16 lo + j of row i2
        __syncthreads();                                  // staging read before the exchange reuses sa
        dit_const(v, a.tc, f);
#pragma unroll
        for (int i = 0; i < 4; i++)
            *(uint4*)(sa + r * ROWP + pad_word(16 * lo + 4 * i)) = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 16; t++) v[t] = sa[r * ROWP + pad_word(lo + 16 * t)];
        dit_tab<false>(v, lo, tw, f);
        const uint2* fsr = a.fsi + i2 * 256 + lo;
        uint32_t* dst = a.out + (b * 256 + i2) * 256 + lo;
#pragma unroll
        for (int t = 0; t < 16; t++) dst[16 * t] = mulw(v[t], __ldg(fsr + 16 * t), f);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launchers
template <class K> static int grid_of(K kern, long long tiles, size_t smem) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    static const int cap_env = [] {
        const char* e = getenv("MMNTT_CTAS_PER_SM");   // experiment knob: cap resident CTAs per SM
        return e ? atoi(e) : 0;
    }();
    if (cap_env > 0 && per_sm > cap_env) per_sm = cap_env;
    if (per_sm < 1) per_sm = 1;
    long long cap = (long long)num_sms() * per_sm;
    return (int)(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
}

// 3-D map of 32-bit words {256 columns, rows per batch row, batch}, box {32, box_rows, 1}
static mm_status make_col_map(CUtensorMap* tm, const void* base, long long rows, long long batch, long long bstride_words,
                              int box_rows) {
    auto enc = tma_encoder();
    if (!enc) return set_err(MM_E_CUDA, "cuTensorMapEncodeTiled is not available");
    cuuint64_t dims[3] = {256, (cuuint64_t)rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {1024, (cuuint64_t)bstride_words * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(MM_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return MM_OK;
}

template <bool HALF, bool MASK, bool VEC, bool TMA>
static mm_status col_fwd_k(const ColFwdArgs& a, cudaStream_t st) {
    auto kern = k_col_fwd<HALF, MASK, VEC, TMA>;
    const size_t smem = ColFwdSmem<HALF>::bytes;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    if (TMA) {
        mm_status s = make_col_map(&tm, a.in, a.in_len / 256, a.nbatch, a.in_bs, ColFwdSmem<HALF>::RIN);
        if (s != MM_OK) return s;
    }
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    {
        LaunchScope ls("ntt_cols_fwd", st);
        kern<<<grid_of(kern, a.nbatch * 8, smem), NT, smem, st>>>(tm, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
mm_status launch_col_fwd(const ColFwdArgs& a, cudaStream_t st) {
    const bool half = a.in_len <= (1 << 15);
    const bool mask = a.in_len != (half ? (1 << 15) : (1 << 16));
    const bool vec = a.in_bs % 4 == 0 && ((uintptr_t)a.in & 15) == 0;
    // whole 256-element rows at 16-byte aligned strides: the tensor-map load
    const bool tma = vec && a.in_len % 256 == 0 && tma_encoder() != nullptr;
    if (tma) return half ? col_fwd_k<true, false, true, true>(a, st) : col_fwd_k<false, false, true, true>(a, st);
    if (half) {
        if (!mask) return vec ? col_fwd_k<true, false, true, false>(a, st) : col_fwd_k<true, false, false, false>(a, st);
        return vec ? col_fwd_k<true, true, true, false>(a, st) : col_fwd_k<true, true, false, false>(a, st);
    }
    if (!mask) return vec ? col_fwd_k<false, false, true, false>(a, st) : col_fwd_k<false, false, false, false>(a, st);
    return vec ? col_fwd_k<false, true, true, false>(a, st) : col_fwd_k<false, true, false, false>(a, st);
}
mm_status launch_row_pmul(const RowPmulArgs& a, cudaStream_t st) {
    if (a.nrows % 16) return set_err(MM_E_UNSUPPORTED_SIZE, "row count %lld is not a multiple of 16", a.nrows);
    {
        LaunchScope ls("pmul_rows_fourstep", st);
        k_row_pmul<<<grid_of(k_row_pmul, a.nrows / 16, 0), NT, 0, st>>>(a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
mm_status launch_row_fwd(const RowArgs32& a, cudaStream_t st) {
    if (a.nrows % 16 || (((uintptr_t)a.out) & 15)) return set_err(MM_E_ARG, "row pass needs 16-row tiles, aligned rows");
    {
        LaunchScope ls("ntt_rows_fwd", st);
        k_row_fwd<<<grid_of(k_row_fwd, a.nrows / 16, 0), NT, 0, st>>>(a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
mm_status launch_row_inv(const RowArgs32& a, cudaStream_t st) {
    if (a.nrows % 16 || (((uintptr_t)a.in) & 15)) return set_err(MM_E_ARG, "row pass needs 16-row tiles, aligned rows");
    {
        LaunchScope ls("ntt_rows_inv", st);
        k_row_inv<<<grid_of(k_row_inv, a.nrows / 16, 0), NT, 0, st>>>(a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
mm_status launch_row_fwd_nat(const RowArgs32& a, cudaStream_t st) {
    if (a.nrows % 256 || (((uintptr_t)a.out) & 15)) return set_err(MM_E_ARG, "natural row pass needs whole 2^16 rows");
    {
        LaunchScope ls("ntt_rows_fwd_natural", st);
        k_row_fwd_nat<<<grid_of(k_row_fwd_nat, a.nrows / 16, 0), NT, 0, st>>>(a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
mm_status launch_row_inv_nat(const RowArgs32& a, cudaStream_t st) {
    if (a.nrows % 256 || (((uintptr_t)a.in) & 15)) return set_err(MM_E_ARG, "natural row pass needs whole 2^16 rows");
    {
        LaunchScope ls("ntt_rows_inv_natural", st);
        k_row_inv_nat<<<grid_of(k_row_inv_nat, a.nrows / 16, 0), NT, 0, st>>>(a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
mm_status launch_col_inv(const ColInvArgs& a, cudaStream_t st) {
    if (a.in_bs % 4 || ((uintptr_t)a.in & 15)) return set_err(MM_E_ARG, "inverse column pass needs 16-byte aligned rows");
    auto kern = a.out_len == (1 << 16) ? k_col_inv<false> : k_col_inv<true>;
    CUtensorMap tm;
    mm_status s = make_col_map(&tm, a.in, 256, a.nbatch, a.in_bs, 256);
    if (s != MM_OK) return s;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)COL_INV_SMEM));
    {
        LaunchScope ls("ntt_cols_inv", st);
        kern<<<grid_of(kern, a.nbatch * 8, COL_INV_SMEM), NT, COL_INV_SMEM, st>>>(tm, a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

}  // namespace f32
}  // namespace mm
