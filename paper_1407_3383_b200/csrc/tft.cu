// tft.cu -- inverse truncated Fourier transform along the columns of
// Algorithm 1.
//
// A truncated product keeps only lambda = ceil(l / n1) rows of the four-step
// layout (Algorithm 1's output A(w^[i]_k), i < lambda n1).  After the inverse
// row passes, column j1 holds C(w2^[t]) for t < lambda, where C(X) =
// sum_{j2 < lambda} c_{j2 n1 + j1} X^j2 (coefficients beyond lambda vanish)
// and w2 = w^n1.  Recovering c from those lambda values is the inverse TFT of
// [40] (van der Hoeven): over the DIF network of length n2, with outputs
// [0, l) and inputs [l, N) known, descend one half at a time --
//   l >= N/2: invert the first half completely (u_i = x_i + y_i), turn the
//             known inputs y_i (i >= l - N/2) into known inputs of the second
//             half, v_i = (u_i - 2 y_i) w_i, and descend into it;
//   l <  N/2: the first half's inputs u_i = x_i + y_i are known for i >= l;
//             descend into the first half;
// and on the way back recover x_i, y_i = (u_i +- v_i / w_i) / 2, resp.
// x_i = u_i - y_i.  The control flow depends only on (n2, lambda), so one
// CTA runs it for a tile of 32 columns together: the column tile sits in
// shared memory as [t][32] (a warp touches one row, 32 banks), every step
// spreads (butterfly, column) pairs over the block with a barrier between
// steps, and the inverse blocks run two DIT levels per pass (radix 4 in
// registers).  Twiddles are block-uniform (smem broadcast).  Values are
// canonical in [0, p), p < 2^30.
#include "common.h"
#include "arith.cuh"
#include "tft.h"

namespace mm {
namespace tft {

__device__ __forceinline__ uint32_t addm(uint32_t x, uint32_t y, uint32_t p) { const uint32_t s = x + y; return s >= p ? s - p : s; }
__device__ __forceinline__ uint32_t subm(uint32_t x, uint32_t y, uint32_t p) { return x >= y ? x - y : x + p - y; }
__device__ __forceinline__ uint32_t mulc(uint32_t x, uint2 w, uint32_t p) {   // Function 8, canonical
    const uint32_t c = __umulhi(x, w.y);
    const uint32_t r = x * w.x - c * p;
    return r >= p ? r - p : r;
}

constexpr int NT = 256, C = 32;

// inverse DIT over rows [bb, bb + h) of the tile (bit-mirrored values ->
// natural), times `scale` = h^-1: a radix-2 level first when log2 h is odd,
// then pairs of levels (m, 2m) per pass
__device__ __forceinline__ void full_inverse(uint32_t* s, int bb, int h, const uint2* twi, uint2 scale, uint32_t p) {
    if (h == 1) return;
    int m = 1;
    const int lg = 31 - __clz(h);
    if (lg & 1) {
        const bool last = h == 2;
        for (int e = threadIdx.x; e < (h >> 1) * C; e += NT) {
            const int j = (e >> 5) << 1, c = e & (C - 1);
            uint32_t* r = s + (bb + j) * C + c;
            const uint32_t x = r[0], y = r[C];
            uint32_t u = addm(x, y, p), v = subm(x, y, p);
            if (last) { u = mulc(u, scale, p); v = mulc(v, scale, p); }
            r[0] = u;
            r[C] = v;
        }
        __syncthreads();
        m = 2;
    }
    for (; m < h; m <<= 2) {
        const bool last = 4 * m == h;
        for (int e = threadIdx.x; e < (h >> 2) * C; e += NT) {
            const int q = e >> 5, c = e & (C - 1), k = q & (m - 1), j = ((q - k) << 2) + k;
            uint32_t* r = s + (bb + j) * C + c;
            uint32_t x0 = r[0], x1 = r[m * C], x2 = r[2 * m * C], x3 = r[3 * m * C];
            const uint2 w1 = twi[m + k], w2 = twi[2 * m + k], w3 = twi[3 * m + k];
            uint32_t t = mulc(x1, w1, p);
            x1 = subm(x0, t, p); x0 = addm(x0, t, p);
            t = mulc(x3, w1, p);
            x3 = subm(x2, t, p); x2 = addm(x2, t, p);
            t = mulc(x2, w2, p);
            x2 = subm(x0, t, p); x0 = addm(x0, t, p);
            t = mulc(x3, w3, p);
            x3 = subm(x1, t, p); x1 = addm(x1, t, p);
            if (last) { x0 = mulc(x0, scale, p); x1 = mulc(x1, scale, p); x2 = mulc(x2, scale, p); x3 = mulc(x3, scale, p); }
            r[0] = x0; r[m * C] = x1; r[2 * m * C] = x2; r[3 * m * C] = x3;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NT) k_col_itft(ItftArgs a) {
    extern __shared__ uint32_t sm[];
    const int n2 = 1 << a.k2;
    uint2* twf = (uint2*)sm;          // column level tables (forward, inverse)
    uint2* twi = twf + n2;
    uint32_t* s = (uint32_t*)(twi + n2);
    const uint32_t p = a.p;
    for (int i = threadIdx.x; i < n2; i += NT) { twf[i] = a.lvl_f[i]; twi[i] = a.lvl_i[i]; }
    const long long groups = a.n1 / C, ntiles = groups * a.nbatch;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long b = tile / groups;
        const long long col0 = (tile - b * groups) * C;
        const uint32_t* src = a.in + b * a.in_bs + col0;
        // rows t < lambda of 32 columns (canonicalised); rows beyond lambda are the known (zero) inputs
        for (int e = threadIdx.x; e < n2 * C; e += NT) {
            const int t = e >> 5, c = e & (C - 1);
            uint32_t x = t < a.lam ? src[(long long)t * a.n1 + c] : 0u;
            x = x >= 2 * p ? x - 2 * p : x;        // row-pass output is in [0, 4p)
            s[e] = x >= p ? x - p : x;
        }
        __syncthreads();
        unsigned kinds = 0;
        int bb = 0, N = n2, l = a.lam, lg = a.k2, depth = 0;      // N = 2^lg
        while (N > 1 && l > 0 && l < N) {
            const int h = N >> 1;
            if (l >= h) {
                full_inverse(s, bb, h, twi, a.inv_pow2[lg - 1], p);   // first half, scaled h^-1
                for (int e = threadIdx.x; e < (2 * h - l) * C; e += NT) {
                    const int i = l - h + (e >> 5), c = e & (C - 1);
                    const uint32_t y = s[(bb + h + i) * C + c];
                    const uint32_t x = subm(s[(bb + i) * C + c], y, p);
                    s[(bb + i) * C + c] = x;
                    s[(bb + h + i) * C + c] = mulc(subm(x, y, p), twf[h + i], p);
                }
                bb += h; l -= h;
            } else {
                kinds |= 1u << depth;
                for (int e = threadIdx.x; e < (h - l) * C; e += NT) {
                    const int i = l + (e >> 5), c = e & (C - 1);
                    s[(bb + i) * C + c] = addm(s[(bb + i) * C + c], s[(bb + h + i) * C + c], p);
                }
            }
            __syncthreads();
            N = h; lg--; depth++;
        }
        if (l == N) full_inverse(s, bb, N, twi, a.inv_pow2[lg], p);
        while (depth > 0) {
            depth--;
            const int h = N;
            N <<= 1;
            if (kinds >> depth & 1) {      // first-half descent: x_i = u_i - y_i, i < l
                for (int e = threadIdx.x; e < l * C; e += NT) {
                    const int i = e >> 5, c = e & (C - 1);
                    s[(bb + i) * C + c] = subm(s[(bb + i) * C + c], s[(bb + h + i) * C + c], p);
                }
            } else {                       // second-half descent: (u_i +- v_i / w_i) / 2, i < l
                bb -= h;
                for (int e = threadIdx.x; e < l * C; e += NT) {
                    const int i = e >> 5, c = e & (C - 1);
                    const uint32_t u = s[(bb + i) * C + c], t = mulc(s[(bb + h + i) * C + c], twi[h + i], p);
                    s[(bb + i) * C + c] = mulc(addm(u, t, p), a.inv2, p);
                    s[(bb + h + i) * C + c] = mulc(subm(u, t, p), a.inv2, p);
                }
                l += h;
            }
            __syncthreads();
        }
        // coefficients c_{t n1 + col} for t < lambda, truncated to out_len
        uint32_t* dst = a.out + b * a.out_bs + col0;
        for (int e = threadIdx.x; e < a.lam * C; e += NT) {
            const int t = e >> 5, c = e & (C - 1);
            if ((long long)t * a.n1 + col0 + c < a.out_len) dst[(long long)t * a.n1 + c] = s[e];
        }
        __syncthreads();
    }
}

mm_status launch_col_itft(const ItftArgs& a0, cudaStream_t st) {
    ItftArgs a = a0;
    if (a.k2 < 1 || a.k2 > 10) return set_err(MM_E_UNSUPPORTED_SIZE, "inverse TFT columns of 2^%d points", a.k2);
    const int n2 = 1 << a.k2;
    a.cols = C;
    if (a.n1 % C) return set_err(MM_E_UNSUPPORTED_SIZE, "n1 = %lld not a multiple of %d", a.n1, C);
    const size_t smem = (size_t)n2 * (C * sizeof(uint32_t) + 2 * sizeof(uint2));
    MM_CUDA_TRY(cudaFuncSetAttribute(k_col_itft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long tiles = a.n1 / C * a.nbatch;
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_col_itft, NT, smem);
    if (per < 1) per = 1;
    const int grid = (int)(tiles < (long long)num_sms() * per ? tiles : (long long)num_sms() * per);
    {
        LaunchScope ls("tft_cols_inv", st);
        k_col_itft<<<grid, NT, smem, st>>>(a);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

}  // namespace tft
}  // namespace mm
