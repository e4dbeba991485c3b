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
// x_i = u_i - y_i.  One warp runs the (uniform) control flow of one column,
// held transposed in shared memory; values canonical in [0, p), p < 2^30.
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

constexpr int NT = 256;

// inverse DIF block of size h (bit-mirrored values -> natural inputs), times h^-1
__device__ __forceinline__ void full_inverse(uint32_t* s, int h, const uint2* twi, uint2 invh, uint32_t p, int lane) {
    for (int m = 1; m < h; m <<= 1) {
        for (int idx = lane; idx < h / 2; idx += 32) {
            const int k = idx & (m - 1), j = ((idx - k) << 1) + k;
            const uint32_t x = s[j], t = mulc(s[j + m], twi[m + k], p);
            s[j] = addm(x, t, p);
            s[j + m] = subm(x, t, p);
        }
        __syncwarp();
    }
    for (int i = lane; i < h; i += 32) s[i] = mulc(s[i], invh, p);
    __syncwarp();
}

__global__ void __launch_bounds__(NT) k_col_itft(ItftArgs a) {
    extern __shared__ uint32_t sm[];
    const int n2 = 1 << a.k2, C = a.cols, pitch = n2 + 1;
    const uint32_t p = a.p;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long groups = a.n1 / C, ntiles = groups * a.nbatch;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long b = tile / groups;
        const long long col0 = (tile - b * groups) * C;
        const uint32_t* src = a.in + b * a.in_bs + col0;
        // rows t < lambda of C columns -> sm[c pitch + t]; zeros beyond lambda (known inputs)
        for (int e = threadIdx.x; e < n2 * C; e += NT) {
            const int t = e / C, c = e - t * C;
            sm[c * pitch + t] = t < a.lam ? src[(long long)t * a.n1 + c] : 0u;
        }
        __syncthreads();
        for (int c = warp; c < C; c += NT / 32) {
            uint32_t* s = sm + c * pitch;
            int stb[12], stn[12], stl[12], stk[12], depth = 0;
            int bb = 0, N = n2, l = a.lam, lg = a.k2;      // N = 2^lg
            while (N > 1 && l > 0 && l < N) {
                const int h = N >> 1;
                if (l >= h) {
                    full_inverse(s + bb, h, a.lvl_i, a.inv_pow2[lg - 1], p, lane);   // scale h^-1
                    for (int i = l - h + lane; i < h; i += 32) {
                        const uint32_t y = s[bb + h + i];
                        const uint32_t x = subm(s[bb + i], y, p);
                        s[bb + i] = x;
                        s[bb + h + i] = mulc(subm(x, y, p), a.lvl_f[h + i], p);
                    }
                    __syncwarp();
                    stb[depth] = bb; stn[depth] = N; stl[depth] = l; stk[depth] = 0; depth++;
                    bb += h; N = h; l -= h; lg--;
                } else {
                    for (int i = l + lane; i < h; i += 32) s[bb + i] = addm(s[bb + i], s[bb + h + i], p);
                    __syncwarp();
                    stb[depth] = bb; stn[depth] = N; stl[depth] = l; stk[depth] = 1; depth++;
                    N = h; lg--;
                }
            }
            if (l == N && N > 1) full_inverse(s + bb, N, a.lvl_i, a.inv_pow2[lg], p, lane);
            while (depth > 0) {
                depth--;
                const int b0 = stb[depth], h = stn[depth] >> 1, l0 = stl[depth];
                if (stk[depth] == 0) {
                    for (int i = lane; i < l0 - h; i += 32) {
                        const uint32_t u = s[b0 + i], t = mulc(s[b0 + h + i], a.lvl_i[h + i], p);   // t = v / w_i
                        s[b0 + i] = mulc(addm(u, t, p), a.inv2, p);
                        s[b0 + h + i] = mulc(subm(u, t, p), a.inv2, p);
                    }
                } else {
                    for (int i = lane; i < l0; i += 32) s[b0 + i] = subm(s[b0 + i], s[b0 + h + i], p);
                }
                __syncwarp();
            }
        }
        __syncthreads();
        // coefficients c_{t n1 + col} for t < lambda, truncated to out_len
        uint32_t* dst = a.out + b * a.out_bs + col0;
        for (int e = threadIdx.x; e < a.lam * C; e += NT) {
            const int t = e / C, c = e - t * C;
            if ((long long)t * a.n1 + col0 + c < a.out_len) dst[(long long)t * a.n1 + c] = sm[c * pitch + t];
        }
        __syncthreads();
    }
}

mm_status launch_col_itft(const ItftArgs& a0, cudaStream_t st) {
    ItftArgs a = a0;
    if (a.k2 < 1 || a.k2 > 10) return set_err(MM_E_UNSUPPORTED_SIZE, "inverse TFT columns of 2^%d points", a.k2);
    const int n2 = 1 << a.k2;
    a.cols = 8192 / n2 < 32 ? 8192 / n2 : 32;
    if (a.cols < 8) a.cols = 8;
    if (a.n1 % a.cols) return set_err(MM_E_UNSUPPORTED_SIZE, "n1 = %lld not a multiple of %d", a.n1, a.cols);
    const size_t smem = (size_t)a.cols * (n2 + 1) * sizeof(uint32_t);
    MM_CUDA_TRY(cudaFuncSetAttribute(k_col_itft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long tiles = a.n1 / a.cols * a.nbatch;
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
