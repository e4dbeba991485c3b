// tft.h -- inverse truncated Fourier transform over the columns of a
// truncated four-step product (tft.cu).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>
#include "../../include/mmntt.h"

namespace mm {
namespace tft {

struct ItftArgs {
    const uint32_t* in;     // [nbatch][lam][n1] (row stride n1, batch stride in_bs)
    uint32_t* out;          // [nbatch][out_len] (batch stride out_bs): coefficient t n1 + j1
    long long nbatch, in_bs, out_bs, out_len, n1;
    int k2, lam, cols;      // column length 2^k2, lambda rows kept, columns per tile (launcher)
    uint32_t p;
    const uint2* lvl_f;     // column level tables (root w^n1 and its inverse), Shoup pairs
    const uint2* lvl_i;
    uint2 inv2;             // 2^-1 and (2^j)^-1, j <= k2, with companions
    uint2 inv_pow2[11];
};

mm_status launch_col_itft(const ItftArgs& a, cudaStream_t st);

}  // namespace tft
}  // namespace mm
