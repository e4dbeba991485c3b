// fast32.h -- host interface of the specialised 32-bit four-step kernels
// (ntt_fast32.cu) for n = 2^16 = n2 x n1 with n1 = n2 = 256 (BASELINE C3:
// products of two polynomials of degree < 2^15 over p < 2^30).
//
// The generic tile kernels (ntt_kernels.cuh) serve every size; these three
// kernels are the same Algorithm 1 with l = n, written for the
// one shape the headline workload uses so that every index is a compile-time
// constant and each element crosses shared memory once per pass:
//
//   k_col_fwd  : steps 1-2 -- 32 columns per tile, column DIF of length 256
//                (two radix-16 register groups, one shared-memory exchange),
//                times w^(j1 [i2]_8); inputs with la <= n/2 skip the zero half.
//   k_row_pmul : steps 3-4 of both operands, the pointwise product,
//                the inverse steps 4-3 and the inverse step-2 twiddle with
//                n^-1 folded into its table -- 16 rows per tile.
//   k_col_inv  : inverse step 1 (column DIT) and canonical output, truncated
//                to the product length.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>
#include "../../include/mmntt.h"

namespace mm {
namespace f32 {

struct Tw15 { uint2 w[16]; };        // level-table entries 1..15 (w_{2m}^i, m = 1, 2, 4, 8), by value
struct Fld { uint32_t p, p2, pinv; };

struct ColFwdArgs {
    const uint32_t* in;
    uint32_t* out;
    long long nbatch, in_bs, in_len, out_bs;
    const uint2* lvl;   // column level table (256 entries, root w^n1)
    const uint2* fs;    // step-2 table [i2 * 256 + j1] = w^(j1 [i2]_8)
    Tw15 tc;            // lvl[1..15]
    Fld f;
};
struct RowPmulArgs {
    const uint32_t* A;
    const uint32_t* B;
    uint32_t* C;
    long long nrows;    // rows of 256 (batch * 256)
    const uint2* lvl_f; // row level tables (root w^n2 and its inverse)
    const uint2* lvl_i;
    const uint2* fsi;   // [i2 * 256 + j1] = w^-(j1 [i2]_8) n^-1 2^32 mod p
    Tw15 tf, ti;        // lvl_f[1..15], lvl_i[1..15]
    Fld f;
};
struct ColInvArgs {
    const uint32_t* in;
    uint32_t* out;
    long long nbatch, in_bs, out_bs, out_len;
    const uint2* lvl;   // inverse column level table
    Tw15 tc;
    Fld f;
};

// plain row passes for the standalone transforms (mm_ntt_forward / inverse, k = 16)
struct RowArgs32 {
    const uint32_t* in;
    uint32_t* out;
    long long nrows;    // rows of 256
    const uint2* lvl;   // row level table (forward or inverse root)
    const uint2* fsi;   // inverse only: [i2 * 256 + j1] = w^-(j1 [i2]_8) n^-1
    Tw15 tc;            // lvl[1..15]
    Fld f;
};

mm_status launch_col_fwd(const ColFwdArgs& a, cudaStream_t st);
mm_status launch_row_fwd(const RowArgs32& a, cudaStream_t st);
mm_status launch_row_inv(const RowArgs32& a, cudaStream_t st);
mm_status launch_row_pmul(const RowPmulArgs& a, cudaStream_t st);
mm_status launch_col_inv(const ColInvArgs& a, cudaStream_t st);
// NATURAL-order variants of the plain row passes (no permutation pass):
// forward rows -> natural spectrum; natural spectrum -> inverse rows
mm_status launch_row_fwd_nat(const RowArgs32& a, cudaStream_t st);
mm_status launch_row_inv_nat(const RowArgs32& a, cudaStream_t st);

}  // namespace f32
}  // namespace mm
