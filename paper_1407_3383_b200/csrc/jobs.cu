// jobs.cu -- many small independent 32-bit problems in ONE launch.
//
// A CTA per job: forward / inverse transforms of one row of length 2^k
// (k <= 12, single-pass plans), a forward-then-inverse round trip (the
// inverse(forward(x)) = x check of P:923 / BASELINE C1, the forward spectrum
// kept in shared memory between the two), and the product of two
// polynomials (two direct transforms, the entry-wise product with n^-1
// folded in, one inverse).  Small transforms are bound by launch latency, not
// by the GPU (BASELINE C1: 16 round trips of 2^10 plus a 512 x 512 product
// took three dependent launches, ~6 us each); here they take one.  The job
// table travels as a kernel parameter (no upload), the tiles and butterflies
// are the single-pass row kernels' (ntt_core.cuh).
#include <memory>
#include <new>
#include "ntt_kernels.cuh"
#include "jobs.h"

namespace mm {

// one row per tile; two (the second empty) for n = 2, so that the row I/O's
// 16-byte vector loops have a vector to move
template <int LOGL> struct JobLay { typedef RowLayout<uint32_t, LOGL, (1 << LOGL) >= 4 ? 1 : 2> Lay; };
constexpr int JNT = 256;
constexpr size_t JOB_SMEM = 2 * (size_t)RowLayout<uint32_t, 12, 1>::ELEMS * 4;

template <int LOGL> __device__ __forceinline__ void run_job(const DevJob& j, uint32_t* sa, uint32_t* sb) {
    typedef typename JobLay<LOGL>::Lay Lay;
    constexpr int L = 1 << LOGL;
    const Fp32 f = j.f;
    const uint2 zero{0u, 0u};
    auto vec = [](const void* p) { return L >= 4 && ((uintptr_t)p & 15) == 0; };
    const bool nat = j.order == MM_ORDER_NATURAL;
    if (j.kind == MM_JOB_POLY_MUL) {
        // a and b as the two rows of one tile: both forward transforms run in
        // the same passes (a small transform leaves most threads idle)
        typedef RowLayout<uint32_t, LOGL, 2> Lay2;
        static_assert(Lay2::SROW == Lay::SROW, "row pitch independent of the row count");
        const long long lc = j.la + j.lb - 1;
        sb = sa + Lay::SROW;
        load_rows<Fp32, Lay, LOGL, uint32_t, JNT>(sa, j.in, 0, 1, L, j.la, vec(j.in), false);
        if (Lay::C > 1) __syncthreads();   // n = 2: a's load zero-fills the empty second row
        load_rows<Fp32, Lay, LOGL, uint32_t, JNT>(sb, j.in2, 0, 1, L, j.lb, vec(j.in2), false);
        __syncthreads();
        run_tile<Fp32, Lay2, LOGL, false, JNT>(f, sa, j.lvl_f, j.lvl_f);
        constexpr int R = L < 16 ? L : 16;
        for (int ch = threadIdx.x; ch < L / R; ch += JNT) {
            const int base = Lay::chunk_base(0, ch * R);
#pragma unroll
            for (int t = 0; t < R; t++) sa[base + t] = f.mulw(f.mul_redc(sa[base + t], sb[base + t]), j.sc);
        }
        __syncthreads();
        run_tile<Fp32, Lay, LOGL, true, JNT>(f, sa, j.lvl_i, j.lvl_i);
        store_rows<Fp32, Lay, LOGL, uint32_t, EPI_CANON, JNT>(f, sa, j.out, 0, 1, L, lc, vec(j.out), false, nullptr,
                                                            nullptr, nullptr, 0, 0, 0, zero);
        return;
    }
    if (j.kind == MM_JOB_INVERSE) {
        load_rows<Fp32, Lay, LOGL, uint32_t, JNT>(sa, j.in, 0, 1, L, L, vec(j.in), nat);
        __syncthreads();
        run_tile<Fp32, Lay, LOGL, true, JNT>(f, sa, j.lvl_i, j.lvl_i);
        store_rows<Fp32, Lay, LOGL, uint32_t, EPI_SCALE | EPI_CANON, JNT>(f, sa, j.out, 0, 1, L, L, vec(j.out), false,
                                                                        nullptr, nullptr, nullptr, 0, 0, 0, j.sc);
        return;
    }
    // forward (and the first half of a round trip)
    load_rows<Fp32, Lay, LOGL, uint32_t, JNT>(sa, j.in, 0, 1, L, L, vec(j.in), false);
    __syncthreads();
    run_tile<Fp32, Lay, LOGL, false, JNT>(f, sa, j.lvl_f, j.lvl_f);
    if (j.out)
        store_rows<Fp32, Lay, LOGL, uint32_t, EPI_CANON, JNT>(f, sa, j.out, 0, 1, L, L, vec(j.out) && !nat, nat,
                                                            nullptr, nullptr, nullptr, 0, 0, 0, zero);
    if (j.kind != MM_JOB_ROUNDTRIP) return;
    // round trip: the DIF left the spectrum in bit-reversed positions in [0, 2p),
    // exactly the DIT's input
    __syncthreads();
    run_tile<Fp32, Lay, LOGL, true, JNT>(f, sa, j.lvl_i, j.lvl_i);
    store_rows<Fp32, Lay, LOGL, uint32_t, EPI_SCALE | EPI_CANON, JNT>(f, sa, j.out2, 0, 1, L, L, vec(j.out2), false,
                                                                    nullptr, nullptr, nullptr, 0, 0, 0, j.sc);
}

template <int MAXJ> __global__ void __launch_bounds__(JNT) k_jobs(const __grid_constant__ JobPack<MAXJ> pk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* sa = (uint32_t*)smem_raw;
    uint32_t* sb = sa + RowLayout<uint32_t, 12, 1>::ELEMS;
    const DevJob& j = pk.job[blockIdx.x];
    switch (j.k) {
#define MM_JOB_CASE(K) \
    case K: run_job<K>(j, sa, sb); break;
        MM_JOB_CASE(1) MM_JOB_CASE(2) MM_JOB_CASE(3) MM_JOB_CASE(4) MM_JOB_CASE(5) MM_JOB_CASE(6)
        MM_JOB_CASE(7) MM_JOB_CASE(8) MM_JOB_CASE(9) MM_JOB_CASE(10) MM_JOB_CASE(11) MM_JOB_CASE(12)
#undef MM_JOB_CASE
        default: break;
    }
}

template <int MAXJ> static mm_status launch_pack(const JobPack<MAXJ>& pk, cudaStream_t st) {
    auto kern = k_jobs<MAXJ>;
    MM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)JOB_SMEM));
    {
        LaunchScope ls("jobs", st);
        kern<<<pk.n, JNT, JOB_SMEM, st>>>(pk);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

mm_status launch_jobs(const DevJob* jobs, int njobs, cudaStream_t st) {
    for (int j0 = 0; j0 < njobs;) {
        const int n = njobs - j0;
        mm_status s;
        if (n <= JOBS_SMALL) {
            JobPack<JOBS_SMALL> pk;
            pk.n = n;
            for (int i = 0; i < n; i++) pk.job[i] = jobs[j0 + i];
            s = launch_pack(pk, st);
            j0 += n;
        } else {
            std::unique_ptr<JobPack<JOBS_LARGE>> pk(new (std::nothrow) JobPack<JOBS_LARGE>);   // 26 KiB: heap
            if (!pk) return set_err(MM_E_ARG, "out of host memory");
            const int m = n < JOBS_LARGE ? n : JOBS_LARGE;
            pk->n = m;
            for (int i = 0; i < m; i++) pk->job[i] = jobs[j0 + i];
            s = launch_pack(*pk, st);
            j0 += m;
        }
        if (s != MM_OK) return s;
    }
    return MM_OK;
}

}  // namespace mm
