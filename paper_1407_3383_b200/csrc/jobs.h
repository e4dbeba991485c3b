// jobs.h -- device form of the mm_run_jobs table (jobs.cu): one CTA per job,
// the table passed by value as the kernel parameter.
#pragma once
#include "common.h"
#include "arith.cuh"

namespace mm {

struct DevJob {
    int kind, k, order;
    Fp32 f;
    uint2 sc;                  // n^-1 (inverse, round trip) or n^-1 2^32 (product, after REDC), Shoup pair
    const uint2* lvl_f;        // level tables of the single-pass plan
    const uint2* lvl_i;
    const uint32_t* in;
    const uint32_t* in2;
    uint32_t* out;
    uint32_t* out2;
    long long la, lb;
};
constexpr int JOBS_SMALL = 32, JOBS_LARGE = 256;   // JobPack<256>: ~26 KiB of the 32 KiB parameter space
template <int MAXJ> struct JobPack {
    int n;
    DevJob job[MAXJ];
};
mm_status launch_jobs(const DevJob* jobs, int njobs, cudaStream_t st);

}  // namespace mm
