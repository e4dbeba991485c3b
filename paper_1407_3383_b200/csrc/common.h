// common.h -- host-side helpers shared by the library's translation units:
// status / thread-local error text, CUDA error mapping, device queries, and
// host modular arithmetic for plan/context constants.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include "../../include/mmntt.h"

namespace mm {

mm_status set_err(mm_status s, const char *fmt, ...);
int num_sms();
bool debug_checks();
// Stream-ordered allocation from the library's own memory pool (one per
// device, release threshold unlimited: freed blocks stay in the pool for the
// next call instead of going back to the driver at every synchronisation;
// mm_release_cached trims it).  Used for every temporary and workspace.
cudaError_t alloc_async(void **p, size_t bytes, cudaStream_t st);
void trim_pool();
// MMNTT_DEBUG=1 range check of [rows][len] residues at row stride ld (word_bits
// 32 / 64: integers < p; 52: integral doubles in [0, p)); synchronises st
mm_status check_rows(const void *x, int word_bits, size_t rows, size_t len, size_t ld, uint64_t p, cudaStream_t st);

typedef unsigned __int128 u128;
static inline uint64_t hmulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)a * b) % p); }
static inline uint64_t hpowmod(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    b %= p;
    while (e) {
        if (e & 1) r = hmulmod(r, b, p);
        b = hmulmod(b, b, p);
        e >>= 1;
    }
    return r;
}
// Miller-Rabin, deterministic for 64-bit inputs with the first 12 prime bases.
bool hprime(uint64_t n);
static inline int two_adicity(uint64_t p) {
    uint64_t d = p - 1;
    int l = 0;
    while (d && !(d & 1)) { d >>= 1; l++; }
    return l;
}
static inline uint32_t inv_mod_2_32(uint32_t p) {  // Newton: x <- x (2 - p x)
    uint32_t x = p;                                  // correct to 3 bits for odd p
    for (int i = 0; i < 5; i++) x *= 2 - p * x;
    return x;
}

}  // namespace mm

#define MM_CUDA_TRY(call)                                                                   \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) {                                                            \
            cudaGetLastError(); /* clear the sticky-free error so later calls start clean */ \
            return mm::set_err(MM_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
        }                                                                                   \
    } while (0)

#define MM_LAUNCH_CHECK()                                                                    \
    do {                                                                                     \
        cudaError_t e_ = cudaGetLastError();                                                 \
        if (e_ != cudaSuccess)                                                               \
            return mm::set_err(MM_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e_)); \
    } while (0)

namespace mm {
// Instrumentation (mm_launch_count / mm_prof_*): every kernel launch site
// opens a LaunchScope, which counts the launch and, when profiling is on,
// brackets it with CUDA events on the launching stream.
struct LaunchScope {
    LaunchScope(const char *name, cudaStream_t st);
    ~LaunchScope();
    const char *name;
    cudaStream_t st;
    int slot;
};
}  // namespace mm
