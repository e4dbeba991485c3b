// probe.cu -- measurement helpers (not part of the method): integer-issue
// probes that give the ALU roofline of the NTT kernels on this GPU.
//
// mm_probe_butterfly32: every thread keeps 16 residues in registers and runs
// radix-16 DIF groups (the exact Fp32::dif butterfly of the NTT kernels, with
// twiddles held in registers) `iters` times -- no memory traffic, so the rate
// is the integer-pipe ceiling for the 32-bit butterfly.
// mm_probe_butterfly64: the same for the Goldilocks butterfly (radix 8).
#include "common.h"
#include "arith.cuh"
#include "gold.cuh"

namespace mm {

template <int R>
__global__ void __launch_bounds__(256) k_probe_bfly32(Fp32 f, uint2 w0, int iters, uint32_t* sink) {
    uint32_t v[R];
    uint2 w[R / 2];
#pragma unroll
    for (int t = 0; t < R; t++) v[t] = (threadIdx.x * 2654435761u + t * 40503u + blockIdx.x) % f.p;
#pragma unroll
    for (int t = 0; t < R / 2; t++) w[t] = make_uint2(w0.x + t, w0.y + t);   // distinct twiddles (values irrelevant)
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
            for (int t = 0; t < R; t++) {
                if (t & h) continue;
                f.dif(v[t], v[t + h], w[(t & (h - 1)) % (R / 2)]);
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int t = 0; t < R; t++) acc ^= v[t];
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int R>
__global__ void __launch_bounds__(256) k_probe_bfly64(int iters, uint64_t* sink) {
    FpG f;
    uint64_t v[R];
    uint64_t w[R / 2];
#pragma unroll
    for (int t = 0; t < R; t++) v[t] = (uint64_t)(threadIdx.x * 2654435761u + t) * 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int t = 0; t < R / 2; t++) w[t] = 0x123456789ull * (t + 3 + blockIdx.x);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
            for (int t = 0; t < R; t++) {
                if (t & h) continue;
                f.dif(v[t], v[t + h], w[(t & (h - 1)) % (R / 2)]);
            }
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int t = 0; t < R; t++) acc ^= v[t];
    if (acc == 0x12345678ull) sink[0] = acc;
}

// gold.cuh's 8-point Goldilocks DIF (shift twiddles, 3-word delayed
// reduction) on register-resident values: the ALU ceiling of C4 / C5's tiles
// (12 butterflies per call; no memory traffic, no table products)
__global__ void __launch_bounds__(256) k_probe_gold8(int iters, uint64_t* sink) {
    uint64_t v[8];
#pragma unroll
    for (int t = 0; t < 8; t++) v[t] = (uint64_t)(threadIdx.x * 2654435761u + t + blockIdx.x) * 0x9E3779B97F4A7C15ull;
    for (int it = 0; it < iters; it++) gold::dif8<gold::S_FWD>(v);
    uint64_t acc = 0;
#pragma unroll
    for (int t = 0; t < 8; t++) acc ^= v[t];
    if (acc == 0x12345678ull) sink[0] = acc;
}

// Single-instruction issue probes: 8 independent dependency chains per
// thread of one SASS instruction class (inline PTX so ptxas keeps the form):
//   kind 0: mul.lo.u32 -> IMAD       kind 1: mul.hi.u32 -> IMAD.HI
//   kind 2: 3-input add -> IADD3     kind 3: min(a + b, c) -> VIADDMNMX
//   kind 4: IMAD.HI + 2 IADD3 interleaved (pipe overlap)
//   kind 5: fma.rn.f64 -> DFMA (the FP64 pipe of Functions 16 / 18)
template <int KIND>
__global__ void __launch_bounds__(256) k_probe_issue(uint32_t seed, int iters, uint32_t* sink) {
    uint32_t x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
    const uint32_t k = seed | 1u, c = seed ^ 0x5bd1e995u;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 8; r++) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if (KIND == 0) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
                if (KIND == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
                if (KIND == 2) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(k), "r"(c));
                if (KIND == 3) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; min.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(k), "r"(c));
                if (KIND == 4) {
                    asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
                    asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(k), "r"(c));
                    asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(c), "r"(k));
                }
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) acc ^= x[i];
    if (acc == 0x12345678u) sink[0] = acc;
}
__global__ void __launch_bounds__(256) k_probe_dfma(double seed, int iters, double* sink) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = seed * (threadIdx.x + 1) + i;
    const double k = 0.999999, c = 1e-9;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 8; r++)
#pragma unroll
            for (int i = 0; i < 8; i++) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(k), "d"(c));
    }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) acc += x[i];
    if (acc == 1234.5) sink[0] = acc;
}

}  // namespace mm

using namespace mm;

// Runs instruction probe `kind` once; *ms = kernel time, *ops = warp
// instructions of the probed class executed (per SM per clock = ops /
// (ms 1e-3 x SMs x clock)).
extern "C" mm_status mm_probe_issue(int kind, int iters, double* ms, double* ops, void* stream) {
    if (!ms || !ops || iters <= 0 || kind < 0 || kind > 5) return set_err(MM_E_ARG, "bad probe arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int blocks = num_sms() * 8, threads = 256;
    void* sink = nullptr;
    MM_CUDA_TRY(cudaMalloc(&sink, 16));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    {
        LaunchScope ls("probe_issue", st);
        switch (kind) {
            case 0: k_probe_issue<0><<<blocks, threads, 0, st>>>(12345u, iters, (uint32_t*)sink); break;
            case 1: k_probe_issue<1><<<blocks, threads, 0, st>>>(12345u, iters, (uint32_t*)sink); break;
            case 2: k_probe_issue<2><<<blocks, threads, 0, st>>>(12345u, iters, (uint32_t*)sink); break;
            case 3: k_probe_issue<3><<<blocks, threads, 0, st>>>(12345u, iters, (uint32_t*)sink); break;
            case 4: k_probe_issue<4><<<blocks, threads, 0, st>>>(12345u, iters, (uint32_t*)sink); break;
            default: k_probe_dfma<<<blocks, threads, 0, st>>>(1.5, iters, (double*)sink); break;
        }
    }
    cudaEventRecord(b, st);
    cudaError_t e = cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return set_err(MM_E_CUDA, "probe failed: %s", cudaGetErrorString(e));
    *ms = t;
    *ops = (double)blocks * (threads / 32) * iters * 64.0 * (kind == 4 ? 3.0 : 1.0);
    return MM_OK;
}

// Runs the probe once on `stream` and returns the kernel time in ms through
// *ms (events on the launching stream) and the butterfly count through *bfly.
extern "C" mm_status mm_probe_butterfly(int word_bits, int iters, double* ms, double* bfly, void* stream) {
    if (!ms || !bfly || iters <= 0) return set_err(MM_E_ARG, "bad probe arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int blocks = num_sms() * 8, threads = 256;
    void* sink = nullptr;
    MM_CUDA_TRY(cudaMalloc(&sink, 16));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double per_iter;
    cudaEventRecord(a, st);
    {
        LaunchScope ls("probe_butterfly", st);
        if (word_bits == 32) {
            Fp32 f;
            f.p = 998244353u;
            f.p2 = 2 * f.p;
            f.pinv = inv_mod_2_32(f.p);
            k_probe_bfly32<16><<<blocks, threads, 0, st>>>(f, make_uint2(12345u, 67890u), iters, (uint32_t*)sink);
            per_iter = 32.0;
        } else if (word_bits == 65) {      // Goldilocks 8-point split (gold.cuh)
            k_probe_gold8<<<blocks, threads, 0, st>>>(iters, (uint64_t*)sink);
            per_iter = 12.0;
        } else {
            k_probe_bfly64<8><<<blocks, threads, 0, st>>>(iters, (uint64_t*)sink);
            per_iter = 12.0;
        }
    }
    cudaEventRecord(b, st);
    cudaError_t e = cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return set_err(MM_E_CUDA, "probe failed: %s", cudaGetErrorString(e));
    *ms = t;
    *bfly = (double)blocks * threads * iters * per_iter;
    return MM_OK;
}
