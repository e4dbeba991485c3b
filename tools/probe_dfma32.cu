// probe_dfma32.cu -- standalone measurement tool (not part of the library):
// the 32-bit lazy butterfly with the quotient of x w / p taken on the FP64
// pipe (one DFMA rounding toward -inf, the floating-point quotient of the
// paper's section 3) instead of IMAD.HI (Function 8's umulhi), register
// resident.  Each variant is first checked against u64 % on the device.
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/probe_dfma32 tools/probe_dfma32.cu
//   tools/bin/probe_dfma32       (prints one JSON object)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <math.h>
#include <stdlib.h>

struct Fld { uint32_t p, p2; };
struct TwS { uint32_t w, ws; };                 // Shoup: w, floor(w 2^32 / p)
struct TwD { double c, k; uint32_t w, pad; };   // c = RD(w / p), k = RD(2^52 - 2^52 c)

__device__ __forceinline__ uint32_t umn(uint32_t a, uint32_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t add_sub(uint32_t x, uint32_t y, uint32_t c) {
    uint32_t t;
    asm("{ .reg .u32 r; add.u32 r, %1, %2; sub.u32 %0, r, %3; }" : "=r"(t) : "r"(x), "r"(y), "r"(c));
    return t;
}
__device__ __forceinline__ uint32_t mulw_s(uint32_t x, TwS w, uint32_t p) {
    uint32_t c = __umulhi(x, w.ws);
    return x * w.w - c * p;
}
// q = floor(x c + tau) in {floor(x w / p) - 1, floor(x w / p)}: X = 2^52 + x as a
// bit pattern, V = RD(X c + k) = 2^52 + q; x w - q p in [0, 2p) mod 2^32.
__device__ __forceinline__ uint32_t mulw_d(uint32_t x, const TwD& w, uint32_t p) {
    double X = __hiloint2double(0x43300000, (int)x);
    double V = __fma_rd(X, w.c, w.k);
    uint32_t q = (uint32_t)__double2loint(V);
    return x * w.w - q * p;
}
template <int MODE> struct Bf;
template <> struct Bf<0> {
    typedef TwS W;
    __device__ static __forceinline__ uint32_t mul(uint32_t x, const W& w, uint32_t p) { return mulw_s(x, w, p); }
};
template <> struct Bf<2> {
    typedef TwD W;
    __device__ static __forceinline__ uint32_t mul(uint32_t x, const W& w, uint32_t p) { return mulw_d(x, w, p); }
};
template <> struct Bf<1> {
    typedef TwD W;
    __device__ static __forceinline__ uint32_t mul(uint32_t x, const W& w, uint32_t p) { return mulw_d(x, w, p); }
};

// d = x - y + 2p written into the low word of a pair whose high word already
// holds 0x43300000 (so X = 2^52 + d needs no per-butterfly move)
__device__ __forceinline__ uint32_t mulw_pair(uint64_t& S, uint32_t x, uint32_t y, const TwD& w, const Fld& f) {
    asm("{ .reg .u32 lo, hi, r; mov.b64 {lo, hi}, %0; add.u32 r, %1, %3; sub.u32 lo, r, %2; mov.b64 %0, {lo, hi}; }"
        : "+l"(S) : "r"(x), "r"(y), "r"(f.p2));
    double V = __fma_rd(__longlong_as_double((long long)S), w.c, w.k);
    uint32_t q = (uint32_t)__double2loint(V);
    return (uint32_t)S * w.w - q * f.p;
}
template <int MODE>
__device__ __forceinline__ void dif(uint32_t& x, uint32_t& y, const typename Bf<MODE>::W& w, const Fld& f) {
    uint32_t t = add_sub(x, y, f.p2);
    uint32_t d = add_sub(x, f.p2, y);
    x = umn(x + y, t);
    y = Bf<MODE>::mul(d, w, f.p);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_check(const typename Bf<MODE>::W* tw, const uint32_t* xs, uint32_t* out, int n, int ntw, Fld f) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = Bf<MODE>::mul(xs[i], tw[i % ntw], f.p);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_bfly(const typename Bf<MODE>::W* tw, Fld f, int iters, uint32_t* sink) {
    typedef typename Bf<MODE>::W W;
    uint32_t v[16];
    W w[8];
#pragma unroll
    for (int t = 0; t < 16; t++) v[t] = (threadIdx.x * 2654435761u + t * 40503u + blockIdx.x) % f.p;
#pragma unroll
    for (int t = 0; t < 8; t++) w[t] = tw[(t + threadIdx.x) & 63];
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
            for (int t = 0; t < 16; t++) {
                if (t & h) continue;
                dif<MODE>(v[t], v[t + h], w[(t & (h - 1)) % 8], f);
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int t = 0; t < 16; t++) acc ^= v[t];
    if (acc == 0x12345678u) sink[0] = acc;
}
__global__ void __launch_bounds__(256) k_bfly_pair(const TwD* tw, Fld f, int iters, uint32_t* sink) {
    uint32_t v[16];
    TwD w[8];
    uint64_t S[8];
#pragma unroll
    for (int t = 0; t < 16; t++) v[t] = (threadIdx.x * 2654435761u + t * 40503u + blockIdx.x) % f.p;
#pragma unroll
    for (int t = 0; t < 8; t++) { w[t] = tw[(t + threadIdx.x) & 63]; S[t] = 0x4330000000000000ull; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1) {
            int k = 0;
#pragma unroll
            for (int t = 0; t < 16; t++) {
                if (t & h) continue;
                uint32_t x = v[t], y = v[t + h];
                uint32_t tt = add_sub(x, y, f.p2);
                v[t + h] = mulw_pair(S[k++], x, y, w[(t & (h - 1)) % 8], f);
                v[t] = umn(x + y, tt);
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int t = 0; t < 16; t++) acc ^= v[t];
    if (acc == 0x12345678u) sink[0] = acc;
}

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static uint64_t nxt() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; }

// exact host constants: c = RD(w / p) (53-bit), k = RD(2^52 - 2^52 c)
static TwD make_d(uint32_t w, uint32_t p) {
    TwD t;
    double c = (double)w / (double)p;               // round to nearest
    if (fma(c, (double)p, -(double)w) > 0) c = nextafter(c, 0.0);   // sign of c p - w is exact
    t.c = c;
    double k = 4503599627370496.0 - 4503599627370496.0 * c;          // 2^52 c exact; difference rounded
    // make k <= 2^52 - 2^52 c exactly: compare with fma
    if (k + 4503599627370496.0 * c > 4503599627370496.0) k = nextafter(k, 0.0);
    t.k = k;
    t.w = w;
    t.pad = 0;
    return t;
}

int main() {
    const uint32_t p = 998244353u;
    Fld f{p, 2 * p};
    const int NTW = 64, N = 1 << 22;
    TwS hs[NTW];
    TwD hd[NTW];
    for (int i = 0; i < NTW; i++) {
        uint32_t w = i < 4 ? (uint32_t[]){1u, p - 1, 2u, p / 2}[i] : (uint32_t)(nxt() % p);
        hs[i] = TwS{w, (uint32_t)(((uint64_t)w << 32) / p)};
        hd[i] = make_d(w, p);
    }
    uint32_t* hx = (uint32_t*)malloc(N * 4);
    for (int i = 0; i < N; i++) {
        uint64_t r = nxt();
        hx[i] = i < 64 ? (uint32_t)(i < 32 ? i : 0xFFFFFFFFu - (i - 32)) : (uint32_t)r;   // full 32-bit range
    }
    TwS* ds; TwD* dd; uint32_t *dx, *dout, *sink;
    cudaMalloc(&ds, sizeof(hs)); cudaMalloc(&dd, sizeof(hd));
    cudaMalloc(&dx, N * 4); cudaMalloc(&dout, N * 4); cudaMalloc(&sink, 16);
    cudaMemcpy(ds, hs, sizeof(hs), cudaMemcpyHostToDevice);
    cudaMemcpy(dd, hd, sizeof(hd), cudaMemcpyHostToDevice);
    cudaMemcpy(dx, hx, N * 4, cudaMemcpyHostToDevice);
    uint32_t* ho = (uint32_t*)malloc(N * 4);
    int bad[2] = {0, 0};
    for (int mode = 0; mode < 2; mode++) {
        if (mode == 0) k_check<0><<<N / 256, 256>>>(ds, dx, dout, N, NTW, f);
        else k_check<1><<<N / 256, 256>>>(dd, dx, dout, N, NTW, f);
        cudaMemcpy(ho, dout, N * 4, cudaMemcpyDeviceToHost);
        for (int i = 0; i < N; i++) {
            uint32_t w = hs[i % NTW].w;
            uint64_t want = (uint64_t)hx[i] * w % p;
            if (ho[i] >= 2 * p || ho[i] % p != want) bad[mode]++;
        }
    }
    int dev;
    cudaGetDevice(&dev);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8, iters = 4000;
    double rate[3];
    for (int mode = 0; mode < 3; mode++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        float best = 1e30f;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(a);
            if (mode == 0) k_bfly<0><<<blocks, 256>>>(ds, f, iters, sink);
            else if (mode == 1) k_bfly<1><<<blocks, 256>>>(dd, f, iters, sink);
            else k_bfly_pair<<<blocks, 256>>>(dd, f, iters, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        rate[mode] = (double)blocks * 256 * iters * 32.0 / (best * 1e-3) / 1e9;
    }
    printf("{\"check_bad\": [%d, %d], \"shoup_Gbfly_s\": %.1f, \"dfma_Gbfly_s\": %.1f, \"pair_Gbfly_s\": %.1f, \"ratio\": %.3f, \"sms\": %d, \"clk_mhz\": %d, \"err\": \"%s\"}\n",
           bad[0], bad[1], rate[0], rate[1], rate[2], rate[2] / rate[0], sms, clk / 1000, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
