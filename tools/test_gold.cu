// test_gold.cu -- device checks of gold.cuh's primitives against u128 %:
// mulpow<E> for every E in [0, 192), neg, dif8 / dit8 / dif4 / dit4 against
// the definition sum on random and extreme (2^64 - 1, p, p - 1, 0) inputs.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1407_3383_b200/csrc -o tools/bin/test_gold tools/test_gold.cu
#include <cstdio>
#include "gold.cuh"
using namespace mm;
typedef unsigned __int128 u128;
__device__ uint64_t rm(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) % gold::P); }
__device__ uint64_t rpow(uint64_t b, int e) { uint64_t r = 1; while (e) { if (e & 1) r = rm(r, b); b = rm(b, b); e >>= 1; } return r; }
__device__ uint64_t mix(uint64_t z) { z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }
__device__ uint64_t smp(uint64_t i) {
    const uint64_t e[6] = {0, 1, gold::P - 1, gold::P, ~0ull, gold::P + 5};
    uint64_t w = mix(i * 0x9E3779B97F4A7C15ull + 7);
    return (i % 7) < 6 && (i & 8) ? e[i % 6] : w;   // lazy inputs anywhere in [0, 2^64)
}
template <int E> __device__ void chk1(uint64_t x, unsigned* bad) {
    if (gold::mulpow<E>(x) % gold::P != rm(x % gold::P, rpow(2, E))) atomicAdd(bad, 1u);
}
template <int... Es> __device__ void chkall(uint64_t x, unsigned* bad, std::integer_sequence<int, Es...>) { (chk1<Es>(x, bad), ...); }
// naive DFT of R points with root 2^(S * 64 / R) (w_R = w_64^(64/R)); out in bit-reversed positions (fwd)
template <int R> __device__ void naive(const uint64_t* x, uint64_t* X, int S, bool bitrev_out, bool bitrev_in) {
    const uint64_t w = rpow(2, (S * (64 / R)) % 192);
    const int lg = R == 8 ? 3 : 2;
    for (int k = 0; k < R; k++) {
        u128 acc = 0;
        for (int j = 0; j < R; j++) {
            int jj = bitrev_in ? (int)(__brev(j) >> (32 - lg)) : j;
            acc = (acc + rm(x[jj] % gold::P, rpow(w, j * k))) % gold::P;
        }
        int pos = bitrev_out ? (int)(__brev(k) >> (32 - lg)) : k;
        X[pos] = (uint64_t)acc;
    }
}
__global__ void k(unsigned* bad, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint64_t x = smp(i);
        chkall(x, bad + 0, std::make_integer_sequence<int, 192>{});
        if (gold::neg(x) % gold::P != (gold::P - x % gold::P) % gold::P) atomicAdd(bad + 1, 1u);
        uint64_t v[8], e[8];
        for (int t = 0; t < 8; t++) v[t] = smp(8 * i + t + 12345);
        naive<8>(v, e, gold::S_FWD, true, false);
        gold::dif8<gold::S_FWD>(v);
        for (int t = 0; t < 8; t++) if (v[t] % gold::P != e[t]) atomicAdd(bad + 2, 1u);
        for (int t = 0; t < 8; t++) v[t] = smp(8 * i + t + 999);
        naive<8>(v, e, gold::S_INV, false, true);
        gold::dit8<gold::S_INV>(v);
        for (int t = 0; t < 8; t++) if (v[t] % gold::P != e[t]) atomicAdd(bad + 3, 1u);
        for (int t = 0; t < 4; t++) v[t] = smp(4 * i + t + 555);
        naive<4>(v, e, gold::S_FWD, true, false);
        gold::dif4<gold::S_FWD>(v);
        for (int t = 0; t < 4; t++) if (v[t] % gold::P != e[t]) atomicAdd(bad + 4, 1u);
        for (int t = 0; t < 4; t++) v[t] = smp(4 * i + t + 777);
        naive<4>(v, e, gold::S_INV, false, true);
        gold::dit4<gold::S_INV>(v);
        for (int t = 0; t < 4; t++) if (v[t] % gold::P != e[t]) atomicAdd(bad + 5, 1u);
    }
}
int main() {
    unsigned* bad;
    cudaMalloc(&bad, 8 * sizeof(unsigned));
    cudaMemset(bad, 0, 8 * sizeof(unsigned));
    k<<<148, 128>>>(bad, 1 << 16);
    unsigned h[8];
    cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    cudaError_t err = cudaDeviceSynchronize();
    printf("{\"mulpow\": %u, \"neg\": %u, \"dif8\": %u, \"dit8\": %u, \"dif4\": %u, \"dit4\": %u, \"cuda\": \"%s\"}\n", h[0], h[1], h[2],
           h[3], h[4], h[5], cudaGetErrorString(err));
    return (h[0] | h[1] | h[2] | h[3] | h[4] | h[5]) || err != cudaSuccess;
}
