// Explicit instantiations of the 32-bit column-pass and fused-product launchers.
#include "ntt_kernels.cuh"
namespace mm {
template mm_status launch_cols<Fp32, false, uint32_t, uint32_t>(const Fp32&, const ColArgs<Fp32>&, cudaStream_t);
template mm_status launch_cols<Fp32, true, uint32_t, uint32_t>(const Fp32&, const ColArgs<Fp32>&, cudaStream_t);
template mm_status launch_pmul<Fp32, uint32_t, uint32_t>(const Fp32&, const PmulArgs<Fp32>&, cudaStream_t);
}  // namespace mm
