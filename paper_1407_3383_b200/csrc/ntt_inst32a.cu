// Explicit instantiations of the 32-bit row-pass launchers (see ntt_kernels.cuh).
#include "ntt_kernels.cuh"
namespace mm {
template mm_status launch_rows<Fp32, false, uint32_t, uint32_t>(const Fp32&, const RowArgs<Fp32>&, cudaStream_t);
template mm_status launch_rows<Fp32, true, uint32_t, uint32_t>(const Fp32&, const RowArgs<Fp32>&, cudaStream_t);
}  // namespace mm
