// Explicit instantiations of the Goldilocks column-pass and fused-product launchers.
#include "ntt_kernels.cuh"
namespace mm {
template mm_status launch_cols<FpG, false, uint64_t, uint64_t>(const FpG&, const ColArgs<FpG>&, cudaStream_t);
template mm_status launch_cols<FpG, true, uint64_t, uint64_t>(const FpG&, const ColArgs<FpG>&, cudaStream_t);
template mm_status launch_cols<FpG, false, uint16_t, uint64_t>(const FpG&, const ColArgs<FpG>&, cudaStream_t);
template mm_status launch_pmul<FpG, uint64_t, uint64_t>(const FpG&, const PmulArgs<FpG>&, cudaStream_t);
template mm_status launch_pmul<FpG, uint16_t, uint64_t>(const FpG&, const PmulArgs<FpG>&, cudaStream_t);
}  // namespace mm
