// Explicit instantiations of the Goldilocks row-pass launchers.
#include "ntt_kernels.cuh"
namespace mm {
template mm_status launch_rows<FpG, false, uint64_t, uint64_t>(const FpG&, const RowArgs<FpG>&, cudaStream_t);
template mm_status launch_rows<FpG, true, uint64_t, uint64_t>(const FpG&, const RowArgs<FpG>&, cudaStream_t);
}  // namespace mm
