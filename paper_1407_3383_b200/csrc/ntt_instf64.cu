// Explicit instantiations of the FP64 (word_bits 52, paper §3) launchers.
#include "ntt_kernels.cuh"
namespace mm {
template mm_status launch_rows<FpD, false, double, double>(const FpD&, const RowArgs<FpD>&, cudaStream_t);
template mm_status launch_rows<FpD, true, double, double>(const FpD&, const RowArgs<FpD>&, cudaStream_t);
template mm_status launch_cols<FpD, false, double, double>(const FpD&, const ColArgs<FpD>&, cudaStream_t);
template mm_status launch_cols<FpD, true, double, double>(const FpD&, const ColArgs<FpD>&, cudaStream_t);
template mm_status launch_pmul<FpD, double, double>(const FpD&, const PmulArgs<FpD>&, cudaStream_t);
}  // namespace mm
