// Launchers and explicit instantiations of the TF32 tensor-core chain kernel
// (thmm_tc.cuh) for UMMA N = 16..80, contraction KP in {N - 8, N}, 1 column
// slice per row (one translation unit per slice count: parallel build).
#include "thmm_launch.cuh"
#include "thmm_tc.cuh"

namespace thmm {

template <int NP, int KP, int H>
cudaError_t chain_tc_attributes(cudaFuncAttributes* attr) {
  return cudaFuncGetAttributes(attr, chain_tc_kernel<NP, KP, H>);
}
template <int NP, int KP, int H>
cudaError_t chain_tc_setup(int max_dynamic_smem) {
  return cudaFuncSetAttribute(chain_tc_kernel<NP, KP, H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              max_dynamic_smem);
}
template <int NP, int KP, int H>
cudaError_t chain_tc_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_tc_kernel<NP, KP, H><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

#define THMM_INSTANTIATE_TC(NP, KP, H)                                                              \
  template cudaError_t chain_tc_attributes<NP, KP, H>(cudaFuncAttributes*);                        \
  template cudaError_t chain_tc_setup<NP, KP, H>(int);                                             \
  template cudaError_t chain_tc_launch<NP, KP, H>(const ChainArgs&, dim3, int, size_t, cudaStream_t);

THMM_INSTANTIATE_TC(16, 8, 1)
THMM_INSTANTIATE_TC(16, 16, 1)
THMM_INSTANTIATE_TC(32, 24, 1)
THMM_INSTANTIATE_TC(32, 32, 1)
THMM_INSTANTIATE_TC(48, 40, 1)
THMM_INSTANTIATE_TC(48, 48, 1)
THMM_INSTANTIATE_TC(64, 56, 1)
THMM_INSTANTIATE_TC(64, 64, 1)
THMM_INSTANTIATE_TC(80, 72, 1)
THMM_INSTANTIATE_TC(80, 80, 1)

}  // namespace thmm
