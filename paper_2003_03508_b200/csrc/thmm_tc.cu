// Launchers and explicit instantiations of the TF32 tensor-core chain kernel
// (thmm_tc.cuh) for UMMA N = 16..80 and contraction KP in {N - 8, N}.
#include "thmm_launch.cuh"
#include "thmm_tc.cuh"

namespace thmm {

template <int NP, int KP>
cudaError_t chain_tc_attributes(cudaFuncAttributes* attr) {
  return cudaFuncGetAttributes(attr, chain_tc_kernel<NP, KP>);
}
template <int NP, int KP>
cudaError_t chain_tc_setup(int max_dynamic_smem) {
  return cudaFuncSetAttribute(chain_tc_kernel<NP, KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              max_dynamic_smem);
}
template <int NP, int KP>
cudaError_t chain_tc_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_tc_kernel<NP, KP><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

#define THMM_INSTANTIATE_TC(NP, KP)                                                                 \
  template cudaError_t chain_tc_attributes<NP, KP>(cudaFuncAttributes*);                           \
  template cudaError_t chain_tc_setup<NP, KP>(int);                                                \
  template cudaError_t chain_tc_launch<NP, KP>(const ChainArgs&, dim3, int, size_t, cudaStream_t);

THMM_INSTANTIATE_TC(16, 8)
THMM_INSTANTIATE_TC(16, 16)
THMM_INSTANTIATE_TC(32, 24)
THMM_INSTANTIATE_TC(32, 32)
THMM_INSTANTIATE_TC(48, 40)
THMM_INSTANTIATE_TC(48, 48)
THMM_INSTANTIATE_TC(64, 56)
THMM_INSTANTIATE_TC(64, 64)
THMM_INSTANTIATE_TC(80, 72)
THMM_INSTANTIATE_TC(80, 80)

}  // namespace thmm
