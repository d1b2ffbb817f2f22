// thmm_launch.cuh -- host-side launch/attribute wrappers of the kernel templates.
//
// The C-ABI (thmm_capi.cu) sees only these declarations; the definitions are
// compiled once per padded-state-count in thmm_inst_<NT>.cu (explicit
// instantiations), so the ~80 kernel variants build in parallel.
#pragma once

#include <cuda_runtime.h>

#include "thmm_kernels.cuh"
#include "thmm_runs.cuh"
#include "thmm_vec.cuh"

namespace thmm {

// FP64 chain kernel <head tiles, skip last half k-chunk, tail states>.
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_f64_attributes(cudaFuncAttributes* attr);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_f64_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_f64_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s);

// FP32 chain kernel <padded tiles>.
template <int NT>
cudaError_t chain_f32_attributes(cudaFuncAttributes* attr);
template <int NT>
cudaError_t chain_f32_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm);
template <int NT>
cudaError_t chain_f32_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s);

// TF32 tensor-core chain kernel <UMMA N, contraction length, column slices> (thmm_tc.cuh).
template <int NP, int KP, int H>
cudaError_t chain_tc_attributes(cudaFuncAttributes* attr);
template <int NP, int KP, int H>
cudaError_t chain_tc_setup(int max_dynamic_smem);
template <int NP, int KP, int H>
cudaError_t chain_tc_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s);

// Fold kernel <padded tiles, skip>.
template <int NT, bool SKIP>
cudaError_t fold_setup(int smem);
template <int NT, bool SKIP>
cudaError_t fold_launch(const FoldArgs& a, dim3 grid, size_t smem, cudaStream_t s);

// One-launch segment tree <padded tiles, skip>.
template <int NT, bool SKIP>
cudaError_t tree_setup(int smem);
template <int NT, bool SKIP>
cudaError_t tree_launch(const TreeArgs& a, dim3 grid, size_t smem, cudaStream_t s);

// Run-absorbing FP64 chain kernel <head tiles, skip, tail states> (thmm_runs.cuh).
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_runs_attributes(cudaFuncAttributes* attr);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_runs_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_runs_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s);

// Row-stacked vector continuation of collapsed segments <head tiles, skip, tail> (thmm_vec.cuh).
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_vec_attributes(cudaFuncAttributes* attr);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_vec_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_vec_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s);

// Stitched chain: main pass, link pass, per-proposal finish.
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_fwd_setup(int max_dynamic_smem);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_fwd_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_link_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s);
template <int NT, bool SKIP, int TAIL>
cudaError_t stitch_finish_launch(const ChainArgs& a, double* loglik, int32_t* status, double* block, cudaStream_t s);
template <int NT, bool SKIP, int TAIL>
cudaError_t entry_prep_launch(const ChainArgs& a, double2* gent, cudaStream_t s);

#ifdef THMM_DEFINE_LAUNCHERS

template <int NT, bool SKIP, int TAIL>
cudaError_t chain_fwd_setup(int max_dynamic_smem) {
  cudaError_t e = cudaFuncSetAttribute(chain_fwd_kernel<NT, SKIP, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       max_dynamic_smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(chain_link_kernel<NT, SKIP, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              max_dynamic_smem);
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_fwd_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_fwd_kernel<NT, SKIP, TAIL><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_link_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_link_kernel<NT, SKIP, TAIL><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}
template <int NT, bool SKIP, int TAIL>
cudaError_t stitch_finish_launch(const ChainArgs& a, double* loglik, int32_t* status, double* block, cudaStream_t s) {
  stitch_finish_kernel<8 * (NT + (TAIL > 0 ? 1 : 0))><<<a.B, 256, 0, s>>>(a, loglik, status, block);
  return cudaGetLastError();
}
template <int NT, bool SKIP, int TAIL>
cudaError_t entry_prep_launch(const ChainArgs& a, double2* gent, cudaStream_t s) {
  entry_prep_kernel<NT, TAIL><<<a.B, 256, 0, s>>>(a, gent);
  return cudaGetLastError();
}

template <int NT, bool SKIP, int TAIL>
cudaError_t chain_vec_attributes(cudaFuncAttributes* attr) {
  return cudaFuncGetAttributes(attr, chain_vec_kernel<NT, SKIP, TAIL>);
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_vec_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(chain_vec_kernel<NT, SKIP, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       max_dynamic_smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, chain_vec_kernel<NT, SKIP, TAIL>, threads, smem);
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_vec_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_vec_kernel<NT, SKIP, TAIL><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NT, bool SKIP, int TAIL>
cudaError_t chain_runs_attributes(cudaFuncAttributes* attr) {
  return cudaFuncGetAttributes(attr, chain_runs_kernel<NT, SKIP, TAIL>);
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_runs_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(chain_runs_kernel<NT, SKIP, TAIL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, max_dynamic_smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, chain_runs_kernel<NT, SKIP, TAIL>, threads,
                                                       smem);
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_runs_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_runs_kernel<NT, SKIP, TAIL><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}
#define THMM_INSTANTIATE_RUNS(NT, SKIP, TAIL)                                                        \
  template cudaError_t chain_runs_attributes<NT, SKIP, TAIL>(cudaFuncAttributes*);                  \
  template cudaError_t chain_runs_setup<NT, SKIP, TAIL>(int, int, size_t, int*);                    \
  template cudaError_t chain_runs_launch<NT, SKIP, TAIL>(const ChainArgs&, dim3, int, size_t, cudaStream_t); \
  template cudaError_t chain_vec_attributes<NT, SKIP, TAIL>(cudaFuncAttributes*);                   \
  template cudaError_t chain_vec_setup<NT, SKIP, TAIL>(int, int, size_t, int*);                     \
  template cudaError_t chain_vec_launch<NT, SKIP, TAIL>(const ChainArgs&, dim3, int, size_t, cudaStream_t); \
  template cudaError_t chain_fwd_setup<NT, SKIP, TAIL>(int);                                        \
  template cudaError_t chain_fwd_launch<NT, SKIP, TAIL>(const ChainArgs&, dim3, int, size_t, cudaStream_t); \
  template cudaError_t chain_link_launch<NT, SKIP, TAIL>(const ChainArgs&, dim3, int, size_t, cudaStream_t); \
  template cudaError_t stitch_finish_launch<NT, SKIP, TAIL>(const ChainArgs&, double*, int32_t*, double*, cudaStream_t); \
  template cudaError_t entry_prep_launch<NT, SKIP, TAIL>(const ChainArgs&, double2*, cudaStream_t);
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_f64_attributes(cudaFuncAttributes* attr) {
  return cudaFuncGetAttributes(attr, chain_f64_kernel<NT, SKIP, TAIL>);
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_f64_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(chain_f64_kernel<NT, SKIP, TAIL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, max_dynamic_smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, chain_f64_kernel<NT, SKIP, TAIL>, threads, smem);
}
template <int NT, bool SKIP, int TAIL>
cudaError_t chain_f64_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_f64_kernel<NT, SKIP, TAIL><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NT>
cudaError_t chain_f32_attributes(cudaFuncAttributes* attr) {
  return cudaFuncGetAttributes(attr, chain_f32_kernel<NT>);
}
template <int NT>
cudaError_t chain_f32_setup(int max_dynamic_smem, int threads, size_t smem, int* ctas_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(chain_f32_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       max_dynamic_smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, chain_f32_kernel<NT>, threads, smem);
}
template <int NT>
cudaError_t chain_f32_launch(const ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  chain_f32_kernel<NT><<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NT, bool SKIP>
cudaError_t fold_setup(int smem) {
  return cudaFuncSetAttribute(fold_kernel<NT, SKIP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}
template <int NT, bool SKIP>
cudaError_t fold_launch(const FoldArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
  fold_kernel<NT, SKIP><<<grid, NT * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NT, bool SKIP>
cudaError_t tree_setup(int smem) {
  return cudaFuncSetAttribute(tree_fold_kernel<NT, SKIP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}
template <int NT, bool SKIP>
cudaError_t tree_launch(const TreeArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
  tree_fold_kernel<NT, SKIP><<<grid, tree_groups(NT) * NT * 32, smem, s>>>(a);
  return cudaGetLastError();
}

#define THMM_INSTANTIATE_CHAIN64(NT, SKIP, TAIL)                                                      \
  template cudaError_t chain_f64_attributes<NT, SKIP, TAIL>(cudaFuncAttributes*);                    \
  template cudaError_t chain_f64_setup<NT, SKIP, TAIL>(int, int, size_t, int*);                      \
  template cudaError_t chain_f64_launch<NT, SKIP, TAIL>(const ChainArgs&, dim3, int, size_t, cudaStream_t);

#define THMM_INSTANTIATE_NT(NT)                                                                       \
  THMM_INSTANTIATE_CHAIN64(NT, false, 0)                                                              \
  THMM_INSTANTIATE_CHAIN64(NT, true, 0)                                                               \
  template cudaError_t chain_f32_attributes<NT>(cudaFuncAttributes*);                                \
  template cudaError_t chain_f32_setup<NT>(int, int, size_t, int*);                                  \
  template cudaError_t chain_f32_launch<NT>(const ChainArgs&, dim3, int, size_t, cudaStream_t);      \
  template cudaError_t fold_setup<NT, false>(int);                                                   \
  template cudaError_t fold_setup<NT, true>(int);                                                    \
  template cudaError_t fold_launch<NT, false>(const FoldArgs&, dim3, size_t, cudaStream_t);          \
  template cudaError_t fold_launch<NT, true>(const FoldArgs&, dim3, size_t, cudaStream_t);          \
  template cudaError_t tree_setup<NT, false>(int);                                                   \
  template cudaError_t tree_setup<NT, true>(int);                                                    \
  template cudaError_t tree_launch<NT, false>(const TreeArgs&, dim3, size_t, cudaStream_t);          \
  template cudaError_t tree_launch<NT, true>(const TreeArgs&, dim3, size_t, cudaStream_t);

// Head/tail variants exist for NT head tiles 1..9 and tails 1..4.
#define THMM_INSTANTIATE_TAILS(NT)      \
  THMM_INSTANTIATE_CHAIN64(NT, false, 1) \
  THMM_INSTANTIATE_CHAIN64(NT, false, 2) \
  THMM_INSTANTIATE_CHAIN64(NT, false, 3) \
  THMM_INSTANTIATE_CHAIN64(NT, false, 4)

#endif  // THMM_DEFINE_LAUNCHERS

}  // namespace thmm
