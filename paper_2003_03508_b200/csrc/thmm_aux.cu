// thmm_aux.cu -- batched per-proposal work around the likelihood:
// stationary distributions of B transition matrices in one launch.
//
// Reference core.stationary_distribution (core.py:350-388): power iteration
// pi <- pi Gamma / sum from the uniform vector until the max-norm change is
// below 1e-12, at most 1e5 sweeps (RuntimeError otherwise).  In the MCMC
// driver this runs once per proposal when delta is tied to Gamma
// (bayes.py:305-311); here one CTA iterates one proposal's chain.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "thmm.h"

namespace {

constexpr int kThreads = 128;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One CTA per proposal; thread c owns column c (K <= 80 <= kThreads).
__global__ void __launch_bounds__(kThreads) stationary_kernel(const double* __restrict__ gammas, int K,
                                                              double tol, int max_iter, double* __restrict__ out,
                                                              int32_t* __restrict__ status) {
  extern __shared__ double sm[];
  double* g = sm;              // K*K
  double* pi = g + K * K;      // K
  double* red = pi + K;        // 2 * (kThreads/32)
  const int b = blockIdx.x, c = threadIdx.x, lane = c & 31, warp = c >> 5;
  constexpr int NW = kThreads / 32;
  const double* src = gammas + static_cast<size_t>(b) * K * K;
  for (int i = c; i < K * K; i += kThreads) g[i] = src[i];
  if (c < K) pi[c] = 1.0 / K;
  __syncthreads();
  bool converged = false;
  for (int it = 0; it < max_iter; ++it) {
    double nxt = 0.0;
    if (c < K)
      for (int r = 0; r < K; ++r) nxt = fma(pi[r], g[r * K + c], nxt);
    double s = warp_sum(c < K ? nxt : 0.0);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double total = 0.0;
    for (int w = 0; w < NW; ++w) total += red[w];
    nxt /= total;
    double d = warp_max(c < K ? fabs(nxt - pi[c]) : 0.0);
    __syncthreads();  // everyone has read red[] and pi[]
    if (lane == 0) red[NW + warp] = d;
    if (c < K) pi[c] = nxt;
    __syncthreads();
    double diff = 0.0;
    for (int w = 0; w < NW; ++w) diff = fmax(diff, red[NW + w]);
    if (diff < tol) {
      converged = true;
      break;
    }
  }
  if (c < K) out[static_cast<size_t>(b) * K + c] = pi[c];
  if (c == 0) status[b] = converged ? THMM_OK : THMM_ECOLLAPSE;
}

void aux_err(char* err, size_t errlen, const char* fmt, ...) {
  if (!err || errlen == 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

}  // namespace

extern "C" int thmm_stationary(const double* gammas, int32_t K, int32_t B, double tol, int32_t max_iter,
                               int device, double* out, int32_t* status, char* err, size_t errlen) {
  if (!gammas || !out || !status || K < 1 || K > THMM_MAX_STATES || B < 1 || max_iter < 1) {
    aux_err(err, errlen, "invalid arguments to thmm_stationary");
    return THMM_EINVAL;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    aux_err(err, errlen, "CUDA device %d not available", device);
    return THMM_ECUDA;
  }
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  const size_t gbytes = static_cast<size_t>(B) * K * K * sizeof(double);
  double *dg = nullptr, *dout = nullptr;
  int32_t* dst = nullptr;
  cudaError_t e = cudaMalloc(&dg, gbytes);
  if (e == cudaSuccess) e = cudaMalloc(&dout, static_cast<size_t>(B) * K * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&dst, static_cast<size_t>(B) * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemcpy(dg, gammas, gbytes, cudaMemcpyHostToDevice);
  const size_t smem = (static_cast<size_t>(K) * K + K + 2 * (kThreads / 32)) * sizeof(double);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(stationary_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) {
    stationary_kernel<<<B, kThreads, smem>>>(dg, K, tol, max_iter, dout, dst);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, static_cast<size_t>(B) * K * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(status, dst, static_cast<size_t>(B) * sizeof(int32_t), cudaMemcpyDeviceToHost);
  cudaFree(dg);
  cudaFree(dout);
  cudaFree(dst);
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess) {
    aux_err(err, errlen, "CUDA error %s in thmm_stationary", cudaGetErrorName(e));
    cudaGetLastError();
    return THMM_ECUDA;
  }
  for (int b = 0; b < B; ++b)
    if (status[b] != THMM_OK) {
      aux_err(err, errlen,
              "power iteration did not reach the stationary distribution within %d sweeps; the chain is too "
              "close to reducible or periodic",
              max_iter);
      return THMM_ECOLLAPSE;
    }
  return THMM_OK;
}
