// 2-D host->device copies with short rows (K=50 N=1e7 staged chunks: 14208 rows x 88-180 records).
//   nvcc -O3 -o tools/microbench/h2d_2d_small tools/microbench/h2d_2d_small.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
int main() {
  const size_t n = 10000000, S = 14208, L = n / S;
  double* h = static_cast<double*>(aligned_alloc(4096, n * 8));
  for (size_t i = 0; i < n; ++i) h[i] = i;
  cudaHostRegister(h, n * 8, cudaHostRegisterMapped | cudaHostRegisterPortable);
  double* d;
  cudaMalloc(&d, n * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t C : {1, 2, 4, 8, 16}) {
    const size_t w = L / C;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0, s);
      for (size_t c = 0; c < C; ++c) cudaMemcpy2DAsync(d + c * w, L * 8, h + c * w, L * 8, w * 8, S, cudaMemcpyDefault, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) printf("C=%2zu rows %zu x %5zu B: %.3f ms = %.1f GB/s\n", C, S, w * 8, ms, S * w * C * 8 / (ms * 1e6));
    }
  }
  return 0;
}
