// Host->device copy rate of the staged stitched path's 2-D slices (rows =
// segments, width = one time chunk of a segment) against one contiguous copy
// of the same bytes, from registered (page-locked in place) host memory.
//   nvcc -O3 -o tools/microbench/h2d_2d tools/microbench/h2d_2d.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

int main() {
  const size_t n = 100000000;  // records (lon array, 8 B each)
  double* h = static_cast<double*>(aligned_alloc(4096, n * 8));
  for (size_t i = 0; i < n; ++i) h[i] = static_cast<double>(i);
  cudaHostRegister(h, n * 8, cudaHostRegisterMapped | cudaHostRegisterPortable);
  double* d;
  cudaMalloc(&d, n * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](auto fn, size_t bytes, const char* what) {
    fn();
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 3; ++r) fn();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 3;
    printf("%-60s %8.3f ms  %6.1f GB/s (%s)\n", what, ms, bytes / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  };
  timed([&] { cudaMemcpyAsync(d, h, n * 8, cudaMemcpyDefault, s); }, n * 8, "1-D, 800 MB");
  const size_t segs[] = {14208, 5208, 14208};
  const size_t chunks[] = {8, 2, 16};
  for (int k = 0; k < 3; ++k) {
    const size_t S = segs[k], L = n / S, C = chunks[k], w = L / C;
    char what[128];
    snprintf(what, sizeof what, "2-D, %zu rows x %zu B (pitch %zu B), all %zu chunks", S, w * 8, L * 8, C);
    timed([&] {
      for (size_t c = 0; c < C; ++c)
        cudaMemcpy2DAsync(d + c * w, L * 8, h + c * w, L * 8, w * 8, S, cudaMemcpyDefault, s);
    }, S * w * C * 8, what);
    // misaligned rows (segment starts not 16-byte multiples)
    snprintf(what, sizeof what, "2-D misaligned (+1 record), %zu rows x %zu B", S, w * 8);
    timed([&] {
      for (size_t c = 0; c < C; ++c)
        cudaMemcpy2DAsync(d + 1 + c * w, L * 8, h + 1 + c * w, L * 8, (w - 1) * 8, S - 1, cudaMemcpyDefault, s);
    }, (S - 1) * (w - 1) * C * 8, what);
  }
  return 0;
}
