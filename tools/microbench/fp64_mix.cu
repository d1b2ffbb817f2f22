// Do DMMA (FP64 tensor) and DFMA (FP64 SIMT) share one pipe on sm_100a?
// Per loop iteration: NM mma.sync m8n8k4 f64 (3 independent accumulators) and
// NF independent DFMAs; time DMMA-only, DFMA-only and mixed loops.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF>
__global__ void mix(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i % 3][0]), "+d"(c[i % 3][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 3; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

// Interleaved: after every DMMA, NFI DFMAs (fine-grained mixing).
template <int NM, int NFI>
__global__ void mix_fine(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  double f[NM * NFI > 0 ? NM * NFI : 1];
#pragma unroll
  for (int i = 0; i < NM * NFI; ++i) f[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i % 3][0]), "+d"(c[i % 3][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int j = 0; j < NFI; ++j) asm volatile("fma.rn.f64 %0, %0, %1, %2;\n" : "+d"(f[i * NFI + j]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int i = 0; i < 3; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < NM * NFI; ++i) s += f[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NM, int NFI>
float run_fine(double* out, int warps) {
  const int iters = 20000;
  mix_fine<NM, NFI><<<148 * 2, 32 * warps>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix_fine<NM, NFI><<<148 * 2, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <int NM, int NF>
float run(double* out, int warps) {
  const int iters = 20000;
  mix<NM, NF><<<148 * 2, 32 * warps>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<NM, NF><<<148 * 2, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 16);
  for (int w : {8, 16}) {
    const float m = run<18, 0>(out, w), d = run<0, 16>(out, w), x = run<18, 16>(out, w);
    const float d8 = run<0, 8>(out, w), x8 = run<18, 8>(out, w);
    printf("warps/CTA %2d (2 CTA/SM): 18 DMMA %.3f ms | 16 DFMA %.3f ms | both %.3f ms (sum %.3f, max %.3f)\n", w, m, d,
           x, m + d, m > d ? m : d);
    printf("                          18 DMMA %.3f ms |  8 DFMA %.3f ms | both %.3f ms (sum %.3f)\n", m, d8, x8, m + d8);
  }
  for (int w : {8, 16}) {
    const float m = run<18, 0>(out, w), d = run<0, 18>(out, w), x = run_fine<18, 1>(out, w);
    printf("warps/CTA %2d: 18 DMMA %.3f ms | 18 DFMA %.3f ms | 18 x (DMMA, DFMA) interleaved %.3f ms (sum %.3f)\n", w,
           m, d, x, m + d);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
