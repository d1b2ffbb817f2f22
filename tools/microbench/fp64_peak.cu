// FP64 pipe microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Measures sustained flop/s with many independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma16_loop(double* out, int iters) {
  // m16n8k16: A 8 doubles, B 4 doubles, C 4 doubles per thread
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

// latency: single chain, one warp
__global__ void dmma_lat(double* out, long long* cyc, int iters) {
  double a = 1.0, b = 1.0, c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = c0 + c1; }
}

int main() {
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  long long* cyc; cudaMalloc(&cyc, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", p.name, sms, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  auto run = [&](const char* name, auto kern, int threads, int blocks_per_sm, double flop_per_thread_iter) {
    kern<<<sms * blocks_per_sm, threads>>>(out, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<sms * blocks_per_sm, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)sms * blocks_per_sm * threads * iters * flop_per_thread_iter;
    printf("%-28s threads %4d blk/sm %2d : %8.3f ms  %7.2f TFLOP/s  err=%s\n", name, threads, blocks_per_sm, ms,
           flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  // m8n8k4: 8*8*4*2 = 512 flop per warp per mma -> 16 flop per thread
  for (int w : {4, 8, 16}) {
    run("dmma m8n8k4 ch8", dmma_loop<8>, 32 * w, 1, 8 * 16.0);
    run("dmma m8n8k4 ch4", dmma_loop<4>, 32 * w, 1, 4 * 16.0);
    run("dmma m16n8k16 ch4", dmma16_loop<4>, 32 * w, 1, 4 * 16 * 8 * 16 * 2 / 32.0);
    run("dfma ch8", dfma_loop<8>, 32 * w, 1, 8 * 2.0);
  }
  run("dmma m8n8k4 ch8", dmma_loop<8>, 256, 2, 8 * 16.0);
  run("dmma m8n8k4 ch2", dmma_loop<2>, 256, 4, 2 * 16.0);
  run("dfma ch8", dfma_loop<8>, 256, 4, 8 * 2.0);
  dmma_lat<<<1, 32>>>(out, cyc, 1000); cudaDeviceSynchronize();
  dmma_lat<<<1, 32>>>(out, cyc, 10000); cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dmma m8n8k4 dependent latency: %.2f cycles\n", c / 10000.0);
  return 0;
}
