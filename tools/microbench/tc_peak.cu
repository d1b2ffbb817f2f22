// tcgen05.mma kind::tf32 throughput at the chain kernel's shapes: one CTA per
// SM, one elected thread issues back-to-back M=128 x N x K=8 MMAs (A in TMEM,
// B in shared memory), committing every `chunk` MMAs.  Reports TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_peak tc_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N>
__global__ void __launch_bounds__(128, 1) tc_peak(int iters, int ntiles, float* out) {
  __shared__ __align__(16) uint32_t b[N * 8 * 10];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < N * 80; i += blockDim.x) b[i] = 0x3f800000u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = slot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t addr = smem_u32(b);
  uint64_t desc = (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
                  ((uint64_t)((80 / 4 * 128) >> 4) << 32) | (1ull << 46);
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      for (int t = 0; t < ntiles; ++t) {
        const uint32_t d = tb + t * N;   // D of tile t
        const uint32_t a = tb + 256;     // shared A region (values irrelevant)
        for (int kk = 0; kk < 10; ++kk)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                       "r"(a + 8 * kk), "l"(desc + 16 * kk), "r"(idesc), "r"(kk));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&bar)));
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase));
      phase ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1.f;
}

template <int N>
void run(int ntiles) {
  float* out;
  cudaMalloc(&out, 4);
  const int iters = 2000;
  tc_peak<N><<<148, 128>>>(10, ntiles, out);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  tc_peak<N><<<148, 128>>>(iters, ntiles, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 148.0 * iters * ntiles * 10 * 2.0 * 128 * N * 8;
  printf("tf32 M=128 N=%3d K=8 x10 per product, %d products per commit: %8.1f TFLOP/s (%s)\n", N, ntiles,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<80>(1);
  run<80>(2);
  run<80>(3);
  run<32>(3);
  run<64>(3);
  run<128>(2);
  return 0;
}
