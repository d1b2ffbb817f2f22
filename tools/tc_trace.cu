// Step-latency anatomy of the TF32 tensor-core chain kernel (thmm_tc.cuh):
// launches chain_tc_kernel directly on synthetic data with the debug trace
// enabled and prints the mean per-step phase durations (clock64 cycles) of
// lane 0 of every warpgroup of CTA 0:
//   wait   mbarrier wait for the tile's MMAs
//   ld     tcgen05.ld of the accumulator row + wait
//   epi    emission scale / max / rescale
//   st     tf32 rounding + tcgen05.st of the next A
//   issue  wait::st + fence + warpgroup barrier + MMA issue + commit
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2003_03508_b200/csrc -o tools/tc_trace tools/tc_trace.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "thmm_tc.cuh"

template <int NP, int KP, int H>
void run(int K, int T, int x3, int64_t n_per_seg) {
  using namespace thmm;
  const int G = (kTcRows * T) / K;
  const int ctas = 148;
  const int64_t nseg = static_cast<int64_t>(ctas) * G;
  const int64_t n = nseg * n_per_seg;
  std::vector<uint8_t> pr(n);
  std::vector<double> lo(n), la(n);
  srand(1);
  for (int64_t i = 0; i < n; ++i) {
    pr[i] = rand() % 10 < 6;
    lo[i] = (rand() / (double)RAND_MAX) * 3 - 1.5;
    la[i] = (rand() / (double)RAND_MAX) * 3 - 1.5;
  }
  std::vector<double> gam(K * K), st(8 * K), del(K, 1.0 / K);
  for (int i = 0; i < K; ++i) {
    double s = 0;
    for (int j = 0; j < K; ++j) s += gam[i * K + j] = 0.5 + rand() / (double)RAND_MAX;
    for (int j = 0; j < K; ++j) gam[i * K + j] /= s;
  }
  for (int j = 0; j < K; ++j) {
    const double p = 0.5;
    st[0 * K + j] = p;
    st[1 * K + j] = 1 - p;
    st[2 * K + j] = (rand() / (double)RAND_MAX) * 2 - 1;
    st[3 * K + j] = (rand() / (double)RAND_MAX) * 2 - 1;
    st[4 * K + j] = 0.7;
    st[5 * K + j] = 0.1;
    st[6 * K + j] = 0.7;
    st[7 * K + j] = 2 * (std::log(0.7) + std::log(0.7));
  }
  uint8_t* dpr;
  double *dlo, *dla, *dg, *ds, *dd, *dm, *de;
  long long* dtr;
  cudaMalloc(&dpr, n);
  cudaMalloc(&dlo, n * 8);
  cudaMalloc(&dla, n * 8);
  cudaMalloc(&dg, K * K * 8);
  cudaMalloc(&ds, 8 * K * 8);
  cudaMalloc(&dd, K * 8);
  cudaMalloc(&dm, nseg * KP * KP * 8);
  cudaMalloc(&de, nseg * 8);
  cudaMalloc(&dtr, 8 * 256 * 6 * 8);
  cudaMemcpy(dpr, pr.data(), n, cudaMemcpyHostToDevice);
  cudaMemcpy(dlo, lo.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dla, la.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dg, gam.data(), K * K * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, st.data(), 8 * K * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, del.data(), K * 8, cudaMemcpyHostToDevice);
  ChainArgs a{};
  a.present = dpr;
  a.lon = dlo;
  a.lat = dla;
  a.lo = 0;
  a.n = n;
  a.nseg = nseg;
  a.K = K;
  a.B = 1;
  a.G = G;
  a.period = 8;
  a.neg_log_2pi = -std::log(2 * M_PI);
  a.P = StateParams{dg, ds, dd};
  a.seg_m = dm;
  a.seg_e = de;
  a.node_stride_b = nseg;
  a.node_offset = 0;
  a.x3 = x3;
  a.trace = dtr;
  const size_t smem = chain_tc_smem_bytes(NP, KP, G, T, H);
  cudaFuncSetAttribute(chain_tc_kernel<NP, KP, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain_tc_kernel<NP, KP, H><<<dim3(ctas, 1), 128 * H * T, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * K * K * K * (double)n / (ms * 1e-3) / 1e12;
    if (rep == 1)
      printf("K=%d NP=%d KP=%d H=%d T=%d G=%d x3=%d: %.3f ms, %.1f TFLOP/s alg (%s)\n", K, NP, KP, H, T, G, x3, ms, tf,
             cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<long long> tr(8 * 256 * 6);
  cudaMemcpy(tr.data(), dtr, tr.size() * 8, cudaMemcpyDeviceToHost);
  const char* names[5] = {"wait", "ld", "epi", "st", "issue"};
  for (int w = 0; w < T; ++w) {
    double acc[5] = {0}, tot = 0;
    int cnt = 0;
    for (int s = 20; s < 200; ++s) {
      const long long* t = &tr[(w * 256 + s) * 6];
      for (int k = 0; k < 5; ++k) acc[k] += t[k + 1] - t[k];
      tot += t[5] - t[0];
      ++cnt;
    }
    printf("  wg %d per step: total %7.1f |", w, tot / cnt);
    for (int k = 0; k < 5; ++k) printf(" %s %6.1f", names[k], acc[k] / cnt);
    printf("\n");
  }
  cudaFree(dpr);
  cudaFree(dlo);
  cudaFree(dla);
  cudaFree(dg);
  cudaFree(ds);
  cudaFree(dd);
  cudaFree(dm);
  cudaFree(de);
  cudaFree(dtr);
}

int main() {
  run<80, 80, 1>(80, 3, 0, 4000);
  run<80, 80, 2>(80, 3, 0, 4000);
  run<80, 80, 2>(80, 2, 0, 4000);
  run<80, 80, 1>(80, 2, 1, 4000);
  run<80, 80, 2>(80, 2, 1, 4000);
  run<64, 56, 2>(50, 4, 0, 4000);
  run<64, 56, 2>(50, 2, 1, 4000);
  run<32, 32, 1>(25, 6, 0, 4000);
  run<32, 32, 2>(25, 4, 0, 4000);
  run<32, 32, 1>(25, 5, 1, 4000);
  run<32, 32, 2>(25, 4, 1, 4000);
  return 0;
}
