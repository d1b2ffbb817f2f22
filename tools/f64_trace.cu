// Block-phase anatomy of the FP64 DMMA chain kernel (thmm_kernels.cuh): runs
// chain_f64_kernel on synthetic data with the debug trace and prints, per
// warp of CTA 0, the mean cycles per 32-step emission block spent in its
// share of the emission fill, the 32 DMMA steps, and the block barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2003_03508_b200/csrc -o tools/f64_trace tools/f64_trace.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "thmm_kernels.cuh"

template <int NT, bool SKIP, int TAIL>
void run(int K, int G, int W, int ctas_per_sm, int64_t n_per_seg) {
  using namespace thmm;
  const int ctas = 148 * ctas_per_sm;
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
    st[0 * K + j] = 0.5;
    st[1 * K + j] = 0.5;
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
  const int KPE = 8 * (NT + (TAIL > 0));
  cudaMalloc(&dpr, n);
  cudaMalloc(&dlo, n * 8);
  cudaMalloc(&dla, n * 8);
  cudaMalloc(&dg, K * K * 8);
  cudaMalloc(&ds, 8 * K * 8);
  cudaMalloc(&dd, K * 8);
  cudaMalloc(&dm, nseg * KPE * KPE * 8);
  cudaMalloc(&de, nseg * 8);
  cudaMalloc(&dtr, 32 * 64 * 4 * 8);
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
  a.trace = dtr;
  const size_t smem = chain_smem_bytes(NT, TAIL, G, W);
  cudaFuncSetAttribute(chain_f64_kernel<NT, SKIP, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain_f64_kernel<NT, SKIP, TAIL><<<dim3(ctas, 1), 32 * W, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 1)
      printf("K=%d NT=%d TAIL=%d G=%d W=%d: %.3f ms, %.2f TFLOP/s alg (%s)\n", K, NT, TAIL, G, W, ms,
             2.0 * K * K * K * (double)n / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<long long> tr(32 * 64 * 4);
  cudaMemcpy(tr.data(), dtr, tr.size() * 8, cudaMemcpyDeviceToHost);
  double fill = 0, steps = 0, bar = 0, tot = 0;
  int cnt = 0;
  for (int w = 0; w < W; ++w)
    for (int b = 4; b < 60; ++b) {
      const long long* t = &tr[(w * 64 + b) * 4];
      fill += t[1] - t[0];
      steps += t[2] - t[1];
      bar += t[3] - t[2];
      tot += t[3] - t[0];
      ++cnt;
    }
  printf("  per 32-step block (mean over warps): total %.0f | fill %.0f (%.1f%%) | steps %.0f (%.1f%%) | barrier %.0f (%.1f%%)\n",
         tot / cnt, fill / cnt, 100 * fill / tot, steps / cnt, 100 * steps / tot, bar / cnt, 100 * bar / tot);
}

int main() {
  run<3, false, 1>(25, 5, 16, 2, 4000);
  run<6, false, 2>(50, 3, 20, 1, 4000);
  run<10, false, 0>(80, 2, 20, 1, 4000);
  return 0;
}
