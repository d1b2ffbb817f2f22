// Step anatomy of the stitched chain's main pass (chain_fwd_kernel,
// thmm_vec.cuh) in the latency regime: W warps per CTA, `ctas` CTAs (one per
// SM), synthetic records at a given present fraction; prints the mean cycles
// per record step in each phase of vec_run (THMM_VEC_TRACE stamps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTHMM_VEC_TRACE -I include \
//        -I paper_2003_03508_b200/csrc -o tools/vec_trace tools/vec_trace.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "thmm_vec.cuh"

template <int NT, bool SKIP, int TAIL>
void run(int K, int W, int ctas, int64_t len, double pfrac, bool batch = false) {
  using namespace thmm;
  const int64_t nseg = static_cast<int64_t>(ctas) * W * 8;
  const int64_t n = nseg * len;
  std::vector<uint8_t> pr(n);
  std::vector<double> lo(n), la(n);
  srand(1);
  for (int64_t i = 0; i < n; ++i) {
    pr[i] = rand() < pfrac * RAND_MAX;
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
  double *dlo, *dla, *dg, *ds, *dd, *dfin, *dfe;
  long long* dtr;
  const int KPE = 8 * (NT + (TAIL > 0));
  cudaMalloc(&dpr, n);
  cudaMalloc(&dlo, n * 8);
  cudaMalloc(&dla, n * 8);
  cudaMalloc(&dg, K * K * 8);
  cudaMalloc(&ds, 8 * K * 8);
  cudaMalloc(&dd, K * 8);
  cudaMalloc(&dfin, nseg * KPE * 8);
  cudaMalloc(&dfe, nseg * 8);
  cudaMalloc(&dtr, ctas * W * 8 * 8);
  cudaMemset(dtr, 0, ctas * W * 8 * 8);
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
  a.period = 8;
  a.neg_log_2pi = -std::log(2 * M_PI);
  a.P = StateParams{dg, ds, dd};
  a.fin = dfin;
  a.fin_e = dfe;
  a.node_stride_b = nseg;
  a.stitch_delta = 1;
  a.trace = dtr;
  a.ebatch = batch ? 1 : 0;
  const size_t smem = vec_smem_bytes(NT, TAIL, W, batch);
  cudaFuncSetAttribute(chain_fwd_kernel<NT, SKIP, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain_fwd_kernel<NT, SKIP, TAIL><<<dim3(ctas, 1), 32 * W, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  std::vector<long long> tr(ctas * W * 8);
  cudaMemcpy(tr.data(), dtr, tr.size() * 8, cudaMemcpyDeviceToHost);
  double ph[8] = {0};
  for (int w = 0; w < ctas * W; ++w)
    for (int k = 0; k < 8; ++k) ph[k] += tr[w * 8 + k];
  const double steps = (double)len * ctas * W;
  const char* names[6] = {"records", "dmma", "consts", "quiet", "present", "scale+renorm"};
  double tot = 0;
  for (int k = 0; k < 6; ++k) tot += ph[k];
  printf("K=%2d W=%2d %s ctas=%3d len=%lld p=%.2f: %.3f ms = %.3f us/step (%s); cycles/step %.0f:", K, W,
         batch ? "batch" : "step ", ctas, (long long)len, pfrac, ms, ms * 1e3 / len,
         cudaGetErrorString(cudaGetLastError()), tot / steps);
  for (int k = 0; k < 6; ++k) printf(" %s %.0f", names[k], ph[k] / steps);
  printf(" | present rows/step %.2f\n", ph[6] / steps);
}

int main(int argc, char** argv) {
  const int wide = argc > 1 ? atoi(argv[1]) : 12;
  for (int W : {1, 4}) {
    for (bool bt : {false, true}) {
      run<1, false, 0>(5, W, 148, 2048, 0.4, bt);
      run<3, false, 1>(25, W, 148, 2048, 0.13, bt);
      run<6, false, 2>(50, W, 148, 1024, 0.4, bt);
      if (W == 1) run<10, false, 0>(80, W, 148, 512, 0.44, bt);
    }
  }
  // full waves (throughput): the plan's warps per CTA
  run<3, false, 1>(25, 20, 148, 2048, 0.13);
  run<6, false, 2>(50, wide, 148, 2048, 0.4);
  run<10, false, 0>(80, wide, 148, 2048, 0.44);
  return 0;
}
