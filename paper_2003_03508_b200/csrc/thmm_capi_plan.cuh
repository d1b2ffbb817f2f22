// thmm_capi_plan.cuh -- chain launch geometry per (device, K, precision) and kernel dispatch.
//
// Implementation part of thmm_capi.cu (one translation unit: included there
// once, after the previous parts; not a standalone header).
#pragma once

namespace {

// Launch geometry of the chain kernel for one (K, precision) on one device.
//   FP64: NT DMMA head tiles + TAIL SIMT tail states (K%8 in 1..4, K >= 9),
//         else NT = ceil(K/8) padded tiles (SKIP when the last half k-chunk
//         is pure padding).  G segments stacked per CTA, W warps (multiple of
//         4, 8W >= G*K).
//   FP32: one thread per stacked row, W warps, G segments.
struct ChainPlan {
  bool ready = false;
  int nt = 1;
  bool skip = false;
  int tail = 0;
  int G = 1, W = 4;
  size_t smem = 0;
  int ctas_per_sm = 1;
  int sms = 148;
  int regs = 0;
  int slices = 1;  // tensor-core plan: column slices per row
};
std::mutex g_plan_mu;
ChainPlan g_plan[64][THMM_MAX_STATES + 1];
ChainPlan g_plan32[64][THMM_MAX_STATES + 1];
ChainPlan g_plan_tc[64][THMM_MAX_STATES + 1][3];
bool g_fold_ready[64][11][2];

bool skip_h1(int K) { return K % 8 == 1; }

// Dispatch fn<NT, SKIP>(...) on runtime (nt, skip).
#define THMM_DISPATCH(nt, skip, fn, ...)                               \
  switch (2 * (nt) + ((skip) ? 1 : 0)) {                               \
    case 2: fn<1, false>(__VA_ARGS__); break;                          \
    case 3: fn<1, true>(__VA_ARGS__); break;                           \
    case 4: fn<2, false>(__VA_ARGS__); break;                          \
    case 5: fn<2, true>(__VA_ARGS__); break;                           \
    case 6: fn<3, false>(__VA_ARGS__); break;                          \
    case 7: fn<3, true>(__VA_ARGS__); break;                           \
    case 8: fn<4, false>(__VA_ARGS__); break;                          \
    case 9: fn<4, true>(__VA_ARGS__); break;                           \
    case 10: fn<5, false>(__VA_ARGS__); break;                         \
    case 11: fn<5, true>(__VA_ARGS__); break;                          \
    case 12: fn<6, false>(__VA_ARGS__); break;                         \
    case 13: fn<6, true>(__VA_ARGS__); break;                          \
    case 14: fn<7, false>(__VA_ARGS__); break;                         \
    case 15: fn<7, true>(__VA_ARGS__); break;                          \
    case 16: fn<8, false>(__VA_ARGS__); break;                         \
    case 17: fn<8, true>(__VA_ARGS__); break;                          \
    case 18: fn<9, false>(__VA_ARGS__); break;                         \
    case 19: fn<9, true>(__VA_ARGS__); break;                          \
    case 20: fn<10, false>(__VA_ARGS__); break;                        \
    case 21: fn<10, true>(__VA_ARGS__); break;                         \
    default: throw CudaError{cudaErrorInvalidValue, "bad padded state count"}; \
  }

// The FP64 chain variants as a flat table indexed by (nt, skip, tail).
struct Chain64Ops {
  cudaError_t (*attributes)(cudaFuncAttributes*);
  cudaError_t (*setup)(int, int, size_t, int*);
  cudaError_t (*launch)(const thmm::ChainArgs&, dim3, int, size_t, cudaStream_t);
};

template <int NT, bool SKIP, int TAIL>
constexpr Chain64Ops ops64() {
  return {thmm::chain_f64_attributes<NT, SKIP, TAIL>, thmm::chain_f64_setup<NT, SKIP, TAIL>,
          thmm::chain_f64_launch<NT, SKIP, TAIL>};
}

#define THMM_OPS_NT(N) ops64<N, false, 0>(), ops64<N, true, 0>()
#define THMM_OPS_TAIL(N) ops64<N, false, 1>(), ops64<N, false, 2>(), ops64<N, false, 3>(), ops64<N, false, 4>()

// index: plain[nt-1][skip] ; tailed[nt-1][tail-1]
const Chain64Ops kPlain[10][2] = {{THMM_OPS_NT(1)}, {THMM_OPS_NT(2)}, {THMM_OPS_NT(3)}, {THMM_OPS_NT(4)},
                                  {THMM_OPS_NT(5)}, {THMM_OPS_NT(6)}, {THMM_OPS_NT(7)}, {THMM_OPS_NT(8)},
                                  {THMM_OPS_NT(9)}, {THMM_OPS_NT(10)}};
const Chain64Ops kTailed[9][4] = {{THMM_OPS_TAIL(1)}, {THMM_OPS_TAIL(2)}, {THMM_OPS_TAIL(3)},
                                  {THMM_OPS_TAIL(4)}, {THMM_OPS_TAIL(5)}, {THMM_OPS_TAIL(6)},
                                  {THMM_OPS_TAIL(7)}, {THMM_OPS_TAIL(8)}, {THMM_OPS_TAIL(9)}};

const Chain64Ops& ops_for(const ChainPlan& p) {
  return p.tail > 0 ? kTailed[p.nt - 1][p.tail - 1] : kPlain[p.nt - 1][p.skip ? 1 : 0];
}

void plan_chain64(int device, int K, ChainPlan& plan) {
  const int r = K % 8;
  if (K >= 9 && r >= 1 && r <= 4) {
    plan.nt = K / 8;
    plan.tail = r;
    plan.skip = false;
  } else {
    plan.nt = (K + 7) / 8;
    plan.tail = 0;
    plan.skip = skip_h1(K);
  }
  const Chain64Ops& ops = ops_for(plan);
  cudaFuncAttributes attr;
  THMM_CUDA(ops.attributes(&attr));
  cudaDeviceProp prop;
  THMM_CUDA(cudaGetDeviceProperties(&prop, device));
  const int regs = std::max(attr.numRegs, 1);
  // warps allowed by the register file (allocation granularity: 8 regs/thread)
  const int w_regs = static_cast<int>(prop.regsPerMultiprocessor / (32 * ((regs + 7) / 8 * 8)));
  const int w_max = std::min({32, attr.maxThreadsPerBlock / 32, w_regs});
  const size_t smem_cap = prop.sharedMemPerBlockOptin;
  int best_g = 1, best_w = 4;
  double best_waste = 2.0;
  for (int G = 1; G <= 8; ++G) {
    const int W = 4 * ((G * K + 31) / 32);
    if (W > w_max || thmm::chain_smem_bytes(plan.nt, plan.tail, G, W) > smem_cap) continue;
    const double waste = 1.0 - static_cast<double>(G * K) / (8.0 * W);
    if (waste < best_waste - 1e-9) {
      best_waste = waste;
      best_g = G;
      best_w = W;
    }
  }
  plan.G = best_g;
  plan.W = best_w;
  plan.smem = thmm::chain_smem_bytes(plan.nt, plan.tail, best_g, best_w);
  plan.regs = regs;
  int occ = 0;
  // Opt in to the full per-CTA shared memory; occupancy follows the actual launch size.
  THMM_CUDA(ops.setup(static_cast<int>(smem_cap), 32 * best_w, plan.smem, &occ));
  plan.ctas_per_sm = std::max(occ, 1);
  plan.sms = prop.multiProcessorCount;
  plan.ready = true;
}

const ChainPlan& chain_plan(int device, int K) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  ChainPlan& plan = g_plan[device & 63][K];
  if (!plan.ready) plan_chain64(device, K, plan);
  return plan;
}

// FP32 plan: one thread per stacked row; W warps (multiple of 4) and G
// segments chosen to use as many rows as the register file and shared
// memory allow while wasting at most ~10% of them.
template <int NT, bool SKIP>
void plan_chain32(int device, int K, ChainPlan& plan) {
  cudaFuncAttributes attr;
  THMM_CUDA(thmm::chain_f32_attributes<NT>(&attr));
  cudaDeviceProp prop;
  THMM_CUDA(cudaGetDeviceProperties(&prop, device));
  const int regs = std::max(attr.numRegs, 1);
  const int w_regs = static_cast<int>(prop.regsPerMultiprocessor / (32 * ((regs + 7) / 8 * 8)));
  const int w_max = std::min({32, attr.maxThreadsPerBlock / 32, w_regs});
  const size_t smem_cap = prop.sharedMemPerBlockOptin;
  int best_g = 1, best_w = std::max(1, (K + 31) / 32);
  int best_rows = -1;
  for (int W = 4; W <= w_max; W += 4) {
    const int G = std::min(64, (32 * W) / K);
    if (G < 1 || thmm::chain32_smem_bytes(NT, G, 32 * W) > smem_cap) continue;
    const double waste = 1.0 - static_cast<double>(G * K) / (32.0 * W);
    if (waste > 0.10) continue;
    if (G * K > best_rows) {
      best_rows = G * K;
      best_g = G;
      best_w = W;
    }
  }
  if (best_rows < 0) {  // fall back to the least wasteful fitting shape
    double best_waste = 2.0;
    for (int W = 1; W <= w_max; ++W) {
      const int G = std::min(64, (32 * W) / K);
      if (G < 1 || thmm::chain32_smem_bytes(NT, G, 32 * W) > smem_cap) continue;
      const double waste = 1.0 - static_cast<double>(G * K) / (32.0 * W);
      if (waste < best_waste) {
        best_waste = waste;
        best_g = G;
        best_w = W;
      }
    }
  }
  plan.nt = NT;
  plan.G = best_g;
  plan.W = best_w;
  plan.smem = thmm::chain32_smem_bytes(NT, best_g, 32 * best_w);
  plan.regs = regs;
  int occ = 0;
  THMM_CUDA(thmm::chain_f32_setup<NT>(static_cast<int>(smem_cap), 32 * best_w, plan.smem, &occ));
  plan.ctas_per_sm = std::max(occ, 1);
  plan.sms = prop.multiProcessorCount;
  plan.ready = true;
}

const ChainPlan& chain_plan32(int device, int K) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  ChainPlan& plan = g_plan32[device & 63][K];
  if (!plan.ready) THMM_DISPATCH(padded(K) / 8, false, plan_chain32, device, K, plan);
  return plan;
}

// TF32 tensor-core plan: UMMA N = np, contraction kp, T tiles of 128 rows
// (W = 4T warps), G whole segments per CTA (G K <= 128 T).  T is the largest
// tile count that TMEM (T * cols <= 512), the register budget and shared
// memory allow while wasting at most ~20% of the rows; THMM_TC_TILES
// overrides it (tuning).
#define THMM_TC_DISPATCH_H(np, kp, h, fn, ...)                                         \
  switch ((np) * 10000 + (kp) * 10 + (h)) {                                           \
    case 160081: fn<16, 8, 1>(__VA_ARGS__); break;                                     \
    case 160082: fn<16, 8, 2>(__VA_ARGS__); break;                                     \
    case 160161: fn<16, 16, 1>(__VA_ARGS__); break;                                    \
    case 160162: fn<16, 16, 2>(__VA_ARGS__); break;                                    \
    case 320241: fn<32, 24, 1>(__VA_ARGS__); break;                                    \
    case 320242: fn<32, 24, 2>(__VA_ARGS__); break;                                    \
    case 320321: fn<32, 32, 1>(__VA_ARGS__); break;                                    \
    case 320322: fn<32, 32, 2>(__VA_ARGS__); break;                                    \
    case 480401: fn<48, 40, 1>(__VA_ARGS__); break;                                    \
    case 480402: fn<48, 40, 2>(__VA_ARGS__); break;                                    \
    case 480481: fn<48, 48, 1>(__VA_ARGS__); break;                                    \
    case 480482: fn<48, 48, 2>(__VA_ARGS__); break;                                    \
    case 640561: fn<64, 56, 1>(__VA_ARGS__); break;                                    \
    case 640562: fn<64, 56, 2>(__VA_ARGS__); break;                                    \
    case 640641: fn<64, 64, 1>(__VA_ARGS__); break;                                    \
    case 640642: fn<64, 64, 2>(__VA_ARGS__); break;                                    \
    case 800721: fn<80, 72, 1>(__VA_ARGS__); break;                                    \
    case 800722: fn<80, 72, 2>(__VA_ARGS__); break;                                    \
    case 800801: fn<80, 80, 1>(__VA_ARGS__); break;                                    \
    case 800802: fn<80, 80, 2>(__VA_ARGS__); break;                                    \
    default: throw CudaError{cudaErrorInvalidValue, "bad tensor-core tile shape"};    \
  }

template <int NP, int KP, int H>
void tc_attr(cudaFuncAttributes* attr) { THMM_CUDA((thmm::chain_tc_attributes<NP, KP, H>(attr))); }
template <int NP, int KP, int H>
void tc_setup(int smem) { THMM_CUDA((thmm::chain_tc_setup<NP, KP, H>(smem))); }
template <int NP, int KP, int H>
void tc_launch(const thmm::ChainArgs& a, dim3 grid, int threads, size_t smem, cudaStream_t s) {
  THMM_CUDA((thmm::chain_tc_launch<NP, KP, H>(a, grid, threads, smem, s)));
}

// Column slices per row: 2 (two warps per TMEM lane quarter share a row's
// epilogue, halving its latency) for wide rows, 1 for narrow ones;
// THMM_TC_SLICES overrides (tuning).
int tc_slices(int np) {
  const char* env = std::getenv("THMM_TC_SLICES");
  if (env && (std::atoi(env) == 1 || std::atoi(env) == 2)) return std::atoi(env);
  return np >= 48 ? 2 : 1;
}

void plan_chain_tc(int device, int K, bool x3, ChainPlan& plan) {
  const int np = thmm::tc_np(K), kp = thmm::tc_kp(K), h = tc_slices(np);
  cudaFuncAttributes attr;
  THMM_TC_DISPATCH_H(np, kp, h, tc_attr, &attr);
  cudaDeviceProp prop;
  THMM_CUDA(cudaGetDeviceProperties(&prop, device));
  const size_t smem_cap = prop.sharedMemPerBlockOptin;
  const int t_max = std::min({thmm::tc_max_tiles(np, kp, h), 512 / thmm::tc_cols(np, kp, x3),
                              attr.maxThreadsPerBlock / thmm::tc_tile_threads(h)});
  const char* env = std::getenv("THMM_TC_TILES");
  const int forced = env ? std::atoi(env) : 0;
  int best_t = 0, best_g = 0, fit_t = 0, fit_g = 0;
  double min_waste = 2.0;
  for (int T = 1; T <= t_max; ++T) {
    int G = (thmm::kTcRows * T) / K;  // small K: as many segments as shared memory holds
    while (G > 1 && thmm::chain_tc_smem_bytes(np, kp, G, T, h) > smem_cap) --G;
    if (G < 1 || thmm::chain_tc_smem_bytes(np, kp, G, T, h) > smem_cap) continue;
    if (forced > 0 && T != forced) continue;
    const double waste = 1.0 - static_cast<double>(G * K) / (thmm::kTcRows * T);
    if (waste <= 0.20) best_t = T, best_g = G;  // largest T wasting <= 20% of the rows (more tiles hide the epilogue)
    if (waste < min_waste - 1e-9) min_waste = waste, fit_t = T, fit_g = G;
  }
  if (best_t == 0) best_t = fit_t, best_g = fit_g;
  if (best_t == 0) throw CudaError{cudaErrorInvalidValue, "no tensor-core plan fits"};
  plan.nt = np;
  plan.tail = kp;
  plan.skip = x3;
  plan.G = best_g;
  plan.W = best_t * thmm::tc_tile_threads(h) / 32;
  plan.ctas_per_sm = 1;
  plan.smem = thmm::chain_tc_smem_bytes(np, kp, best_g, best_t, h);
  plan.regs = attr.numRegs;
  plan.slices = h;
  THMM_TC_DISPATCH_H(np, kp, h, tc_setup, static_cast<int>(smem_cap));
  plan.sms = prop.multiProcessorCount;
  plan.ready = true;
}

// mode: 0 tf32, 1 3xTF32 (A_lo columns in TMEM), 2 2xTF32 (same columns as tf32)
const ChainPlan& chain_plan_tc(int device, int K, int mode) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  ChainPlan& plan = g_plan_tc[device & 63][K][mode];
  if (!plan.ready) plan_chain_tc(device, K, mode == 1, plan);
  return plan;
}

int tc_mode(int precision) { return precision == THMM_TF32X3 ? 1 : (precision == THMM_TF32X2 ? 2 : 0); }
bool is_tc(int precision) { return precision == THMM_TF32 || precision == THMM_TF32X3 || precision == THMM_TF32X2; }

const ChainPlan& plan_for(int device, int K, int precision) {
  switch (precision) {
    case THMM_F32: return chain_plan32(device, K);
    case THMM_TF32: return chain_plan_tc(device, K, 0);
    case THMM_TF32X3: return chain_plan_tc(device, K, 1);
    case THMM_TF32X2: return chain_plan_tc(device, K, 2);
    default: return chain_plan(device, K);
  }
}

// ---- run-absorbing FP64 chain (thmm_runs.cuh) -----------------------------
ChainPlan g_plan_runs[64][THMM_MAX_STATES + 1];

// The run-absorbing chain variants as a flat table (head tiles, skip, tail).
struct RunsOps {
  cudaError_t (*attributes)(cudaFuncAttributes*);
  cudaError_t (*setup)(int, int, size_t, int*);
  cudaError_t (*launch)(const thmm::ChainArgs&, dim3, int, size_t, cudaStream_t);
};
template <int NT, bool SKIP, int TAIL>
constexpr RunsOps runs_ops() {
  return {thmm::chain_runs_attributes<NT, SKIP, TAIL>, thmm::chain_runs_setup<NT, SKIP, TAIL>,
          thmm::chain_runs_launch<NT, SKIP, TAIL>};
}
#define THMM_RUNS_PLAIN(N) {runs_ops<N, false, 0>(), runs_ops<N, true, 0>()}
#define THMM_RUNS_TAILS(N) {runs_ops<N, false, 1>(), runs_ops<N, false, 2>(), runs_ops<N, false, 3>(), runs_ops<N, false, 4>()}
// plain[nt-1][skip] (nt = padded tiles 1..10); tailed[nt-1][tail-1] (nt = head tiles 1..9)
const RunsOps kRunsPlain[10][2] = {THMM_RUNS_PLAIN(1), THMM_RUNS_PLAIN(2), THMM_RUNS_PLAIN(3), THMM_RUNS_PLAIN(4),
                                   THMM_RUNS_PLAIN(5), THMM_RUNS_PLAIN(6), THMM_RUNS_PLAIN(7), THMM_RUNS_PLAIN(8),
                                   THMM_RUNS_PLAIN(9), THMM_RUNS_PLAIN(10)};
const RunsOps kRunsTailed[9][4] = {THMM_RUNS_TAILS(1), THMM_RUNS_TAILS(2), THMM_RUNS_TAILS(3),
                                   THMM_RUNS_TAILS(4), THMM_RUNS_TAILS(5), THMM_RUNS_TAILS(6),
                                   THMM_RUNS_TAILS(7), THMM_RUNS_TAILS(8), THMM_RUNS_TAILS(9)};

const RunsOps& runs_ops_for(const ChainPlan& p) {
  return p.tail > 0 ? kRunsTailed[p.nt - 1][p.tail - 1] : kRunsPlain[p.nt - 1][p.skip ? 1 : 0];
}

// Same column split as the record-by-record kernel (plan_chain64): DMMA head
// tiles + SIMT tail for K % 8 in 1..4 (K >= 9), else padded tiles.  One
// segment per group of padded-K/8 warps, 16 warps per CTA.
void plan_runs(int device, int K, ChainPlan& plan) {
  const int r = K % 8;
  if (K >= 9 && r >= 1 && r <= 4) {
    plan.nt = K / 8;
    plan.tail = r;
    plan.skip = false;
  } else {
    plan.nt = (K + 7) / 8;
    plan.tail = 0;
    plan.skip = skip_h1(K);
  }
  const int rt = padded(K) / 8;
  const RunsOps& ops = runs_ops_for(plan);
  cudaFuncAttributes attr;
  THMM_CUDA(ops.attributes(&attr));
  cudaDeviceProp prop;
  THMM_CUDA(cudaGetDeviceProperties(&prop, device));
  plan.G = thmm::runs_groups(plan.nt, plan.tail);
  plan.W = plan.G * rt;
  plan.smem = thmm::runs_smem_bytes(plan.nt, plan.tail, plan.G);
  plan.regs = attr.numRegs;
  int occ = 0;
  THMM_CUDA(ops.setup(static_cast<int>(prop.sharedMemPerBlockOptin), 32 * plan.W, plan.smem, &occ));
  plan.ctas_per_sm = std::max(occ, 1);
  plan.sms = prop.multiProcessorCount;
  plan.ready = true;
}

const ChainPlan& runs_plan(int device, int K) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  ChainPlan& plan = g_plan_runs[device & 63][K];
  if (!plan.ready) plan_runs(device, K, plan);
  return plan;
}

// Run-absorbing chain mode: 0 never, 1 always (tests, tuning), -1 by the
// cost model.  Initialised from THMM_RUNS, changed by thmm_set_runs_mode.
std::atomic<int> g_runs_mode{-2};
int runs_env() {
  int v = g_runs_mode.load(std::memory_order_relaxed);
  if (v == -2) {
    const char* e = std::getenv("THMM_RUNS");
    v = e ? std::atoi(e) : -1;
    if (v < -1 || v > 1) v = -1;
    int expect = -2;
    if (!g_runs_mode.compare_exchange_strong(expect, v)) v = expect;
  }
  return v;
}

// Chunk limits R the run-absorbing chain uses (thmm::runs_r).
constexpr int kRunsR[6] = {2, 3, 4, 8, 16, 32};

// Steps per record of the run-absorbing chain for every chunk limit R in
// kRunsR (the rule of chain_runs_kernel: a record starts a step when present,
// or absent at a run position that is a multiple of R, runs restarting every
// 32 records), estimated from up to `windows` evenly spaced 32-record
// windows; ratio[R] (index R <= 32).
void estimate_runs_ratios(const uint8_t* present, int64_t n, double* ratio, int64_t windows = 512) {
  const int64_t nwin = (n + thmm::kRunWin - 1) / thmm::kRunWin;
  const int64_t take = std::min<int64_t>(nwin, windows);
  int64_t steps[6] = {0, 0, 0, 0, 0, 0}, recs = 0, present_cnt = 0;
  for (int64_t k = 0; k < take; ++k) {
    const int64_t w = take == nwin ? k : (k * nwin) / take;
    const int64_t t0 = w * thmm::kRunWin, cnt = std::min<int64_t>(thmm::kRunWin, n - t0);
    int rstart = 0;
    for (int i = 0; i < cnt; ++i) {
      if (present[t0 + i]) {
        for (auto& v : steps) ++v;
        ++present_cnt;
        rstart = i + 1;
      } else {
        for (int r = 0; r < 6; ++r) steps[r] += ((i - rstart) % kRunsR[r]) == 0;
      }
    }
    recs += cnt;
  }
  for (int r = 0; r <= 32; ++r) ratio[r] = -1.0;
  if (recs)
    for (int r = 0; r < 6; ++r) ratio[kRunsR[r]] = static_cast<double>(steps[r]) / static_cast<double>(recs);
  if (recs) ratio[0] = static_cast<double>(present_cnt) / static_cast<double>(recs);  // fraction of events
}

bool runs_eligible(int K, int precision) { return precision == THMM_F64 && K >= 1 && K <= THMM_MAX_STATES; }

// Use the run-absorbing chain when its work -- steps x padded rows, with the
// same per-tile column work as the record-by-record kernel (x1.2 per-window
// overhead for one- and two-tile rows) -- undercuts that kernel's records x
// K stacked rows by 5%.  Calibrated on B200 with tools/runs_probe.py.
// Rows wider than 4 tiles also need a long enough stream to amortise the
// per-CTA table of powers (R-1 products of up to 80 x 80 in the prologue):
// below ~2.6e5 records the record-by-record kernel wins (round-1 latency probe; tools/latency_breakdown.py).
constexpr int64_t kRunsMinRecordsWide = 262144;

bool use_runs(int K, int precision, double ratio, int64_t n) {
  if (!runs_eligible(K, precision)) return false;
  const int env = runs_env();
  if (env == 0) return false;
  if (env == 1) return true;
  if (!(ratio > 0.0)) return false;
  if (padded(K) > 32 && n < kRunsMinRecordsWide) return false;
  const int KP = padded(K);
  return ratio * KP * (KP <= 16 ? 1.2 : 1.0) < 0.95 * K;
}

double obs_runs_ratio(thmm_obs obs, int K) { return obs->runs_ratio[thmm::runs_r_for_k(K)]; }

bool runs_for(thmm_obs obs, int K, int precision, int64_t n = -1) {
  return use_runs(K, precision, obs_runs_ratio(obs, K), n < 0 ? obs->n : n);
}

void launch_chain_runs(const thmm::ChainArgs& a, const ChainPlan& plan, int64_t ctas, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(ctas), static_cast<unsigned>(a.B));
  THMM_CUDA(runs_ops_for(plan).launch(a, grid, 32 * plan.W, plan.smem, s));
  ++g_launches;
}


// ---- rank-one collapse + row-stacked vector continuation (thmm_vec.cuh) ----
ChainPlan g_plan_vec[64][THMM_MAX_STATES + 1];

template <int NT, bool SKIP, int TAIL>
constexpr RunsOps vec_ops() {
  return {thmm::chain_vec_attributes<NT, SKIP, TAIL>, thmm::chain_vec_setup<NT, SKIP, TAIL>,
          thmm::chain_vec_launch<NT, SKIP, TAIL>};
}
#define THMM_VEC_PLAIN(N) {vec_ops<N, false, 0>(), vec_ops<N, true, 0>()}
#define THMM_VEC_TAILS(N) {vec_ops<N, false, 1>(), vec_ops<N, false, 2>(), vec_ops<N, false, 3>(), vec_ops<N, false, 4>()}
const RunsOps kVecPlain[10][2] = {THMM_VEC_PLAIN(1), THMM_VEC_PLAIN(2), THMM_VEC_PLAIN(3), THMM_VEC_PLAIN(4),
                                  THMM_VEC_PLAIN(5), THMM_VEC_PLAIN(6), THMM_VEC_PLAIN(7), THMM_VEC_PLAIN(8),
                                  THMM_VEC_PLAIN(9), THMM_VEC_PLAIN(10)};
const RunsOps kVecTailed[9][4] = {THMM_VEC_TAILS(1), THMM_VEC_TAILS(2), THMM_VEC_TAILS(3),
                                  THMM_VEC_TAILS(4), THMM_VEC_TAILS(5), THMM_VEC_TAILS(6),
                                  THMM_VEC_TAILS(7), THMM_VEC_TAILS(8), THMM_VEC_TAILS(9)};

const RunsOps& vec_ops_for(const ChainPlan& p) {
  return p.tail > 0 ? kVecTailed[p.nt - 1][p.tail - 1] : kVecPlain[p.nt - 1][p.skip ? 1 : 0];
}

// The stitched chain's kernels (same geometry as the vector kernel).
struct StitchOps {
  cudaError_t (*setup)(int);
  cudaError_t (*fwd)(const thmm::ChainArgs&, dim3, int, size_t, cudaStream_t);
  cudaError_t (*link)(const thmm::ChainArgs&, dim3, int, size_t, cudaStream_t);
  cudaError_t (*finish)(const thmm::ChainArgs&, double*, int32_t*, double*, cudaStream_t);
  cudaError_t (*prep)(const thmm::ChainArgs&, double2*, cudaStream_t);
};
template <int NT, bool SKIP, int TAIL>
constexpr StitchOps stitch_ops() {
  return {thmm::chain_fwd_setup<NT, SKIP, TAIL>, thmm::chain_fwd_launch<NT, SKIP, TAIL>,
          thmm::chain_link_launch<NT, SKIP, TAIL>, thmm::stitch_finish_launch<NT, SKIP, TAIL>,
          thmm::entry_prep_launch<NT, SKIP, TAIL>};
}
#define THMM_ST_PLAIN(N) {stitch_ops<N, false, 0>(), stitch_ops<N, true, 0>()}
#define THMM_ST_TAILS(N) {stitch_ops<N, false, 1>(), stitch_ops<N, false, 2>(), stitch_ops<N, false, 3>(), stitch_ops<N, false, 4>()}
const StitchOps kStPlain[10][2] = {THMM_ST_PLAIN(1), THMM_ST_PLAIN(2), THMM_ST_PLAIN(3), THMM_ST_PLAIN(4),
                                   THMM_ST_PLAIN(5), THMM_ST_PLAIN(6), THMM_ST_PLAIN(7), THMM_ST_PLAIN(8),
                                   THMM_ST_PLAIN(9), THMM_ST_PLAIN(10)};
const StitchOps kStTailed[9][4] = {THMM_ST_TAILS(1), THMM_ST_TAILS(2), THMM_ST_TAILS(3),
                                   THMM_ST_TAILS(4), THMM_ST_TAILS(5), THMM_ST_TAILS(6),
                                   THMM_ST_TAILS(7), THMM_ST_TAILS(8), THMM_ST_TAILS(9)};
const StitchOps& stitch_ops_for(const ChainPlan& p) {
  return p.tail > 0 ? kStTailed[p.nt - 1][p.tail - 1] : kStPlain[p.nt - 1][p.skip ? 1 : 0];
}

// Same column split as the run-absorbing chain; vec_warps() warps of 8 rows
// (segments) per CTA.
void plan_vec(int device, int K, ChainPlan& plan) {  // (called with g_plan_mu held)
  const int r = K % 8;
  if (K >= 9 && r >= 1 && r <= 4) {
    plan.nt = K / 8;
    plan.tail = r;
    plan.skip = false;
  } else {
    plan.nt = (K + 7) / 8;
    plan.tail = 0;
    plan.skip = skip_h1(K);
  }
  plan.W = thmm::vec_warps(plan.nt + (plan.tail > 0));
  plan.G = 8 * plan.W;
  const RunsOps& ops = vec_ops_for(plan);
  cudaFuncAttributes attr;
  THMM_CUDA(ops.attributes(&attr));
  cudaDeviceProp prop;
  THMM_CUDA(cudaGetDeviceProperties(&prop, device));
  plan.smem = thmm::vec_smem_bytes(plan.nt, plan.tail, plan.W);
  plan.regs = attr.numRegs;
  int occ = 0;
  // (the kernels' static shared memory -- the prologue's mbarrier -- comes off the opt-in maximum)
  const int dyn_max = static_cast<int>(prop.sharedMemPerBlockOptin) - 1024;
  THMM_CUDA(ops.setup(dyn_max, 32 * plan.W, plan.smem, &occ));
  THMM_CUDA(stitch_ops_for(plan).setup(dyn_max));
  plan.ctas_per_sm = std::max(occ, 1);
  plan.sms = prop.multiProcessorCount;
  plan.ready = true;
}

const ChainPlan& vec_plan(int device, int K) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  ChainPlan& plan = g_plan_vec[device & 63][K];
  if (!plan.ready) plan_vec(device, K, plan);
  return plan;
}

// Launch shape of a row-stacked kernel for `warps` warps per proposal: the
// plan's W warps per CTA when the launch fills the GPU's CTA slots; below
// that the warps are spread over every SM (W' = ceil(B warps / SMs) per CTA,
// a few warps per SM, one per sub-partition where they fit) instead of packed
// into a few full CTAs -- a chain step is a dependent DMMA/FP64 sequence, so a
// warp sharing its scheduler with four others runs ~4x slower per step.
// Spread launches of at most 8 warps per SM batch their emissions (the
// events of 8 steps at a time, ChainArgs::ebatch) when the 64-row buffers fit:
// a lone warp's per-step emission is a ~25-deep FP64 dependency chain, four
// independent ones per lane hide it (THMM_VEC_BATCH=0/1 forces off/on).
struct VecSpread {
  int W;
  int64_t ctas;  // per proposal
  size_t smem;
  bool batch;
};
VecSpread vec_spread(const ChainPlan& vp, int B, int64_t warps) {
  warps = std::max<int64_t>(1, warps);
  const int64_t slots = static_cast<int64_t>(vp.sms) * vp.ctas_per_sm;
  int64_t W = vp.W;
  static const bool off = [] {
    const char* e = std::getenv("THMM_VEC_SPREAD");
    return e && e[0] == '0';
  }();
  static const int bmode = [] {
    const char* e = std::getenv("THMM_VEC_BATCH");
    return e ? std::atoi(e) : -1;
  }();
  bool spread = false;
  if (!off && static_cast<int64_t>(B) * ((warps + W - 1) / W) < slots) {
    W = std::min<int64_t>(vp.W, std::max<int64_t>(1, (static_cast<int64_t>(B) * warps + vp.sms - 1) / vp.sms));
    spread = true;
  }
  const int w = static_cast<int>(W);
  const size_t sb = thmm::vec_smem_bytes(vp.nt, vp.tail, w, true);
  const bool fits = sb + 1024 <= thmm::kRunsSmemCap;
  const bool batch = bmode == 0 ? false : (bmode == 1 ? fits : (spread && w <= 8 && fits));
  return VecSpread{w, (warps + W - 1) / W, batch ? sb : thmm::vec_smem_bytes(vp.nt, vp.tail, w), batch};
}

void launch_chain_vec(thmm::ChainArgs a, const ChainPlan& plan, const VecSpread& sp, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(sp.ctas), static_cast<unsigned>(a.B));
  a.ebatch = sp.batch ? 1 : 0;
  THMM_CUDA(vec_ops_for(plan).launch(a, grid, 32 * sp.W, sp.smem, s));
  ++g_launches;
}

// Stitch mode: THMM_STITCH=0 disables; thread-local overrides while the host
// repeats an evaluation whose links did not converge (first with segments
// g_stitch_len_scale times longer, then without the stitch).
thread_local bool g_no_stitch = false;
thread_local int g_stitch_len_scale = 1;
std::atomic<int> g_stitch_mode{-2};
int stitch_mode() {
  int v = g_stitch_mode.load(std::memory_order_relaxed);
  if (v == -2) {
    const char* e = std::getenv("THMM_STITCH");
    v = (e && e[0] == '0') ? 0 : 1;
    int expect = -2;
    if (!g_stitch_mode.compare_exchange_strong(expect, v)) v = expect;
  }
  return v;
}

// How a host-array (pinned, B = 1) stitched evaluation reads its records:
// 1 staged into HBM by DMA in time chunks the main pass follows, 2 in place
// over PCIe with every line loaded (one round trip per window), 3 in place,
// coordinates of events only; 0 (default) chooses by the event fraction
// (THMM_STITCH_HOST overrides).
int stitch_host_mode(double event_frac) {
  static const int env = [] {
    const char* e = std::getenv("THMM_STITCH_HOST");
    return e ? std::atoi(e) : 0;
  }();
  if (env >= 1 && env <= 3) return env;
  // B200 e2e (tools/e2e_probe.py): K=50 N=1e7 (40 % events) staged 4.4 ms vs
  // in place 5.3; K=25 N=1e6 (13 %) staged 0.91 vs in place 0.70 (the 2-D
  // copies of short segment slices run below the DMA rate)
  return event_frac >= 0.25 ? 1 : 3;
}

// Collapse mode: THMM_COLLAPSE=0 disables (tests compare both paths); tolerance
// THMM_COLLAPSE_TOL (default 2^-40 relative per entry, i.e. a likelihood
// factor within 1 +- 1e-12 per segment); segments no shorter than
// THMM_COLLAPSE_MINLEN records (default 1024: the burn-in of ~32-64 records
// stays a few percent of a segment).
std::atomic<int> g_collapse_mode{-2};
std::atomic<int> g_collapse_gen{0};  // bumped by thmm_set_collapse_params (graph keys)
int collapse_mode() {
  int v = g_collapse_mode.load(std::memory_order_relaxed);
  if (v == -2) {
    const char* e = std::getenv("THMM_COLLAPSE");
    v = (e && e[0] == '0') ? 0 : 1;
    int expect = -2;
    if (!g_collapse_mode.compare_exchange_strong(expect, v)) v = expect;
  }
  return v;
}
// Mode plus parameter generation: the key recorded with every CUDA graph
// (a graph bakes in the segment split the parameters chose).
int collapse_env() {
  return collapse_mode() + 2 * stitch_mode() + 4 * g_collapse_gen.load(std::memory_order_relaxed);
}
std::atomic<double> g_collapse_tol{0.0};
std::atomic<int64_t> g_collapse_minlen{0};
double collapse_tol() {
  double v = g_collapse_tol.load(std::memory_order_relaxed);
  if (v <= 0.0) {
    const char* e = std::getenv("THMM_COLLAPSE_TOL");
    v = e ? std::atof(e) : 0.0;
    if (!(v > 0.0)) v = 0x1p-40;
    g_collapse_tol.store(v);
  }
  return v;
}
int64_t collapse_min_len() {
  int64_t v = g_collapse_minlen.load(std::memory_order_relaxed);
  if (v <= 0) {
    const char* e = std::getenv("THMM_COLLAPSE_MINLEN");
    const long long x = e ? std::atoll(e) : 0;
    v = x > 0 ? x : 1024;
    g_collapse_minlen.store(v);
  }
  return v;
}

// Gate of the collapse mode: B n >= min_fill x 1024 x (rows of one wave), K > 8;
// 0 = no gate (tests).  Default 0.25.
std::atomic<double> g_collapse_fill{-1.0};
double collapse_min_fill() {
  double v = g_collapse_fill.load(std::memory_order_relaxed);
  if (v < 0.0) {
    v = 0.25;
    g_collapse_fill.store(v);
  }
  return v;
}

// Records between rank-one tests in the burn-in (THMM_COLLAPSE_WIN, 1..32,
// default 8: the synthetic K=80 stream's segments converge after 16-48
// records, most by 24).
int collapse_win() {
  static const int v = [] {
    const char* e = std::getenv("THMM_COLLAPSE_WIN");
    const int x = e ? std::atoi(e) : 0;
    return x >= 1 && x <= 32 ? x : 8;
  }();
  return v;
}

// Segments per proposal of a collapse-mode evaluation, 0 = not this mode:
// FP64, automatic segment count, and a chain long enough that every segment
// keeps >= collapse_min_len() records; one full wave of vector rows
// (8 W rows per CTA x CTAs per SM x SMs) across the B proposals, or fewer.
int64_t collapse_segments(int device, int K, const thmm_config* cfg, int64_t n, int B) {
  if (cfg->precision != THMM_F64 || cfg->segments > 0 || collapse_mode() == 0) return 0;
  const int64_t minlen = collapse_min_len();
  if (n < 2 * minlen) return 0;
  const ChainPlan& vp = vec_plan(device, K);
  const int64_t wave = static_cast<int64_t>(vp.sms) * vp.ctas_per_sm * 8 * vp.W;
  // The vector continuation pays off once it can keep a quarter wave of rows
  // busy for >= 1024 records each (shorter or narrower: latency-bound, and the
  // matrix path's work per record, 2K^3 vs 2K^2, is small at small K); K <= 8
  // stays on the matrix path.
  const double fill = collapse_min_fill();
  if (fill > 0.0 && (K <= 8 || static_cast<double>(B) * static_cast<double>(n) < fill * 1024.0 * wave)) return 0;
  const int64_t per_prop = std::max<int64_t>(1, wave / std::max(B, 1));
  return std::max<int64_t>(1, std::min<int64_t>(per_prop, n / minlen));
}

// Segments of a stitched-chain evaluation, 0 = use the other paths.  Chosen
// by a cost model (gate off: always, for the tests): the matrix paths cost
// n B 2K^3 (x steps/record when the run-absorbing chain runs) at their
// measured DMMA efficiency; the stitched chain n B 2K K_p at its own, or --
// below a wave of rows -- its latency, (n/S + 48 link records) per-step
// warp latencies.  Segments are one wave of vector rows across the B
// proposals, at least 192 records long (links need a few dozen records to
// converge; shorter segments made K=25 links fail).
// Calibration (tools/stitch_latency.py, spread launch + pipelined emissions):
// K=25 N=1e6 stitched 0.31 ms vs matrix 0.48 ms; K=50 N=1.05e5 0.48 vs 1.0 ms;
// K=25 N=1.05e5 0.24 vs 0.11 ms and K=5 N=1e4 0.19 vs 0.033 ms (matrix kept).
int64_t stitch_segments(int device, int K, const thmm_config* cfg, int64_t n, int B, double runs_ratio,
                        double zc_events = -1.0, double events = -1.0) {
  if (cfg->precision != THMM_F64 || cfg->segments > 0 || collapse_mode() == 0 || stitch_mode() == 0) return 0;
  // shortest segment: a link must converge inside it.  Streams with >= 25 %
  // events mix fast (links of a few dozen records; 96-record segments ran
  // without a failed link at K=5/50/80 and cut K=50/80 N=1.05e5 by 35 %);
  // sparse ones 160 (the K=25 stream, 13 % events: links failed at 96-128,
  // none at 144-192; 160 vs 192: K=25 N=1e6 281 -> 242 us).  A failed link
  // repeats the evaluation with segments twice as long.
  const int64_t minlen = std::min<int64_t>(events >= 0.25 ? 96 : 160, collapse_min_len()) * g_stitch_len_scale;
  if (n < 2 * minlen) return 0;
  const ChainPlan& vp = vec_plan(device, K);
  const int64_t wave = static_cast<int64_t>(vp.sms) * vp.ctas_per_sm * 8 * vp.W;
  int64_t S = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(1, wave / std::max(B, 1)), n / minlen));
  const int64_t rows = 8 * vp.W, slots = static_cast<int64_t>(vp.sms) * vp.ctas_per_sm;
  if (B > 1 && n / minlen >= rows && static_cast<int64_t>(B) * ((S + rows - 1) / rows) >= slots) {
    // batches that fill the GPU: whole CTAs per proposal (a CTA stages ONE
    // proposal's Gamma, so a part-filled CTA idles warps), c CTAs each, c minimising
    // waves x (records per segment + ~48 link steps): 256 proposals x 1e6
    // records -> c = 4 (7 waves at 99 % fill) instead of 92 rows (2 waves, 86 %)
    int64_t best_c = 1;
    double best_t = 1e300;
    const int64_t cmax = std::min<int64_t>(n / minlen / rows, 8);
    for (int64_t c = 1; c <= cmax; ++c) {
      const double waves = std::ceil(static_cast<double>(B) * c / static_cast<double>(slots));
      const double t = waves * (static_cast<double>(n) / static_cast<double>(rows * c) + 48.0);
      if (t < best_t * 0.999) {
        best_t = t;
        best_c = c;
      }
    }
    S = rows * best_c;
  }
  if (collapse_min_fill() <= 0.0) return S;  // gate off
  const int KP = padded(K);
  const double peak = 37.1e12, nb = static_cast<double>(n) * B, k = K;
  const double eff_m = KP <= 32 ? 0.5 : (KP <= 56 ? 0.65 : 0.9);
  const double r = (runs_ratio > 0.0 && runs_ratio < 1.0) ? runs_ratio : 1.0;
  const double t_mat = nb * 2.0 * k * k * k * r / (eff_m * peak);
  const double eff_v = KP <= 32 ? 0.2 : (KP <= 56 ? 0.4 : 0.6);
  // per-step latency of a warp of the spread launch (vec_spread, batched
  // emissions), main pass + links, fitted on B200 (tools/stitch_latency.py):
  // K_p = 8: 0.43 us, 32: 0.87, 56: 1.73, 80: 3.87; warps beyond one per
  // sub-partition share it
  const double t_lat = (0.44 - 0.0062 * KP + 0.000613 * KP * KP) * 1e-6;
  const double warps = static_cast<double>(B) * ((S + 7) / 8);
  const double share = std::max(1.0, warps / (4.0 * vp.sms));
  double t_st =
      std::max(nb * 2.0 * k * KP / (eff_v * peak), (static_cast<double>(n) / S + 48.0) * t_lat * share);
  double t_m = t_mat;
  if (zc_events >= 0.0 && stitch_host_mode(zc_events) == 3) {
    // records read in place over PCIe (~25 GB/s of uncached reads; the flag
    // byte plus the 128-byte lines of coordinates that hold an event), once by
    // the matrix paths, ~1.25x by the stitched chain (links re-read the
    // segment heads): K=25 N=1e6, 13 % events: 0.56 vs 0.70 ms (B200)
    const double lines = 1.0 - std::pow(1.0 - std::min(1.0, zc_events), 16.0);
    const double t_pcie = static_cast<double>(n) * (1.0 + 16.0 * lines) / 25e9;
    t_st = std::max(t_st, 1.25 * t_pcie);
    t_m = std::max(t_m, t_pcie);
  }
  return t_st < 0.8 * t_m ? S : 0;
}

template <int NT, bool SKIP>
void prepare_fold(int) {
  THMM_CUDA((thmm::fold_setup<NT, SKIP>(static_cast<int>(fold_smem(NT)))));
  THMM_CUDA((thmm::tree_setup<NT, SKIP>(static_cast<int>(thmm::tree_smem_bytes(NT)))));
}

void ensure_fold(int device, int K) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  const int nt = padded(K) / 8;
  bool& ready = g_fold_ready[device & 63][nt][skip_h1(K)];
  if (!ready) {
    THMM_DISPATCH(nt, skip_h1(K), prepare_fold, device);
    ready = true;
  }
}

bool prof_events(int device) {
  if (g_prof_ev_device != device) {
    for (auto& e : g_prof_ev) {
      if (e) cudaEventDestroy(e);
      e = nullptr;
    }
    for (auto& e : g_prof_ev) THMM_CUDA(cudaEventCreate(&e));
    g_prof_ev_device = device;
  }
  return true;
}

void launch_chain(const thmm::ChainArgs& a, const ChainPlan& plan, int precision, int64_t ctas, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(ctas), static_cast<unsigned>(a.B));
  if (is_tc(precision)) {
    THMM_TC_DISPATCH_H(plan.nt, plan.tail, plan.slices, tc_launch, a, grid, 32 * plan.W, plan.smem, s);
  } else if (precision == THMM_F32) {
#define THMM_F32_LAUNCH(N) \
  case N: THMM_CUDA(thmm::chain_f32_launch<N>(a, grid, 32 * plan.W, plan.smem, s)); break;
    switch (plan.nt) {
      THMM_F32_LAUNCH(1) THMM_F32_LAUNCH(2) THMM_F32_LAUNCH(3) THMM_F32_LAUNCH(4) THMM_F32_LAUNCH(5)
      THMM_F32_LAUNCH(6) THMM_F32_LAUNCH(7) THMM_F32_LAUNCH(8) THMM_F32_LAUNCH(9) THMM_F32_LAUNCH(10)
      default: throw CudaError{cudaErrorInvalidValue, "bad padded state count"};
    }
#undef THMM_F32_LAUNCH
  } else {
    THMM_CUDA(ops_for(plan).launch(a, grid, 32 * plan.W, plan.smem, s));
  }
  ++g_launches;
}

template <int NT, bool SKIP>
void launch_fold(const thmm::FoldArgs& a, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(a.n_out), static_cast<unsigned>(a.B));
  THMM_CUDA((thmm::fold_launch<NT, SKIP>(a, grid, fold_smem(NT), s)));
  ++g_launches;
}


}  // namespace
