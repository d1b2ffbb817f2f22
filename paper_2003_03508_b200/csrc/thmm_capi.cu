// thmm_capi.cu -- C-ABI of the B200 HMM likelihood (declared in include/thmm.h).
//
// Host orchestration only: device-resident observation handles, a per-handle
// workspace (grown, never shrunk, so steady-state calls do no cudaMalloc),
// kernel dispatch over the padded state count, the segment tree, and error
// translation.  The arithmetic lives in thmm_kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "thmm.h"
#include "thmm_launch.cuh"
#include "thmm_tc.cuh"

namespace {

thread_local int g_launches = 0;
thread_local bool g_profile = false;
thread_local double g_prof_chain_ms = 0.0, g_prof_fold_ms = 0.0;
thread_local int64_t g_prof_segments = 0;
thread_local cudaEvent_t g_prof_ev[3] = {nullptr, nullptr, nullptr};
thread_local int g_prof_ev_device = -1;
thread_local bool g_capturing = false;  // inside capture_graph's stream capture

// Profiling events become external event nodes when recorded during capture.
cudaError_t record_prof(cudaEvent_t ev, cudaStream_t s) {
  return g_capturing ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal) : cudaEventRecord(ev, s);
}

// Nodes multiplied per CTA per tree level.  The latency of the one-launch tree
// is ~radix * log_radix(S) sequential products; 4 is near the minimum.
constexpr int kFoldRadix = 4;
constexpr int64_t kMinSegment = 48; // shortest segment the auto split produces
constexpr int64_t kMinFirstChunk = 32768;  // host-array pipeline: smallest first chunk
constexpr int64_t kMinSegmentSmall = 16;   // shortest segment for chains under one wave

void set_err(char* err, size_t errlen, const char* fmt, ...) {
  if (!err || errlen == 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

struct CudaError {
  cudaError_t code;
  const char* what;
};

#define THMM_CUDA(call)                                  \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) throw CudaError{e_, #call};   \
  } while (0)

struct DeviceBuffer {
  void* ptr = nullptr;
  size_t cap = 0;
  void* ensure(size_t bytes) {
    if (bytes > cap) {
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      cap = 0;
      THMM_CUDA(cudaMalloc(&ptr, bytes));
      cap = bytes;
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

struct HostPinned {
  void* ptr = nullptr;
  size_t cap = 0;
  void* ensure(size_t bytes) {
    if (bytes > cap) {
      if (ptr) cudaFreeHost(ptr);
      ptr = nullptr;
      cap = 0;
      THMM_CUDA(cudaMallocHost(&ptr, bytes));
      cap = bytes;
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

struct Workspace {
  DeviceBuffer params;   // gamma | delta | states
  DeviceBuffer nodes_a;  // segment / level nodes (ping)
  DeviceBuffer nodes_b;  // level nodes (pong)
  DeviceBuffer exps_a, exps_b;
  DeviceBuffer result;   // loglik[B] | status[B]
  DeviceBuffer counters; // tree arrival counters (zero between launches)
  HostPinned staging;    // params upload + results download
  cudaEvent_t staged = nullptr;  // last asynchronous use of `staging` (range_nodes_async)
  bool staged_pending = false;
  void release() {
    params.release();
    nodes_a.release();
    nodes_b.release();
    exps_a.release();
    exps_b.release();
    result.release();
    counters.release();
    if (staged) {
      cudaEventSynchronize(staged);
      cudaEventDestroy(staged);
    }
    staged = nullptr;
    staged_pending = false;
    staging.release();
  }
};

}  // namespace

struct thmm_obs_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n = 0;
  int64_t cap = 0;
  uint8_t* present = nullptr;
  double* lon = nullptr;
  double* lat = nullptr;
  Workspace ws;
  std::mutex mu;
  // host-array pipeline: copies on their own stream, one event per chunk
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t chunk_ready[8] = {};
  cudaEvent_t reads_done = nullptr;  // launch-stream point the next upload waits for
  cudaStream_t chunk_streams[8] = {};  // per-chunk chain launches of the host pipeline
  cudaEvent_t chunk_done[8] = {};
  cudaEvent_t params_ready = nullptr;
  // CUDA graphs of the whole evaluation (params H2D, chain, tree, result D2H)
  // for recently used configurations; replayed instead of re-launching.
  struct Graph {
    bool valid = false;
    int K = 0, B = 0, precision = 0, period = 0;
    int64_t segments = 0, lo = 0, hi = 0;
    bool prof = false;
    uintptr_t signature = 0;  // buffer addresses the graph was captured against
    int64_t nseg = 0;
    cudaGraphExec_t exec = nullptr;
    unsigned long long last_use = 0;
  } graphs[4];
  // CUDA graphs of the host-array pipeline (thmm_loglik_host) for recently
  // used pinned source buffers.
  struct HostGraph {
    bool valid = false;
    const void* src[3] = {};
    int64_t n = 0;
    int K = 0, B = 0, precision = 0, period = 0;
    int64_t segments = 0;
    bool prof = false;
    uintptr_t signature = 0;
    int64_t nseg = 0;
    int launches = 0;
    cudaGraphExec_t exec = nullptr;
    unsigned long long last_use = 0;
  } host_graphs[2];
  unsigned long long uses = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) THMM_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int padded(int K) { return ((K + 7) / 8) * 8; }

size_t fold_smem(int nt) { return static_cast<size_t>(nt) * nt * 32 * sizeof(double2) + nt * sizeof(double); }

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

template <int NT, bool SKIP>
void prepare_fold(int) {
  THMM_CUDA((thmm::fold_setup<NT, SKIP>(static_cast<int>(fold_smem(NT)))));
  THMM_CUDA((thmm::tree_setup<NT, SKIP>(static_cast<int>(fold_smem(NT)))));
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

int validate_params(const thmm_params* P, char* err, size_t errlen) {
  if (!P || !P->gamma || !P->delta || !P->states) {
    set_err(err, errlen, "parameter pointers must be non-NULL");
    return THMM_EINVAL;
  }
  if (P->K < 1 || P->K > THMM_MAX_STATES) {
    set_err(err, errlen, "parallel engine supports at most %d states, got %d", THMM_MAX_STATES, P->K);
    return THMM_EINVAL;
  }
  if (P->B < 1 || P->B > 65535) {
    set_err(err, errlen, "batch size must lie in [1, 65535], got %d", P->B);
    return THMM_EINVAL;
  }
  return THMM_OK;
}

// Upload the B parameter sets to the workspace; returns device pointers.
// Copy the B parameter sets into the pinned staging buffer (gamma | delta | states).
// Every call ends with a stream sync, so the previous upload has completed.
cudaEvent_t staged_event(Workspace& ws) {
  if (!ws.staged) THMM_CUDA(cudaEventCreateWithFlags(&ws.staged, cudaEventDisableTiming));
  ws.staged_pending = true;
  return ws.staged;
}

double* stage_params_host(Workspace& ws, const thmm_params* P) {
  if (ws.staged_pending && !g_capturing) {  // an asynchronous call may still be reading the buffer
    THMM_CUDA(cudaEventSynchronize(ws.staged));
    ws.staged_pending = false;
  }
  const size_t K = P->K, B = P->B;
  const size_t n_gamma = B * K * K, n_delta = B * K, n_states = 8 * B * K;
  const size_t bytes = (n_gamma + n_delta + n_states) * sizeof(double);
  double* host = static_cast<double*>(ws.staging.ensure(bytes + 2 * B * sizeof(double)));
  std::memcpy(host, P->gamma, n_gamma * sizeof(double));
  std::memcpy(host + n_gamma, P->delta, n_delta * sizeof(double));
  std::memcpy(host + n_gamma + n_delta, P->states, n_states * sizeof(double));
  return host;
}

thmm::StateParams upload_params(Workspace& ws, const thmm_params* P, cudaStream_t s) {
  const size_t K = P->K, B = P->B;
  const size_t n_gamma = B * K * K, n_delta = B * K, n_states = 8 * B * K;
  const size_t bytes = (n_gamma + n_delta + n_states) * sizeof(double);
  double* host = stage_params_host(ws, P);
  double* dev = static_cast<double*>(ws.params.ensure(bytes));
  THMM_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
  return thmm::StateParams{dev, dev + n_gamma + n_delta, dev + n_gamma};
}

// Segments per proposal: c CTAs of G segments each, with c chosen so that the
// B*c CTAs fill whole waves of resident CTAs (wave efficiency
// (B c / slots) / ceil(B c / slots), ties to the smallest c), never shorter
// than kMinSegment records per segment.
int64_t auto_segments(const ChainPlan& plan, int64_t n, int B) {
  const int64_t slots = static_cast<int64_t>(plan.sms) * plan.ctas_per_sm;
  // Short chains that cannot fill one wave at kMinSegment records per segment
  // use shorter segments (latency: fewer sequential steps and emissions per CTA).
  const int64_t seg_min = B * (n / (kMinSegment * plan.G)) < slots ? kMinSegmentSmall : kMinSegment;
  const int64_t c_max = std::max<int64_t>(1, std::min<int64_t>(n / (seg_min * plan.G), 64 * slots));
  int64_t best_c = 1;
  double best_eff = -1.0;
  for (int64_t c = 1; c <= std::min<int64_t>(c_max, 4 * slots); ++c) {
    const double waves = static_cast<double>(B * c) / slots;
    const double eff = waves / std::ceil(waves - 1e-12);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best_c = c;
    }
  }
  int64_t per_prop = best_c * plan.G;
  if (c_max == 1) per_prop = std::max<int64_t>(1, std::min<int64_t>(plan.G, n / seg_min));
  return std::min<int64_t>(per_prop, n);
}

template <int NT, bool SKIP>
void launch_tree(const thmm::TreeArgs& a, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(a.count[1]), static_cast<unsigned>(a.B));
  THMM_CUDA((thmm::tree_launch<NT, SKIP>(a, grid, fold_smem(NT), s)));
  ++g_launches;
}

// Ordered fold of n0 nodes per proposal (layout given by element strides)
// with the one-launch radix-kFoldRadix tree.  finish: log(delta' M 1) + e ln 2
// into res[0..B) and status into res[B..2B); else the root node of each
// proposal into (out_m [B][KP][KP], out_e [B]).
// Node (b, i) at in_m + i*m_si + b*m_sb doubles, exponent at in_e[i*e_si + b*e_sb].
void run_tree(Workspace& ws, int K, int B, const double* in_m, const double* in_e, int64_t m_si, int64_t m_sb,
              int64_t e_si, int64_t e_sb, int64_t n0, const double* delta, bool finish, double* res,
              double* out_m, double* out_e, cudaStream_t s) {
  const int KP = padded(K), NT = KP / 8;
  thmm::TreeArgs ta{};
  ta.in_m = in_m;
  ta.in_e = in_e;
  ta.m_stride_i = m_si;
  ta.m_stride_b = m_sb;
  ta.e_stride_i = e_si;
  ta.e_stride_b = e_sb;
  ta.radix = kFoldRadix;
  ta.count[0] = n0;
  int levels = 0;
  do {
    if (levels >= thmm::kTreeMaxLevels) throw CudaError{cudaErrorInvalidValue, "segment tree too deep"};
    ta.count[levels + 1] = (ta.count[levels] + kFoldRadix - 1) / kFoldRadix;
    ++levels;
  } while (ta.count[levels] > 1);
  ta.levels = levels;
  int64_t nodes = 0, ctrs = 0;
  for (int l = 1; l < levels; ++l) {
    ta.off[l] = nodes;
    nodes += ta.count[l] * B;
  }
  for (int l = 2; l <= levels; ++l) {
    ta.cnt_off[l] = ctrs;
    ctrs += ta.count[l] * B;
  }
  const size_t node_bytes = static_cast<size_t>(KP) * KP * sizeof(double);
  ta.scratch_m = static_cast<double*>(ws.nodes_b.ensure(std::max<int64_t>(nodes, 1) * node_bytes));
  ta.scratch_e = static_cast<double*>(ws.exps_b.ensure(std::max<int64_t>(nodes, 1) * sizeof(double)));
  const size_t ctr_bytes = std::max<int64_t>(ctrs, 1) * sizeof(unsigned);
  if (ctr_bytes > ws.counters.cap) {
    ws.counters.ensure(ctr_bytes);
    THMM_CUDA(cudaMemsetAsync(ws.counters.ptr, 0, ws.counters.cap, s));
  }
  ta.counters = static_cast<unsigned*>(ws.counters.ptr);
  ta.K = K;
  ta.B = B;
  ta.finish = finish ? 1 : 0;
  ta.delta = delta;
  ta.loglik = res;
  ta.status = res ? reinterpret_cast<int32_t*>(res + B) : nullptr;
  ta.out_m = out_m;
  ta.out_e = out_e;
  THMM_DISPATCH(NT, skip_h1(K), launch_tree, ta, s);
}

cudaStream_t chunk_stream(thmm_obs obs, int c) {
  if (!obs->params_ready) THMM_CUDA(cudaEventCreateWithFlags(&obs->params_ready, cudaEventDisableTiming));
  if (!obs->chunk_streams[c]) THMM_CUDA(cudaStreamCreateWithFlags(&obs->chunk_streams[c], cudaStreamNonBlocking));
  if (!obs->chunk_done[c]) THMM_CUDA(cudaEventCreateWithFlags(&obs->chunk_done[c], cudaEventDisableTiming));
  return obs->chunk_streams[c];
}

// Runs the chain over [lo, hi) for all proposals and folds the segments.
// finish: write loglik/status to ws.result; else write one node per
// proposal to (out_m, out_e).
// chunks > 1 (host-array pipeline): the range is cut into `chunks`
// contiguous sub-ranges, each reduced by its own chain launch once ready[c]
// (the host->device copy of its records) has fired, so the copy of chunk
// c+1 overlaps the tensor work of chunk c; all segment nodes feed one tree.
void run_range(thmm_obs obs, const thmm_params* P, const thmm_config* cfg, cudaStream_t s, bool finish,
               double* out_m, double* out_e, int chunks = 1, const cudaEvent_t* ready = nullptr,
               const int64_t* chunk_bounds = nullptr) {
  const int K = P->K, B = P->B, KP = padded(K);
  const ChainPlan& plan = plan_for(obs->device, K, cfg->precision);
  ensure_fold(obs->device, K);
  const int64_t lo = cfg->lo, hi = cfg->hi > 0 ? cfg->hi : obs->n;
  const int64_t n = hi - lo;
  chunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(chunks, n)));
  int64_t c_nseg[8], c_lo[8], c_n[8], total = 0;
  for (int c = 0; c < chunks; ++c) {
    const int64_t base = n / chunks, rem = n % chunks;
    c_lo[c] = chunk_bounds ? chunk_bounds[c] : c * base + std::min<int64_t>(c, rem);
    c_n[c] = chunk_bounds ? chunk_bounds[c + 1] - chunk_bounds[c] : base + (c < rem ? 1 : 0);
    c_nseg[c] = cfg->segments > 0 ? std::min<int64_t>(cfg->segments, c_n[c]) : auto_segments(plan, c_n[c], B);
    total += c_nseg[c];
  }
  Workspace& ws = obs->ws;
  thmm::StateParams sp = upload_params(ws, P, s);

  const size_t node_bytes = static_cast<size_t>(KP) * KP * sizeof(double);
  double* seg_m = static_cast<double*>(ws.nodes_a.ensure(node_bytes * B * total));
  double* seg_e = static_cast<double*>(ws.exps_a.ensure(sizeof(double) * B * total));

  thmm::ChainArgs ca{};
  ca.present = obs->present;
  ca.lon = obs->lon;
  ca.lat = obs->lat;
  ca.K = K;
  ca.B = B;
  ca.G = plan.G;
  ca.period = cfg->renorm_period;
  ca.neg_log_2pi = -std::log(2.0 * M_PI);
  ca.P = sp;
  ca.seg_m = seg_m;
  ca.seg_e = seg_e;
  ca.node_stride_b = total;
  ca.x3 = tc_mode(cfg->precision);
  g_prof_segments = total;
  const bool prof = g_profile && prof_events(obs->device);
  if (prof) THMM_CUDA(record_prof(g_prof_ev[0], s));
  int64_t offset = 0;
  for (int c = 0; c < chunks; ++c) {
    ca.lo = lo + c_lo[c];
    ca.n = c_n[c];
    ca.nseg = c_nseg[c];
    ca.node_offset = offset;
    if (ready && chunks > 1) {
      // Each chunk's chain on its own stream, behind its copy and the
      // parameter upload, so the kernels of consecutive chunks overlap
      // (no per-launch tail); the tree waits for all of them.
      cudaStream_t cs = chunk_stream(obs, c);
      if (c == 0) THMM_CUDA(cudaEventRecord(obs->params_ready, s));
      THMM_CUDA(cudaStreamWaitEvent(cs, obs->params_ready, 0));
      THMM_CUDA(cudaStreamWaitEvent(cs, ready[c], 0));
      launch_chain(ca, plan, cfg->precision, (c_nseg[c] + plan.G - 1) / plan.G, cs);
      THMM_CUDA(cudaEventRecord(obs->chunk_done[c], cs));
    } else {
      if (ready) THMM_CUDA(cudaStreamWaitEvent(s, ready[c], 0));
      launch_chain(ca, plan, cfg->precision, (c_nseg[c] + plan.G - 1) / plan.G, s);
    }
    offset += c_nseg[c];
  }
  if (ready && chunks > 1)
    for (int c = 0; c < chunks; ++c) THMM_CUDA(cudaStreamWaitEvent(s, obs->chunk_done[c], 0));
  if (prof) THMM_CUDA(record_prof(g_prof_ev[1], s));

  double* res = nullptr;
  if (finish) res = static_cast<double*>(ws.result.ensure(2 * sizeof(double) * B));

  const int64_t nd = static_cast<int64_t>(KP) * KP;
  run_tree(ws, K, B, seg_m, seg_e, nd, total * nd, 1, total, total, sp.delta, finish, res, out_m, out_e, s);
  if (prof) THMM_CUDA(record_prof(g_prof_ev[2], s));
}

// Called after the stream was synchronised.
void prof_collect() {
  if (!g_profile || g_prof_ev_device < 0) return;
  float a = 0.f, b = 0.f;
  if (cudaEventElapsedTime(&a, g_prof_ev[0], g_prof_ev[1]) == cudaSuccess &&
      cudaEventElapsedTime(&b, g_prof_ev[1], g_prof_ev[2]) == cudaSuccess) {
    g_prof_chain_ms = a;
    g_prof_fold_ms = b;
  } else {
    cudaGetLastError();
  }
}

// Results (loglik[B] | status[B]) land in the head of the pinned staging
// buffer (the parameter upload that used it is stream-ordered before).
void enqueue_results(Workspace& ws, int B, cudaStream_t s) {
  double* res = static_cast<double*>(ws.result.ptr);
  double* host = static_cast<double*>(ws.staging.ensure(2 * sizeof(double) * B));
  THMM_CUDA(cudaMemcpyAsync(host, res, 2 * sizeof(double) * B, cudaMemcpyDeviceToHost, s));
}

int read_results(Workspace& ws, int B, cudaStream_t s, double* out, int32_t* status) {
  THMM_CUDA(cudaStreamSynchronize(s));
  const double* host = static_cast<const double*>(ws.staging.ptr);
  const int32_t* st = reinterpret_cast<const int32_t*>(host + B);
  int rc = THMM_OK;
  for (int b = 0; b < B; ++b) {
    out[b] = host[b];
    if (status) status[b] = st[b] ? THMM_ECOLLAPSE : THMM_OK;
    if (st[b]) rc = THMM_ECOLLAPSE;
  }
  return rc;
}

uintptr_t workspace_signature(thmm_obs obs) {
  const Workspace& w = obs->ws;
  uintptr_t h = 1469598103934665603ull;
  const void* ptrs[] = {obs->present, obs->lon, obs->lat, w.params.ptr, w.nodes_a.ptr, w.nodes_b.ptr,
                        w.exps_a.ptr, w.exps_b.ptr, w.result.ptr, w.counters.ptr, w.staging.ptr};
  for (const void* p : ptrs) h = (h ^ reinterpret_cast<uintptr_t>(p)) * 1099511628211ull;
  return h;
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("THMM_GRAPHS");
    return !(v && v[0] == '0');
  }();
  return on;
}

// Record the evaluation just performed (same configuration, buffers already
// sized) as a CUDA graph on the handle's own stream; replayed by later calls.
void capture_graph(thmm_obs obs, const thmm_params* P, const thmm_config* cfg, int64_t hi, bool prof) {
  thmm_obs_s::Graph* slot = &obs->graphs[0];
  for (auto& g : obs->graphs) {
    if (!g.valid) {
      slot = &g;
      break;
    }
    if (g.last_use < slot->last_use) slot = &g;
  }
  if (slot->valid) {
    cudaGraphExecDestroy(slot->exec);
    slot->valid = false;
  }
  const int saved_launches = g_launches;
  const uintptr_t sig = workspace_signature(obs);
  cudaStream_t cs = obs->stream;
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  bool ok = true;
  g_capturing = true;
  try {
    run_range(obs, P, cfg, cs, true, nullptr, nullptr);
    enqueue_results(obs->ws, P->B, cs);
  } catch (const CudaError&) {
    ok = false;
  }
  g_capturing = false;
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(cs, &graph);
  g_launches = saved_launches;
  if (!ok || e != cudaSuccess || graph == nullptr || workspace_signature(obs) != sig) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    return;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  slot->K = P->K;
  slot->B = P->B;
  slot->precision = cfg->precision;
  slot->period = cfg->renorm_period;
  slot->segments = cfg->segments;
  slot->lo = cfg->lo;
  slot->hi = hi;
  slot->prof = prof;
  slot->signature = sig;
  slot->nseg = g_prof_segments;
  slot->exec = exec;
  slot->last_use = ++obs->uses;
  slot->valid = true;
}

int finish_results(Workspace& ws, int B, cudaStream_t s, double* out, int32_t* status) {
  enqueue_results(ws, B, s);
  return read_results(ws, B, s, out, status);
}

int translate(const CudaError& e, char* err, size_t errlen) {
  set_err(err, errlen, "CUDA error %s (%s) in %s", cudaGetErrorName(e.code), cudaGetErrorString(e.code), e.what);
  return THMM_ECUDA;
}

int check_cfg(thmm_obs obs, const thmm_config* cfg, char* err, size_t errlen) {
  if (!cfg) {
    set_err(err, errlen, "config must be non-NULL");
    return THMM_EINVAL;
  }
  if (cfg->renorm_period < 1) {
    set_err(err, errlen, "renorm_period must be a positive integer");
    return THMM_EINVAL;
  }
  if (cfg->precision < THMM_F64 || cfg->precision > THMM_TF32X2) {
    set_err(err, errlen, "precision must be float64, float32, tf32, tf32x3 or tf32x2");
    return THMM_EINVAL;
  }
  if (cfg->segments < 0) {
    set_err(err, errlen, "segments must be positive when given");
    return THMM_EINVAL;
  }
  const int64_t hi = cfg->hi > 0 ? cfg->hi : obs->n;
  if (cfg->lo < 0 || hi > obs->n || cfg->lo >= hi) {
    set_err(err, errlen, "observation range [%lld, %lld) is empty or outside the stream of %lld records",
            (long long)cfg->lo, (long long)hi, (long long)obs->n);
    return THMM_EINVAL;
  }
  return THMM_OK;
}

void ensure_obs_capacity(thmm_obs obs, int64_t n) {
  if (n <= obs->cap) return;
  if (obs->present) cudaFree(obs->present);
  if (obs->lon) cudaFree(obs->lon);
  if (obs->lat) cudaFree(obs->lat);
  obs->present = nullptr;
  obs->lon = obs->lat = nullptr;
  obs->cap = 0;
  THMM_CUDA(cudaMalloc(&obs->present, n));
  THMM_CUDA(cudaMalloc(&obs->lon, n * sizeof(double)));
  THMM_CUDA(cudaMalloc(&obs->lat, n * sizeof(double)));
  obs->cap = n;
}

int upload_obs(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
               cudaMemcpyKind kind, char* err, size_t errlen) {
  if (n < 1) {
    set_err(err, errlen, "observation sequence is empty");
    return THMM_EINVAL;
  }
  if (!present || !lon || !lat) {
    set_err(err, errlen, "observation pointers must be non-NULL");
    return THMM_EINVAL;
  }
  DeviceGuard dg(obs->device);
  // an asynchronous call on another stream may still be reading the records
  if (obs->ws.staged_pending && obs->ws.staged) THMM_CUDA(cudaStreamWaitEvent(obs->stream, obs->ws.staged, 0));
  ensure_obs_capacity(obs, n);
  THMM_CUDA(cudaMemcpyAsync(obs->present, present, n, kind, obs->stream));
  THMM_CUDA(cudaMemcpyAsync(obs->lon, lon, n * sizeof(double), kind, obs->stream));
  THMM_CUDA(cudaMemcpyAsync(obs->lat, lat, n * sizeof(double), kind, obs->stream));
  obs->n = n;
  return THMM_OK;
}

cudaStream_t pick_stream(thmm_obs obs, const thmm_config* cfg) {
  return cfg && cfg->stream ? static_cast<cudaStream_t>(cfg->stream) : obs->stream;
}

// Global per-device workspace for calls without a handle (fold_nodes,
// factor segments).
std::mutex g_ws_mu;
Workspace g_ws[64];

}  // namespace

extern "C" {

int thmm_version(void) { return 100; }

int thmm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int thmm_padded_states(int32_t K) { return padded(K); }

int thmm_last_launch_count(void) { return g_launches; }

int thmm_profile_enable(int on) {
  g_profile = on != 0;
  return THMM_OK;
}

int thmm_profile_last(double* chain_ms, double* fold_ms, int64_t* segments) {
  if (chain_ms) *chain_ms = g_prof_chain_ms;
  if (fold_ms) *fold_ms = g_prof_fold_ms;
  if (segments) *segments = g_prof_segments;
  return THMM_OK;
}

int thmm_plan_info(int32_t K, int32_t precision, int device, int32_t* nt, int32_t* tail, int32_t* G, int32_t* W,
                   int32_t* regs, int32_t* ctas_per_sm) {
  if (K < 1 || K > THMM_MAX_STATES || precision < THMM_F64 || precision > THMM_TF32X2) return THMM_EINVAL;
  if (device < 0 || device >= thmm_device_count()) return THMM_ECUDA;
  try {
    DeviceGuard dg(device);
    const ChainPlan& p = plan_for(device, K, precision);
    if (nt) *nt = p.nt;
    if (tail) *tail = p.tail;
    if (G) *G = p.G;
    if (W) *W = p.W;
    if (regs) *regs = p.regs;
    if (ctas_per_sm) *ctas_per_sm = p.ctas_per_sm;
    return THMM_OK;
  } catch (const CudaError&) {
    return THMM_ECUDA;
  }
}

int thmm_obs_create(const uint8_t* present, const double* lon, const double* lat, int64_t n, int device,
                    thmm_obs* out, char* err, size_t errlen) {
  g_launches = 0;
  if (!out) {
    set_err(err, errlen, "out must be non-NULL");
    return THMM_EINVAL;
  }
  *out = nullptr;
  if (n < 1) {
    set_err(err, errlen, "observation sequence is empty");
    return THMM_EINVAL;
  }
  const int ndev = thmm_device_count();
  if (device < 0 || device >= ndev) {
    set_err(err, errlen, "CUDA device %d not available (%d visible)", device, ndev);
    return THMM_ECUDA;
  }
  thmm_obs obs = new thmm_obs_s();
  obs->device = device;
  try {
    DeviceGuard dg(device);
    THMM_CUDA(cudaStreamCreateWithFlags(&obs->stream, cudaStreamNonBlocking));
    int rc = upload_obs(obs, present, lon, lat, n, cudaMemcpyHostToDevice, err, errlen);
    if (rc == THMM_OK) THMM_CUDA(cudaStreamSynchronize(obs->stream));
    if (rc != THMM_OK) {
      thmm_obs_destroy(obs);
      return rc;
    }
  } catch (const CudaError& e) {
    thmm_obs_destroy(obs);
    return translate(e, err, errlen);
  }
  *out = obs;
  return THMM_OK;
}

int thmm_obs_assign(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                    char* err, size_t errlen) {
  g_launches = 0;
  if (!obs) {
    set_err(err, errlen, "null observation handle");
    return THMM_EINVAL;
  }
  std::lock_guard<std::mutex> lk(obs->mu);
  try {
    int rc = upload_obs(obs, present, lon, lat, n, cudaMemcpyHostToDevice, err, errlen);
    if (rc == THMM_OK) THMM_CUDA(cudaStreamSynchronize(obs->stream));
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

int thmm_obs_assign_device(thmm_obs obs, const uint8_t* d_present, const double* d_lon, const double* d_lat,
                           int64_t n, char* err, size_t errlen) {
  g_launches = 0;
  if (!obs) {
    set_err(err, errlen, "null observation handle");
    return THMM_EINVAL;
  }
  std::lock_guard<std::mutex> lk(obs->mu);
  try {
    int rc = upload_obs(obs, d_present, d_lon, d_lat, n, cudaMemcpyDeviceToDevice, err, errlen);
    if (rc == THMM_OK) THMM_CUDA(cudaStreamSynchronize(obs->stream));
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

int thmm_obs_destroy(thmm_obs obs) {
  if (!obs) return THMM_OK;
  {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(obs->device);
    if (obs->stream) cudaStreamSynchronize(obs->stream);
    if (obs->ws.staged) cudaEventSynchronize(obs->ws.staged);  // last asynchronous call
    if (obs->reads_done) cudaEventDestroy(obs->reads_done);
    for (int c = 0; c < 8; ++c) {
      if (obs->chunk_streams[c]) cudaStreamSynchronize(obs->chunk_streams[c]), cudaStreamDestroy(obs->chunk_streams[c]);
      if (obs->chunk_done[c]) cudaEventDestroy(obs->chunk_done[c]);
    }
    if (obs->params_ready) cudaEventDestroy(obs->params_ready);
    for (auto& g : obs->graphs)
      if (g.valid) cudaGraphExecDestroy(g.exec);
    for (auto& g : obs->host_graphs)
      if (g.valid) cudaGraphExecDestroy(g.exec);
    for (auto& e : obs->chunk_ready)
      if (e) cudaEventDestroy(e);
    if (obs->copy_stream) cudaStreamDestroy(obs->copy_stream);
    if (obs->present) cudaFree(obs->present);
    if (obs->lon) cudaFree(obs->lon);
    if (obs->lat) cudaFree(obs->lat);
    obs->ws.release();
    if (obs->stream) cudaStreamDestroy(obs->stream);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete obs;
  return THMM_OK;
}

int64_t thmm_obs_length(thmm_obs obs) { return obs ? obs->n : -1; }
int thmm_obs_device(thmm_obs obs) { return obs ? obs->device : -1; }

int thmm_loglik(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, double* out, int32_t* status,
                char* err, size_t errlen) {
  g_launches = 0;
  if (!obs || !out) {
    set_err(err, errlen, "null observation handle or output");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  std::lock_guard<std::mutex> lk(obs->mu);
  rc = check_cfg(obs, cfg, err, errlen);
  if (rc != THMM_OK) return rc;
  try {
    DeviceGuard dg(obs->device);
    cudaStream_t s = pick_stream(obs, cfg);
    const int64_t hi = cfg->hi > 0 ? cfg->hi : obs->n;
    const bool prof = g_profile;
    thmm_obs_s::Graph* hit = nullptr;
    if (graphs_enabled()) {
      for (auto& gr : obs->graphs)
        if (gr.valid && gr.K == params->K && gr.B == params->B && gr.precision == cfg->precision &&
            gr.period == cfg->renorm_period && gr.segments == cfg->segments && gr.lo == cfg->lo && gr.hi == hi &&
            gr.prof == prof && gr.signature == workspace_signature(obs))
          hit = &gr;
    }
    if (hit) {
      // Replay: stage the new parameters where the captured H2D copy reads them.
      stage_params_host(obs->ws, params);
      hit->last_use = ++obs->uses;
      THMM_CUDA(cudaGraphLaunch(hit->exec, s));
      g_launches = 2;
      g_prof_segments = hit->nseg;
      rc = read_results(obs->ws, params->B, s, out, status);
    } else {
      run_range(obs, params, cfg, s, true, nullptr, nullptr);
      rc = finish_results(obs->ws, params->B, s, out, status);
      if (graphs_enabled()) capture_graph(obs, params, cfg, hi, prof);
    }
    prof_collect();
    if (rc == THMM_ECOLLAPSE)
      set_err(err, errlen, "running state vector collapsed to zero while combining segments");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

namespace {

// Queue the host->device copy of n host records on the handle's copy stream
// in geometric chunks (event chunk_ready[c] per chunk) behind everything
// already queued on the launch stream s (so a previous asynchronous call has
// finished reading the device buffers).  Fills bounds[0..chunks]; returns chunks.
int enqueue_host_chunks(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                        const thmm_params* params, const thmm_config* cfg, cudaStream_t s, int64_t* bounds) {
    if (!obs->copy_stream) THMM_CUDA(cudaStreamCreateWithFlags(&obs->copy_stream, cudaStreamNonBlocking));
    for (auto& e : obs->chunk_ready)
      if (!e) THMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!obs->reads_done) THMM_CUDA(cudaEventCreateWithFlags(&obs->reads_done, cudaEventDisableTiming));
    THMM_CUDA(cudaEventRecord(obs->reads_done, s));
    THMM_CUDA(cudaStreamWaitEvent(obs->copy_stream, obs->reads_done, 0));
    // Geometric chunks: chunk c+1 is R times chunk c, R ~ (copy rate / chain
    // rate), so each chunk's copy finishes while the previous chunk's chain
    // runs and the GPU waits only for the (small) first chunk; few chunks
    // keep the per-launch tails few.  Whole-stream evaluations only (ranges
    // and explicit segment counts keep the single-launch schedule).
    const bool whole = cfg->lo == 0 && (cfg->hi == 0 || cfg->hi == n) && cfg->segments == 0;
    std::fill(bounds, bounds + 9, int64_t{0});
    int chunks = 1;
    bounds[1] = n;
    if (whole && n >= 2 * kMinFirstChunk) {
      const double chain_rate = 25e12 / (2.0 * params->K * params->K * params->K * params->B);  // records/s
      const double copy_rate = 45e9 / 17.0;                                                     // records/s
      const double R = std::min(8.0, std::max(2.0, copy_rate / chain_rate));
      int C = 1;
      double sum = 1.0, term = 1.0;
      while (C < 8) {  // largest chunk count whose first chunk stays >= kMinFirstChunk
        const double next_sum = sum + term * R;
        if (static_cast<double>(n) / next_sum < kMinFirstChunk) break;
        term *= R;
        sum = next_sum;
        ++C;
      }
      chunks = C;
      double acc = 0.0, t = 1.0;
      for (int c = 0; c < C; ++c) {
        bounds[c] = static_cast<int64_t>(std::llround(static_cast<double>(n) * acc / sum));
        acc += t;
        t *= R;
      }
      bounds[C] = n;
    }
    for (int c = 0; c < chunks; ++c) {
      const int64_t lo = bounds[c], cnt = bounds[c + 1] - bounds[c];
      THMM_CUDA(cudaMemcpyAsync(obs->present + lo, present + lo, cnt, cudaMemcpyHostToDevice, obs->copy_stream));
      THMM_CUDA(cudaMemcpyAsync(obs->lon + lo, lon + lo, cnt * sizeof(double), cudaMemcpyHostToDevice,
                                obs->copy_stream));
      THMM_CUDA(cudaMemcpyAsync(obs->lat + lo, lat + lo, cnt * sizeof(double), cudaMemcpyHostToDevice,
                                obs->copy_stream));
      THMM_CUDA(cudaEventRecord(obs->chunk_ready[c], obs->copy_stream));
    }
    return chunks;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Record the host-array evaluation just performed (chunked copies on the copy
// stream, per-chunk chains on their streams, tree, result copy) as a CUDA
// graph; later calls with the same pinned buffers, sizes and configuration
// replay it after restaging the parameters.
void capture_host_graph(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                        const thmm_params* P, const thmm_config* cfg, cudaStream_t s, bool prof) {
  thmm_obs_s::HostGraph* slot = &obs->host_graphs[0];
  for (auto& g : obs->host_graphs) {
    if (!g.valid) {
      slot = &g;
      break;
    }
    if (g.last_use < slot->last_use) slot = &g;
  }
  if (slot->valid) {
    cudaGraphExecDestroy(slot->exec);
    slot->valid = false;
  }
  const int saved_launches = g_launches;
  const uintptr_t sig = workspace_signature(obs);
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  bool ok = true;
  g_capturing = true;
  g_launches = 0;
  try {
    int64_t bounds[9];
    const int chunks = enqueue_host_chunks(obs, present, lon, lat, n, P, cfg, s, bounds);
    run_range(obs, P, cfg, s, true, nullptr, nullptr, chunks, obs->chunk_ready, bounds);
    enqueue_results(obs->ws, P->B, s);
  } catch (const CudaError&) {
    ok = false;
  }
  g_capturing = false;
  const int launches = g_launches;
  g_launches = saved_launches;
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(s, &graph);
  if (!ok || e != cudaSuccess || graph == nullptr || workspace_signature(obs) != sig) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    return;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  slot->src[0] = present;
  slot->src[1] = lon;
  slot->src[2] = lat;
  slot->n = n;
  slot->K = P->K;
  slot->B = P->B;
  slot->precision = cfg->precision;
  slot->period = cfg->renorm_period;
  slot->segments = cfg->segments;
  slot->prof = prof;
  slot->signature = sig;
  slot->nseg = g_prof_segments;
  slot->launches = launches;
  slot->exec = exec;
  slot->last_use = ++obs->uses;
  slot->valid = true;
}

}  // namespace

int thmm_loglik_host(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                     const thmm_params* params, const thmm_config* cfg, double* out, int32_t* status, char* err,
                     size_t errlen) {
  g_launches = 0;
  if (!obs || !out) {
    set_err(err, errlen, "null observation handle or output");
    return THMM_EINVAL;
  }
  if (n < 1) {
    set_err(err, errlen, "observation sequence is empty");
    return THMM_EINVAL;
  }
  if (!present || !lon || !lat) {
    set_err(err, errlen, "observation pointers must be non-NULL");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  std::lock_guard<std::mutex> lk(obs->mu);
  try {
    DeviceGuard dg(obs->device);
    ensure_obs_capacity(obs, n);
    obs->n = n;
    rc = check_cfg(obs, cfg, err, errlen);
    if (rc != THMM_OK) return rc;
    cudaStream_t s = pick_stream(obs, cfg);
    const bool prof = g_profile;
    // Replay the recorded pipeline (copies from the same pinned host buffers,
    // chunk chains, tree, result copy) when this call repeats an earlier one.
    thmm_obs_s::HostGraph* hit = nullptr;
    const bool graphable = graphs_enabled() && s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread &&
                           is_pinned(present) && is_pinned(lon) && is_pinned(lat);
    if (graphable) {
      const uintptr_t sig = workspace_signature(obs);
      for (auto& g : obs->host_graphs)
        if (g.valid && g.src[0] == present && g.src[1] == lon && g.src[2] == lat && g.n == n && g.K == params->K &&
            g.B == params->B && g.precision == cfg->precision && g.period == cfg->renorm_period &&
            g.segments == cfg->segments && g.prof == prof && g.signature == sig)
          hit = &g;
    }
    if (hit) {
      stage_params_host(obs->ws, params);
      hit->last_use = ++obs->uses;
      THMM_CUDA(cudaGraphLaunch(hit->exec, s));
      g_launches = hit->launches;
      g_prof_segments = hit->nseg;
      rc = read_results(obs->ws, params->B, s, out, status);
    } else {
      int64_t bounds[9];
      const int chunks = enqueue_host_chunks(obs, present, lon, lat, n, params, cfg, s, bounds);
      run_range(obs, params, cfg, s, true, nullptr, nullptr, chunks, obs->chunk_ready, bounds);
      rc = finish_results(obs->ws, params->B, s, out, status);
      if (graphable) capture_host_graph(obs, present, lon, lat, n, params, cfg, s, prof);
    }
    prof_collect();
    if (rc == THMM_ECOLLAPSE)
      set_err(err, errlen, "running state vector collapsed to zero while combining segments");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

namespace {

int range_nodes_impl(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, double* d_m, double* d_e,
                     bool sync, char* err, size_t errlen) {
  g_launches = 0;
  if (!obs || !d_m || !d_e) {
    set_err(err, errlen, "null observation handle or output");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  std::lock_guard<std::mutex> lk(obs->mu);
  rc = check_cfg(obs, cfg, err, errlen);
  if (rc != THMM_OK) return rc;
  try {
    DeviceGuard dg(obs->device);
    cudaStream_t s = pick_stream(obs, cfg);
    run_range(obs, params, cfg, s, false, d_m, d_e);
    if (sync) {
      THMM_CUDA(cudaStreamSynchronize(s));
      prof_collect();
    } else {
      // the next upload into the pinned staging buffer waits for this one
      THMM_CUDA(cudaEventRecord(staged_event(obs->ws), s));
    }
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

}  // namespace

int thmm_range_nodes(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, double* d_m, double* d_e,
                     char* err, size_t errlen) {
  return range_nodes_impl(obs, params, cfg, d_m, d_e, true, err, errlen);
}

int thmm_range_nodes_async(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, double* d_m,
                           double* d_e, char* err, size_t errlen) {
  return range_nodes_impl(obs, params, cfg, d_m, d_e, false, err, errlen);
}

int thmm_range_nodes_host(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                          const thmm_params* params, const thmm_config* cfg, double* d_m, double* d_e, char* err,
                          size_t errlen) {
  g_launches = 0;
  if (!obs || !d_m || !d_e) {
    set_err(err, errlen, "null observation handle or output");
    return THMM_EINVAL;
  }
  if (n < 1) {
    set_err(err, errlen, "observation sequence is empty");
    return THMM_EINVAL;
  }
  if (!present || !lon || !lat) {
    set_err(err, errlen, "observation pointers must be non-NULL");
    return THMM_EINVAL;
  }
  if (cfg && (cfg->lo != 0 || cfg->hi != 0)) {
    set_err(err, errlen, "host-array ranges cover the whole (replaced) stream");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  std::lock_guard<std::mutex> lk(obs->mu);
  try {
    DeviceGuard dg(obs->device);
    ensure_obs_capacity(obs, n);
    obs->n = n;
    rc = check_cfg(obs, cfg, err, errlen);
    if (rc != THMM_OK) return rc;
    cudaStream_t s = pick_stream(obs, cfg);
    int64_t bounds[9];
    const int chunks = enqueue_host_chunks(obs, present, lon, lat, n, params, cfg, s, bounds);
    run_range(obs, params, cfg, s, false, d_m, d_e, chunks, obs->chunk_ready, bounds);
    THMM_CUDA(cudaEventRecord(staged_event(obs->ws), s));
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

int thmm_filtered_state(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, double* out,
                        int32_t* status, char* err, size_t errlen) {
  g_launches = 0;
  if (!obs || !out) {
    set_err(err, errlen, "null observation handle or output");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  std::lock_guard<std::mutex> lk(obs->mu);
  rc = check_cfg(obs, cfg, err, errlen);
  if (rc != THMM_OK) return rc;
  try {
    DeviceGuard dg(obs->device);
    cudaStream_t s = pick_stream(obs, cfg);
    const int K = params->K, B = params->B, KP = padded(K);
    const size_t node = static_cast<size_t>(KP) * KP;
    // root nodes of the whole range, one per proposal, in a dedicated buffer
    double* d_root = static_cast<double*>(obs->ws.result.ensure((node + 1) * B * sizeof(double)));
    run_range(obs, params, cfg, s, false, d_root, d_root + node * B);
    std::vector<double> host((node + 1) * B);
    THMM_CUDA(cudaMemcpyAsync(host.data(), d_root, host.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    THMM_CUDA(cudaStreamSynchronize(s));
    // v = delta' M (normalised), then one transition: (v Gamma) / sum  (reference
    // simforecast._filtered_next_state_dist, simforecast.py:97-118)
    std::vector<double> v(K);
    for (int b = 0; b < B; ++b) {
      const double* m = host.data() + node * b;
      const double* delta = params->delta + static_cast<size_t>(b) * K;
      const double* gamma = params->gamma + static_cast<size_t>(b) * K * K;
      double sum = 0.0;
      for (int c = 0; c < K; ++c) {
        double acc = 0.0;
        for (int r = 0; r < K; ++r) acc += delta[r] * m[r * KP + c];
        v[c] = acc;
        sum += acc;
      }
      double* o = out + static_cast<size_t>(b) * K;
      bool ok = sum > 0.0 && std::isfinite(sum);
      double s2 = 0.0;
      for (int c = 0; c < K && ok; ++c) {
        double acc = 0.0;
        for (int r = 0; r < K; ++r) acc += (v[r] / sum) * gamma[r * K + c];
        o[c] = acc;
        s2 += acc;
      }
      ok = ok && s2 > 0.0;
      for (int c = 0; c < K; ++c) o[c] = ok ? o[c] / s2 : std::nan("");
      if (status) status[b] = ok ? THMM_OK : THMM_ECOLLAPSE;
      if (!ok) rc = THMM_ECOLLAPSE;
    }
    if (rc == THMM_ECOLLAPSE) set_err(err, errlen, "history has zero likelihood under these parameters");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

namespace {

int fold_nodes_impl(const thmm_params* params, int32_t G, const double* d_m, int64_t m_stride_g,
                    const double* d_e, int64_t e_stride_g, int device, void* stream, double* out,
                    int32_t* status, char* err, size_t errlen) {
  g_launches = 0;
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  if (G < 1 || !d_m || !d_e || !out) {
    set_err(err, errlen, "no segment products to combine");
    return THMM_EINVAL;
  }
  if ((reinterpret_cast<uintptr_t>(d_m) & 15) || (G > 1 && (m_stride_g & 1))) {
    set_err(err, errlen, "node matrices must be 16-byte aligned (even node stride)");
    return THMM_EINVAL;
  }
  if (device < 0 || device >= thmm_device_count()) {
    set_err(err, errlen, "CUDA device %d not available", device);
    return THMM_ECUDA;
  }
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Workspace& ws = g_ws[device & 63];
  try {
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int K = params->K, B = params->B, KP = padded(K);
    ensure_fold(device, K);
    thmm::StateParams sp = upload_params(ws, params, s);
    double* res = static_cast<double*>(ws.result.ensure(2 * sizeof(double) * B));
    run_tree(ws, K, B, d_m, d_e, m_stride_g, static_cast<int64_t>(KP) * KP, e_stride_g, 1, G, sp.delta, true, res,
             nullptr, nullptr, s);
    rc = finish_results(ws, B, s, out, status);
    prof_collect();  // chain/tree events of this thread's last thmm_range_nodes_async, now complete
    if (rc == THMM_ECOLLAPSE)
      set_err(err, errlen, "running state vector collapsed to zero while combining segments");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

}  // namespace

int thmm_fold_nodes(const thmm_params* params, int32_t G, const double* d_m, const double* d_e, int device,
                    void* stream, double* out, int32_t* status, char* err, size_t errlen) {
  // nodes arrive as [G][B]: node (g, b) at (g*B + b)
  const int64_t B = params ? params->B : 0, KP = params ? padded(params->K) : 0;
  return fold_nodes_impl(params, G, d_m, B * KP * KP, d_e, B, device, stream, out, status, err, errlen);
}

int thmm_fold_nodes_strided(const thmm_params* params, int32_t G, const double* d_m, int64_t m_stride_g,
                            const double* d_e, int64_t e_stride_g, int device, void* stream, double* out,
                            int32_t* status, char* err, size_t errlen) {
  return fold_nodes_impl(params, G, d_m, m_stride_g, d_e, e_stride_g, device, stream, out, status, err, errlen);
}

// ---------------------------------------------------------------------------
// Peer-memory combine over NVLink / NVSwitch (one process per GPU): every
// rank's root nodes are stored straight into every peer's mailbox by one
// publish kernel (P2P stores through CUDA IPC mappings) and announced with a
// release-ordered flag carrying the evaluation's epoch; a one-warp wait
// kernel acquires all flags, and the segment tree folds the world's nodes in
// rank order from local memory.  No collective library call, no host
// synchronisation before the result read.
// ---------------------------------------------------------------------------
}  // extern "C" (reopened below)

struct thmm_peer_s {
  int device = 0, rank = 0, world = 1;
  int64_t slot = 0;                     // doubles per (parity, rank) slot
  double* mailbox = nullptr;            // [2][world][slot] doubles, then [2][world] u64 flags
  double** peer_box = nullptr;          // device array: mailbox base of every rank
  std::vector<void*> opened;            // IPC mappings of the peers' mailboxes
  double* outbox = nullptr;             // this rank's root nodes [slot]
  double* foldbuf = nullptr;            // the world's nodes, rank order [world][slot]
  unsigned long long* d_epoch = nullptr;  // completed exchanges (device-resident: graph replays advance it)
  int32_t* d_timeout = nullptr;
  int32_t* h_timeout = nullptr;         // pinned copy, read with the results
  // CUDA graph of the device-resident evaluation, replayed with new parameters
  struct {
    bool valid = false;
    int K = 0, B = 0, precision = 0, period = 0;
    int64_t segments = 0;
    bool prof = false;
    uintptr_t signature = 0;
    thmm_obs obs = nullptr;
    int launches = 0;
    int64_t nseg = 0;
    cudaGraphExec_t exec = nullptr;
  } graph;
};

namespace {

size_t peer_bytes(int world, int64_t slot) {
  return static_cast<size_t>(2) * world * slot * sizeof(double) + static_cast<size_t>(2) * world * 8;
}

// Publish this rank's nodes (outbox) into every rank's mailbox slot for the
// next epoch e = *epoch + 1 and release the epoch flag there.
__global__ void peer_publish_kernel(double* const* boxes, const double* outbox, int rank, int world, int64_t slot,
                                    int64_t count, const unsigned long long* epoch) {
  const unsigned long long e = *epoch + 1ull;
  const int parity = static_cast<int>(e & 1ull);
  const int p = blockIdx.x;  // destination rank
  double* base = boxes[p];
  double* dst = base + (static_cast<int64_t>(parity) * world + rank) * slot;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = outbox[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned long long* flag =
        reinterpret_cast<unsigned long long*>(base + static_cast<int64_t>(2) * world * slot) + parity * world + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(flag), "l"(e) : "memory");
  }
}

// Acquire every rank's flag for epoch e, copy the world's nodes (rank order)
// to the fold buffer, then advance *epoch.
__global__ void peer_wait_kernel(const double* box, double* foldbuf, int world, int64_t slot, int64_t count,
                                 unsigned long long* epoch, int32_t* timeout) {
  const unsigned long long e = *epoch + 1ull;
  const int parity = static_cast<int>(e & 1ull);
  const int r = threadIdx.x;
  if (r < world) {
    const unsigned long long* flag =
        reinterpret_cast<const unsigned long long*>(box + static_cast<int64_t>(2) * world * slot) + parity * world + r;
    const long long t0 = clock64();
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(flag) : "memory");
      if (v == e) break;
      if (clock64() - t0 > 8000000000LL) {  // ~4 s: a peer never published
        atomicOr(timeout, 1);
        break;
      }
      __nanosleep(200);
    }
  }
  __syncthreads();
  const double* src = box + static_cast<int64_t>(parity) * world * slot;
  for (int64_t i = threadIdx.x; i < static_cast<int64_t>(world) * slot; i += blockDim.x) foldbuf[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) *epoch = e;
}

}  // namespace

extern "C" {

int thmm_peer_create(int device, int rank, int world, int64_t slot_doubles, thmm_peer* out, void* ipc_handle,
                     char* err, size_t errlen) {
  if (!out || !ipc_handle || world < 1 || rank < 0 || rank >= world || slot_doubles < 1) {
    set_err(err, errlen, "invalid peer configuration");
    return THMM_EINVAL;
  }
  if (device < 0 || device >= thmm_device_count()) {
    set_err(err, errlen, "CUDA device %d not available", device);
    return THMM_ECUDA;
  }
  thmm_peer p = new thmm_peer_s;
  p->device = device;
  p->rank = rank;
  p->world = world;
  p->slot = slot_doubles + (slot_doubles & 1);  // 16-byte aligned slots (nodes are read as double2)
  try {
    DeviceGuard dg(device);
    THMM_CUDA(cudaMalloc(&p->mailbox, peer_bytes(world, p->slot)));
    THMM_CUDA(cudaMemset(p->mailbox, 0, peer_bytes(world, p->slot)));
    THMM_CUDA(cudaMalloc(&p->peer_box, sizeof(double*) * world));
    THMM_CUDA(cudaMalloc(&p->outbox, sizeof(double) * p->slot));
    THMM_CUDA(cudaMalloc(&p->foldbuf, sizeof(double) * p->slot * world));
    THMM_CUDA(cudaMalloc(&p->d_epoch, sizeof(unsigned long long)));
    THMM_CUDA(cudaMemset(p->d_epoch, 0, sizeof(unsigned long long)));
    THMM_CUDA(cudaMalloc(&p->d_timeout, sizeof(int32_t)));
    THMM_CUDA(cudaMemset(p->d_timeout, 0, sizeof(int32_t)));
    THMM_CUDA(cudaMallocHost(&p->h_timeout, sizeof(int32_t)));
    *p->h_timeout = 0;
    cudaIpcMemHandle_t h;
    THMM_CUDA(cudaIpcGetMemHandle(&h, p->mailbox));
    std::memcpy(ipc_handle, &h, sizeof(h));
    THMM_CUDA(cudaDeviceSynchronize());
  } catch (const CudaError& e) {
    thmm_peer_destroy(p);
    return translate(e, err, errlen);
  }
  *out = p;
  return THMM_OK;
}

int thmm_peer_open(thmm_peer p, const void* handles, char* err, size_t errlen) {
  if (!p || !handles) {
    set_err(err, errlen, "null peer or handles");
    return THMM_EINVAL;
  }
  try {
    DeviceGuard dg(p->device);
    std::vector<double*> boxes(p->world, nullptr);
    for (int r = 0; r < p->world; ++r) {
      if (r == p->rank) {
        boxes[r] = p->mailbox;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + static_cast<size_t>(r) * sizeof(h), sizeof(h));
      void* ptr = nullptr;
      THMM_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      p->opened.push_back(ptr);
      boxes[r] = static_cast<double*>(ptr);
    }
    THMM_CUDA(cudaMemcpy(p->peer_box, boxes.data(), sizeof(double*) * p->world, cudaMemcpyHostToDevice));
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

}  // extern "C" (reopened below)

namespace {

// One peer-combined evaluation on stream s: chain + tree into the outbox,
// publish, wait (+ copy the world's nodes to the fold buffer), fold, result
// and timeout-flag copies to pinned host memory.  Every pointer is fixed, so
// the whole sequence can be captured as a CUDA graph and replayed.
void enqueue_peer_eval(thmm_peer p, thmm_obs obs, const uint8_t* present, const double* lon, const double* lat,
                       int64_t n, const thmm_params* params, const thmm_config* cfg, cudaStream_t s) {
  const int K = params->K, B = params->B, KP = padded(K);
  const int64_t nodes = static_cast<int64_t>(B) * KP * KP;
  const int64_t count = nodes + B;
  if (present) {
    int64_t bounds[9];
    const int chunks = enqueue_host_chunks(obs, present, lon, lat, n, params, cfg, s, bounds);
    run_range(obs, params, cfg, s, false, p->outbox, p->outbox + nodes, chunks, obs->chunk_ready, bounds);
  } else {
    run_range(obs, params, cfg, s, false, p->outbox, p->outbox + nodes);
  }
  peer_publish_kernel<<<p->world, 256, 0, s>>>(p->peer_box, p->outbox, p->rank, p->world, p->slot, count,
                                                p->d_epoch);
  THMM_CUDA(cudaGetLastError());
  peer_wait_kernel<<<1, 256, 0, s>>>(p->mailbox, p->foldbuf, p->world, p->slot, count, p->d_epoch, p->d_timeout);
  THMM_CUDA(cudaGetLastError());
  g_launches += 2;
  Workspace& ws = obs->ws;
  const double* delta = static_cast<const double*>(ws.params.ptr) + static_cast<size_t>(B) * K * K;
  double* res = static_cast<double*>(ws.result.ensure(2 * sizeof(double) * B));
  run_tree(ws, K, B, p->foldbuf, p->foldbuf + nodes, p->slot, static_cast<int64_t>(KP) * KP, p->slot, 1, p->world,
           delta, true, res, nullptr, nullptr, s);
  enqueue_results(ws, B, s);
  THMM_CUDA(cudaMemcpyAsync(p->h_timeout, p->d_timeout, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
}

void capture_peer_graph(thmm_peer p, thmm_obs obs, const thmm_params* params, const thmm_config* cfg,
                        cudaStream_t s, bool prof) {
  if (p->graph.valid) {
    cudaGraphExecDestroy(p->graph.exec);
    p->graph.valid = false;
  }
  const int saved = g_launches;
  const uintptr_t sig = workspace_signature(obs);
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  bool ok = true;
  g_capturing = true;
  g_launches = 0;
  try {
    enqueue_peer_eval(p, obs, nullptr, nullptr, nullptr, 0, params, cfg, s);
  } catch (const CudaError&) {
    ok = false;
  }
  g_capturing = false;
  const int launches = g_launches;
  g_launches = saved;
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(s, &graph);
  if (!ok || e != cudaSuccess || graph == nullptr || workspace_signature(obs) != sig) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    return;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  p->graph.K = params->K;
  p->graph.B = params->B;
  p->graph.precision = cfg->precision;
  p->graph.period = cfg->renorm_period;
  p->graph.segments = cfg->segments;
  p->graph.prof = prof;
  p->graph.signature = sig;
  p->graph.obs = obs;
  p->graph.launches = launches;
  p->graph.nseg = g_prof_segments;
  p->graph.exec = exec;
  p->graph.valid = true;
}

}  // namespace

extern "C" {

int thmm_peer_loglik(thmm_peer p, thmm_obs obs, const uint8_t* present, const double* lon, const double* lat,
                     int64_t n, const thmm_params* params, const thmm_config* cfg, double* out, int32_t* status,
                     char* err, size_t errlen) {
  g_launches = 0;
  if (!p || !obs || !out) {
    set_err(err, errlen, "null peer, observation handle or output");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  const int K = params->K, B = params->B, KP = padded(K);
  const int64_t count = static_cast<int64_t>(B) * KP * KP + B;
  if (count > p->slot || obs->device != p->device) {
    set_err(err, errlen, "peer mailbox too small for this batch (or on another device)");
    return THMM_EINVAL;
  }
  const bool host = present != nullptr;
  if (host && (!lon || !lat || n < 1)) {
    set_err(err, errlen, "observation pointers must be non-NULL");
    return THMM_EINVAL;
  }
  std::lock_guard<std::mutex> lk(obs->mu);
  try {
    DeviceGuard dg(obs->device);
    if (host) {
      ensure_obs_capacity(obs, n);
      obs->n = n;
    }
    rc = check_cfg(obs, cfg, err, errlen);
    if (rc != THMM_OK) return rc;
    if (host && (cfg->lo != 0 || cfg->hi != 0)) {
      set_err(err, errlen, "host-array ranges cover the whole (replaced) stream");
      return THMM_EINVAL;
    }
    cudaStream_t s = pick_stream(obs, cfg);
    const bool prof = g_profile;
    const bool graphable = !host && graphs_enabled() && s != nullptr && s != cudaStreamLegacy &&
                           s != cudaStreamPerThread;
    const auto& g = p->graph;
    if (graphable && g.valid && g.obs == obs && g.K == K && g.B == B && g.precision == cfg->precision &&
        g.period == cfg->renorm_period && g.segments == cfg->segments && g.prof == prof &&
        g.signature == workspace_signature(obs)) {
      stage_params_host(obs->ws, params);
      THMM_CUDA(cudaGraphLaunch(g.exec, s));
      g_launches = g.launches;
      g_prof_segments = g.nseg;
      rc = read_results(obs->ws, B, s, out, status);
    } else {
      enqueue_peer_eval(p, obs, present, lon, lat, n, params, cfg, s);
      if (host) THMM_CUDA(cudaEventRecord(staged_event(obs->ws), s));
      rc = read_results(obs->ws, B, s, out, status);
      if (graphable) capture_peer_graph(p, obs, params, cfg, s, prof);
    }
    prof_collect();
    if (*p->h_timeout) {
      set_err(err, errlen, "peer combine timed out waiting for another rank's node");
      return THMM_ECUDA;
    }
    if (rc == THMM_ECOLLAPSE)
      set_err(err, errlen, "running state vector collapsed to zero while combining segments");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

int thmm_peer_destroy(thmm_peer p) {
  if (!p) return THMM_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  if (p->graph.valid) cudaGraphExecDestroy(p->graph.exec);
  for (void* ptr : p->opened) cudaIpcCloseMemHandle(ptr);
  if (p->mailbox) cudaFree(p->mailbox);
  if (p->peer_box) cudaFree(p->peer_box);
  if (p->outbox) cudaFree(p->outbox);
  if (p->foldbuf) cudaFree(p->foldbuf);
  if (p->d_epoch) cudaFree(p->d_epoch);
  if (p->d_timeout) cudaFree(p->d_timeout);
  if (p->h_timeout) cudaFreeHost(p->h_timeout);
  if (prev >= 0) cudaSetDevice(prev);
  delete p;
  return THMM_OK;
}

int thmm_emissions(thmm_obs obs, const thmm_params* params, int64_t lo, int64_t hi, double* out, char* err,
                   size_t errlen) {
  g_launches = 0;
  if (!obs || !out) {
    set_err(err, errlen, "null observation handle or output");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  if (lo < 0 || hi > obs->n || lo >= hi) {
    set_err(err, errlen, "observation range is empty or outside the stream");
    return THMM_EINVAL;
  }
  std::lock_guard<std::mutex> lk(obs->mu);
  try {
    DeviceGuard dg(obs->device);
    cudaStream_t s = obs->stream;
    Workspace& ws = obs->ws;
    thmm::StateParams sp = upload_params(ws, params, s);
    const int64_t n = hi - lo, total = n * params->K;
    double* d = static_cast<double*>(ws.nodes_a.ensure(total * sizeof(double)));
    const int threads = 256;
    const int64_t blocks = (total + threads - 1) / threads;
    thmm::emission_table_kernel<<<static_cast<unsigned>(blocks), threads, 0, s>>>(
        obs->present, obs->lon, obs->lat, lo, n, params->K, sp.states, params->B, -std::log(2.0 * M_PI), d);
    ++g_launches;
    THMM_CUDA(cudaGetLastError());
    THMM_CUDA(cudaMemcpyAsync(out, d, total * sizeof(double), cudaMemcpyDeviceToHost, s));
    THMM_CUDA(cudaStreamSynchronize(s));
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

int thmm_factor_segments(const double* factors, int64_t n, int32_t K, int64_t segments, int32_t renorm_period,
                         int device, double* out_m, double* out_log_scale, char* err, size_t errlen) {
  g_launches = 0;
  if (!factors || !out_m || !out_log_scale) {
    set_err(err, errlen, "null pointer argument");
    return THMM_EINVAL;
  }
  if (n < 1) {
    set_err(err, errlen, "factor chain is empty");
    return THMM_EINVAL;
  }
  if (K < 1 || K > THMM_MAX_STATES) {
    set_err(err, errlen, "parallel engine supports at most %d states, got %d", THMM_MAX_STATES, K);
    return THMM_EINVAL;
  }
  if (segments < 1 || segments > n) {
    set_err(err, errlen, "cannot cut a chain of %lld factors into %lld segments", (long long)n,
            (long long)segments);
    return THMM_EINVAL;
  }
  if (renorm_period < 1) {
    set_err(err, errlen, "renorm_period must be a positive integer");
    return THMM_EINVAL;
  }
  if (device < 0 || device >= thmm_device_count()) {
    set_err(err, errlen, "CUDA device %d not available", device);
    return THMM_ECUDA;
  }
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Workspace& ws = g_ws[device & 63];
  try {
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    const int KP = padded(K), NT = KP / 8;
    ensure_fold(device, K);
    const size_t node = static_cast<size_t>(KP) * KP;
    double* dm = static_cast<double*>(ws.nodes_a.ensure(node * n * sizeof(double)));
    double* de = static_cast<double*>(ws.exps_a.ensure(n * sizeof(double)));
    THMM_CUDA(cudaMemsetAsync(dm, 0, node * n * sizeof(double), s));
    THMM_CUDA(cudaMemsetAsync(de, 0, n * sizeof(double), s));
    THMM_CUDA(cudaMemcpy2DAsync(dm, KP * sizeof(double), factors, K * sizeof(double), K * sizeof(double),
                                static_cast<size_t>(n) * K, cudaMemcpyHostToDevice, s));
    // rows of each factor land at stride KP; factor f occupies rows [f*KP, f*KP+K) after the fix-up below
    if (K != KP) {
      // cudaMemcpy2D above packed n*K rows contiguously at pitch KP; spread them to KP rows per factor.
      double* tmp = static_cast<double*>(ws.nodes_b.ensure(node * n * sizeof(double)));
      THMM_CUDA(cudaMemsetAsync(tmp, 0, node * n * sizeof(double), s));
      THMM_CUDA(cudaMemcpy2DAsync(tmp, KP * KP * sizeof(double), dm, K * KP * sizeof(double),
                                  K * KP * sizeof(double), n, cudaMemcpyDeviceToDevice, s));
      dm = tmp;
    }
    double* om = static_cast<double*>(ws.result.ensure((node + 1) * segments * sizeof(double)));
    double* oe = om + node * segments;
    thmm::FoldArgs fa{};
    fa.in_m = dm;
    fa.in_e = de;
    fa.stride_i = 1;
    fa.stride_b = n;
    fa.n_in = n;
    fa.n_out = segments;
    fa.K = K;
    fa.B = 1;
    fa.out_m = om;
    fa.out_e = oe;
    THMM_DISPATCH(NT, skip_h1(K), launch_fold, fa, s);
    std::vector<double> host((node + 1) * segments);
    THMM_CUDA(cudaMemcpyAsync(host.data(), om, host.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    THMM_CUDA(cudaStreamSynchronize(s));
    for (int64_t sgi = 0; sgi < segments; ++sgi) {
      const double* m = host.data() + node * sgi;
      double mx = 0.0;
      for (int r = 0; r < K; ++r)
        for (int c = 0; c < K; ++c) mx = std::max(mx, m[r * KP + c]);
      double* dst = out_m + static_cast<size_t>(sgi) * K * K;
      const double e = host[node * segments + sgi];
      for (int r = 0; r < K; ++r)
        for (int c = 0; c < K; ++c) dst[r * K + c] = mx > 0.0 ? m[r * KP + c] / mx : 0.0;
      out_log_scale[sgi] = mx > 0.0 ? e * M_LN2 + std::log(mx) : 0.0;
    }
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

}  // extern "C"
