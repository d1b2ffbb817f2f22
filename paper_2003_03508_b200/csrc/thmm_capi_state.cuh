// thmm_capi_state.cuh -- handles, device/pinned buffers, per-handle workspace.
//
// Implementation part of thmm_capi.cu (one translation unit: included there
// once, after the previous parts; not a standalone header).
#pragma once

namespace {

thread_local int g_launches = 0;
thread_local bool g_profile = false;
thread_local double g_prof_chain_ms = 0.0, g_prof_fold_ms = 0.0;
thread_local int64_t g_prof_segments = 0;
thread_local bool g_prof_runs = false;  // last evaluation used the run-absorbing chain
thread_local cudaEvent_t g_prof_ev[4] = {nullptr, nullptr, nullptr, nullptr};
thread_local bool g_prof_collapse = false;  // last evaluation ran the rank-one collapse (burn-in + vector kernels)
thread_local double g_prof_burn_ms = 0.0, g_prof_vec_ms = 0.0;
thread_local bool g_prof_stitch = false;    // last evaluation ran the stitched chain
std::atomic<long long> g_stitch_reruns{0};  // stitched evaluations repeated on the collapse path
thread_local int g_prof_ev_device = -1;
thread_local bool g_capturing = false;  // inside capture_graph's stream capture

// Profiling events become external event nodes when recorded during capture.
cudaError_t record_prof(cudaEvent_t ev, cudaStream_t s) {
  return g_capturing ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal) : cudaEventRecord(ev, s);
}

// Nodes multiplied per CTA per tree level.  The latency of the one-launch tree
// is ~radix * log_radix(S) sequential products; 4 is near the minimum.

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
  DeviceBuffer col;      // rank-one collapse state: r | d | rho [nodes][KP] each, meta [nodes][2]
  int64_t col_nodes = 0; // layout of the last collapse-mode evaluation
  int col_kp = 0;
  DeviceBuffer stitch;   // stitched chain: fin [nodes][KP] | fin_e [nodes] | link [nodes] | link_fail [B] (int)
  DeviceBuffer recs;     // staged copy of pinned host records (batched zero-copy evaluations)
  size_t stitch_fail_off = 0;
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
    col.release();
    stitch.release();
    recs.release();
    stitch_fail_off = 0;
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
  // steps per record of the run-absorbing chain per chunk limit R (index R),
  // estimated from the host flags at upload; < 0 when unknown
  double runs_ratio[33] = {-1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0,
                           -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0,
                           -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0};
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
    bool runs = false;  // captured with the run-absorbing chain
    bool runs_key = false;  // runs_for() at capture (the graph-key part of the kernel choice)
    int cmode = -1;     // collapse mode at capture (collapse_env())
    int launches = 0;
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
    int64_t lo = 0, hi = 0;
    bool prof = false;
    bool runs = false;
    int cmode = -1;
    bool mapped = false;  // zero-copy evaluation (records read from the host buffers)
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


}  // namespace
