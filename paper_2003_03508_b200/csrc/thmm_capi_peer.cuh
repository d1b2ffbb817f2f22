// thmm_capi_peer.cuh -- peer-memory combine over NVLink/NVSwitch (thmm_peer_*).
//
// Implementation part of thmm_capi.cu (one translation unit: included there
// once, after the previous parts; not a standalone header).
#pragma once

// ---------------------------------------------------------------------------
// Peer-memory combine over NVLink / NVSwitch (one process per GPU): every
// rank's root nodes are stored straight into every peer's mailbox by one
// publish kernel (P2P stores through CUDA IPC mappings) and announced with a
// release-ordered flag carrying the evaluation's epoch; a one-warp wait
// kernel acquires all flags, and the segment tree folds the world's nodes in
// rank order from local memory.  No collective library call, no host
// synchronisation before the result read.
// ---------------------------------------------------------------------------

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
    bool runs = false;
    bool runs_key = false;
    int cmode = -1;
    const void* src[3] = {};  // zero-copy evaluations: the pinned host buffers read in place
    int64_t n = 0;
    int64_t lo = 0, hi = 0;   // record range the graph evaluates (hi resolved: 0 -> the stream length)
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
// src: records read in place from pinned host memory (zero-copy); else
// present != NULL: host records copied into the handle, pipelined; else the
// handle's device records.
void enqueue_peer_eval(thmm_peer p, thmm_obs obs, const uint8_t* present, const double* lon, const double* lat,
                       int64_t n, const thmm_params* params, const thmm_config* cfg, cudaStream_t s,
                       const MappedSource* src = nullptr) {
  const int K = params->K, B = params->B, KP = padded(K);
  const int64_t nodes = static_cast<int64_t>(B) * KP * KP;
  const int64_t count = nodes + B;
  if (src) {
    run_range(obs, params, cfg, s, false, p->outbox, p->outbox + nodes, 1, nullptr, nullptr, src);
  } else if (present) {
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
                        cudaStream_t s, bool prof, const void* const* host = nullptr,
                        const MappedSource* src = nullptr) {
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
    enqueue_peer_eval(p, obs, nullptr, nullptr, nullptr, 0, params, cfg, s, src);
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
  p->graph.runs = g_prof_runs;
  p->graph.runs_key = runs_for(obs, params->K, cfg->precision);
  p->graph.cmode = collapse_env();
  p->graph.precision = cfg->precision;
  p->graph.period = cfg->renorm_period;
  p->graph.segments = cfg->segments;
  p->graph.prof = prof;
  p->graph.signature = sig;
  p->graph.obs = obs;
  for (int i = 0; i < 3; ++i) p->graph.src[i] = src ? host[i] : nullptr;
  p->graph.n = src ? src->n : 0;
  p->graph.lo = cfg->lo;
  p->graph.hi = cfg->hi != 0 ? cfg->hi : (src ? src->n : obs->n);
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
    // Pinned host records are read in place (zero-copy; the handle keeps its
    // own records); pageable ones replace the handle's records, copy pipelined.
    MappedSource src;
    const bool mapped = host && mapped_source(present, lon, lat, n, src);
    // validate before the handle is touched (a rejected call keeps its records)
    rc = host ? check_cfg_n(n, cfg, err, errlen) : check_cfg(obs, cfg, err, errlen);
    if (rc != THMM_OK) return rc;
    if (host && (cfg->lo != 0 || cfg->hi != 0)) {
      set_err(err, errlen, "host-array ranges cover the whole (replaced) stream");
      return THMM_EINVAL;
    }
    if (host && !mapped) {
      ensure_obs_capacity(obs, n);
      obs->n = n;
    }
    cudaStream_t s = pick_stream(obs, cfg);
    const bool prof = g_profile;
    const bool graphable = (!host || mapped) && graphs_enabled() && s != nullptr && s != cudaStreamLegacy &&
                           s != cudaStreamPerThread;
    const void* hsrc[3] = {mapped ? present : nullptr, mapped ? lon : nullptr, mapped ? lat : nullptr};
    const auto& g = p->graph;
    // the graph bakes in the record range: a handle whose stream was replaced
    // by a shorter one (same buffers) must not replay the old range
    const int64_t hi_res = cfg->hi != 0 ? cfg->hi : (mapped ? n : obs->n);
    // (a zero-copy graph is keyed by the host buffers: same buffers, same decision)
    if (graphable && g.valid && g.obs == obs && g.K == K && g.B == B && g.precision == cfg->precision &&
        g.lo == cfg->lo && g.hi == hi_res &&
        g.period == cfg->renorm_period && g.segments == cfg->segments && g.prof == prof &&
        g.signature == workspace_signature(obs) && (mapped || g.runs_key == runs_for(obs, K, cfg->precision)) && g.cmode == collapse_env() &&
        g.src[0] == hsrc[0] && g.src[1] == hsrc[1] && g.src[2] == hsrc[2] && g.n == (mapped ? n : 0)) {
      stage_params_host(obs->ws, params);
      THMM_CUDA(cudaGraphLaunch(g.exec, s));
      g_launches = g.launches;
      g_prof_segments = g.nseg;
      g_prof_runs = g.runs;
      rc = read_results(obs->ws, B, s, out, status);
    } else {
      if (mapped) estimate_source(src);
      enqueue_peer_eval(p, obs, present, lon, lat, n, params, cfg, s, mapped ? &src : nullptr);
      if (host && !mapped) THMM_CUDA(cudaEventRecord(staged_event(obs->ws), s));
      rc = read_results(obs->ws, B, s, out, status);
      if (graphable) capture_peer_graph(p, obs, params, cfg, s, prof, hsrc, mapped ? &src : nullptr);
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

}  // extern "C"
