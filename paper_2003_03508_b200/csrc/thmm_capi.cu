// thmm_capi.cu -- C-ABI of the B200 HMM likelihood (declared in include/thmm.h).
//
// Host orchestration only: device-resident observation handles, a per-handle
// workspace (grown, never shrunk, so steady-state calls do no cudaMalloc),
// kernel dispatch over the padded state count, the segment tree, and error
// translation.  The arithmetic lives in thmm_kernels.cuh.
//
// One translation unit in five files: thmm_capi_state.cuh (handles, buffers,
// workspace), thmm_capi_plan.cuh (launch geometry, kernel dispatch),
// thmm_capi_eval.cuh (one evaluation: staging, chain, tree, graphs, host
// pipeline), this file (the public entry points) and thmm_capi_peer.cuh
// (the peer-memory combine).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "thmm.h"
#include "thmm_launch.cuh"
#include "thmm_tc.cuh"

#include "thmm_capi_state.cuh"
#include "thmm_capi_plan.cuh"
#include "thmm_capi_eval.cuh"

namespace {
int emissions_impl(thmm_obs obs, const thmm_params* params, int64_t lo, int64_t hi, double* out, char* err,
                   size_t errlen, bool chain);
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

int thmm_runs_info(thmm_obs obs, int32_t K, int32_t precision, int32_t* active, double* steps_per_record,
                   int32_t* G, int32_t* W, int32_t* regs, int32_t* ctas_per_sm, int32_t* R) {
  if (!obs) return THMM_EINVAL;
  if (K < 1 || K > THMM_MAX_STATES || precision < THMM_F64 || precision > THMM_TF32X2) return THMM_EINVAL;
  try {
    DeviceGuard dg(obs->device);
    const bool on = runs_for(obs, K, precision);
    if (active) *active = on ? 1 : 0;
    if (steps_per_record) *steps_per_record = runs_eligible(K, precision) ? obs_runs_ratio(obs, K) : -1.0;
    if (R) *R = runs_eligible(K, precision) ? thmm::runs_r_for_k(K) : 0;
    if (runs_eligible(K, precision)) {
      const ChainPlan& p = runs_plan(obs->device, K);
      if (G) *G = p.G;
      if (W) *W = p.W;
      if (regs) *regs = p.regs;
      if (ctas_per_sm) *ctas_per_sm = p.ctas_per_sm;
    } else {
      if (G) *G = 0;
      if (W) *W = 0;
      if (regs) *regs = 0;
      if (ctas_per_sm) *ctas_per_sm = 0;
    }
    return THMM_OK;
  } catch (const CudaError&) {
    return THMM_ECUDA;
  }
}

int thmm_profile_runs(void) { return g_prof_runs ? 1 : 0; }

int thmm_set_runs_mode(int mode) {
  if (mode < -1 || mode > 1) return THMM_EINVAL;
  runs_env();  // settle the environment default first
  g_runs_mode.store(mode);
  return THMM_OK;
}

int thmm_set_collapse_mode(int mode) {
  if (mode < 0 || mode > 1) return THMM_EINVAL;
  collapse_mode();
  g_collapse_mode.store(mode);
  return THMM_OK;
}

int thmm_set_collapse_params(double tol, int64_t min_len, double min_fill) {
  if (tol < 0.0 || min_len < 0) return THMM_EINVAL;
  if (tol > 0.0) g_collapse_tol.store(tol);
  if (min_len > 0) g_collapse_minlen.store(min_len);
  if (min_fill > 0.0) g_collapse_fill.store(min_fill);
  if (min_fill < 0.0) g_collapse_fill.store(0.0);
  g_collapse_gen.fetch_add(1);
  return THMM_OK;
}

int thmm_collapse_stats(thmm_obs obs, int64_t* nodes_out, int64_t* collapsed, double* records_burned) {
  if (!obs) return THMM_EINVAL;
  std::lock_guard<std::mutex> lk(obs->mu);
  const int64_t nodes = obs->ws.col_nodes;
  if (nodes_out) *nodes_out = nodes;
  if (!obs->ws.col.ptr || nodes == 0) return THMM_EINVAL;
  const size_t need = sizeof(double) * nodes;
  const int K_slots = obs->ws.col_kp;
  try {
    DeviceGuard dg(obs->device);
    std::vector<double> meta(2 * nodes);
    THMM_CUDA(cudaStreamSynchronize(obs->stream));
    const double* base = static_cast<const double*>(obs->ws.col.ptr) + 3 * nodes * K_slots;
    THMM_CUDA(cudaMemcpy(meta.data(), base, 2 * need, cudaMemcpyDeviceToHost));
    int64_t c = 0;
    double burned = 0.0;
    for (int64_t i = 0; i < nodes; ++i)
      if (meta[2 * i] >= 0.0) {
        ++c;
        burned += meta[2 * i];
      }
    if (collapsed) *collapsed = c;
    if (records_burned) *records_burned = burned;
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, nullptr, 0);
  }
}

int thmm_profile_phases(double* burn_ms, double* vec_ms) {
  const bool on = g_prof_collapse || g_prof_stitch;
  if (burn_ms) *burn_ms = on ? g_prof_burn_ms : -1.0;
  if (vec_ms) *vec_ms = on ? g_prof_vec_ms : -1.0;
  return g_prof_stitch ? 2 : (g_prof_collapse ? 1 : 0);
}

int thmm_stitch_shard(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, int32_t first,
                      double* d_block, char* err, size_t errlen) {
  return stitch_shard_impl(obs, params, cfg, first, d_block, nullptr, 0, nullptr, err, errlen);
}

int thmm_stitch_shard_host(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                           const thmm_params* params, const thmm_config* cfg, int32_t first, double* d_block,
                           char* err, size_t errlen) {
  if (n < 1) {
    set_err(err, errlen, "observation sequence is empty");
    return THMM_EINVAL;
  }
  if (!present || !lon || !lat) {
    set_err(err, errlen, "observation pointers must be non-NULL");
    return THMM_EINVAL;
  }
  const HostShard host{present, lon, lat, n};
  return stitch_shard_impl(obs, params, cfg, first, d_block, nullptr, 0, nullptr, err, errlen, &host);
}

int thmm_stitch_link(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, const double* d_prev,
                     int64_t prev_stride, double* d_link, char* err, size_t errlen) {
  if (!d_prev || !d_link) {
    set_err(err, errlen, "null device buffer");
    return THMM_EINVAL;
  }
  return stitch_shard_impl(obs, params, cfg, 0, nullptr, d_prev, prev_stride, d_link, err, errlen);
}

int64_t thmm_stitch_segments(thmm_obs obs, int32_t K, int32_t B) {
  if (!obs || K < 1 || K > THMM_MAX_STATES || B < 1) return 0;
  try {
    DeviceGuard dg(obs->device);
    thmm_config c{};
    c.precision = THMM_F64;
    c.renorm_period = 8;
    return stitch_segments(obs->device, K, &c, obs->n, B,
                           runs_for(obs, K, THMM_F64) ? obs_runs_ratio(obs, K) : 1.0, -1.0, obs->runs_ratio[0]);
  } catch (const CudaError&) {
    return 0;
  }
}

int thmm_profile_collect(void) {
  prof_collect();
  return THMM_OK;
}

int thmm_set_stitch_mode(int mode) {
  if (mode < 0 || mode > 1) return THMM_EINVAL;
  stitch_mode();
  g_stitch_mode.store(mode);
  return THMM_OK;
}

long long thmm_stitch_reruns(void) { return g_stitch_reruns.load(); }

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

int thmm_host_register(const void* ptr, size_t bytes, char* err, size_t errlen) {
  if (!ptr || bytes == 0) {
    set_err(err, errlen, "null or empty host range");
    return THMM_EINVAL;
  }
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, ptr) == cudaSuccess && attr.type != cudaMemoryTypeUnregistered) {
    set_err(err, errlen, "host range is already page-locked or device memory");
    return THMM_EINVAL;  // (e.g. torch pin_memory): usable as is, nothing to register
  }
  cudaGetLastError();
  const cudaError_t e = cudaHostRegister(const_cast<void*>(ptr), bytes,
                                         cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_err(err, errlen, cudaGetErrorString(e));
    return THMM_EINVAL;
  }
  return THMM_OK;
}

int thmm_host_unregister(const void* ptr) {
  if (!ptr) return THMM_EINVAL;
  if (cudaHostUnregister(const_cast<void*>(ptr)) != cudaSuccess) {
    cudaGetLastError();
    return THMM_EINVAL;
  }
  return THMM_OK;
}
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
            gr.prof == prof && gr.signature == workspace_signature(obs) &&
            gr.runs_key == runs_for(obs, params->K, cfg->precision, hi - cfg->lo) && gr.cmode == collapse_env())
          hit = &gr;
    }
    if (hit) {
      // Replay: stage the new parameters where the captured H2D copy reads them.
      stage_params_host(obs->ws, params);
      hit->last_use = ++obs->uses;
      THMM_CUDA(cudaGraphLaunch(hit->exec, s));
      g_launches = hit->launches;
      g_prof_segments = hit->nseg;
      g_prof_runs = hit->runs;
      rc = read_results(obs->ws, params->B, s, out, status);
    } else {
      run_range(obs, params, cfg, s, true, nullptr, nullptr);
      rc = finish_results(obs->ws, params->B, s, out, status);
      if (graphs_enabled() && rc != kStitchFailed) capture_graph(obs, params, cfg, hi, prof);
    }
    if (rc == kStitchFailed) rc = rerun_without_stitch(obs, params, cfg, s, nullptr, out, status);
    prof_collect();
    if (rc == THMM_ECOLLAPSE)
      set_err(err, errlen, "running state vector collapsed to zero while combining segments");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}


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
    // validate against the new length before the handle is touched: a
    // rejected call leaves the handle's records as they were
    rc = check_cfg_n(n, cfg, err, errlen);
    if (rc != THMM_OK) return rc;
    ensure_obs_capacity(obs, n);
    obs->n = n;
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
        if (g.valid && !g.mapped && g.src[0] == present && g.src[1] == lon && g.src[2] == lat && g.n == n &&
            g.K == params->K &&
            g.B == params->B && g.precision == cfg->precision && g.period == cfg->renorm_period &&
            g.segments == cfg->segments && g.lo == cfg->lo && g.hi == cfg->hi && g.prof == prof &&
            g.signature == sig && g.cmode == collapse_env())
          hit = &g;
    }
    if (hit) {
      stage_params_host(obs->ws, params);
      hit->last_use = ++obs->uses;
      THMM_CUDA(cudaGraphLaunch(hit->exec, s));
      g_launches = hit->launches;
      g_prof_segments = hit->nseg;
      g_prof_runs = hit->runs;
      rc = read_results(obs->ws, params->B, s, out, status);
    } else {
      int64_t bounds[9];
      const int chunks = enqueue_host_chunks(obs, present, lon, lat, n, params, cfg, s, bounds);
      run_range(obs, params, cfg, s, true, nullptr, nullptr, chunks, obs->chunk_ready, bounds);
      rc = finish_results(obs->ws, params->B, s, out, status);
      if (graphable && rc != kStitchFailed) capture_host_graph(obs, present, lon, lat, n, params, cfg, s, prof);
    }
    if (rc == kStitchFailed) rc = rerun_without_stitch(obs, params, cfg, s, nullptr, out, status);
    prof_collect();
    if (rc == THMM_ECOLLAPSE)
      set_err(err, errlen, "running state vector collapsed to zero while combining segments");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}


int thmm_loglik_mapped(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
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
  MappedSource src;
  {
    DeviceGuard dg(obs->device);
    if (!mapped_source(present, lon, lat, n, src))  // pageable memory: the pipelined copy
      return thmm_loglik_host(obs, present, lon, lat, n, params, cfg, out, status, err, errlen);
  }
  // a batch reads every record once per proposal; a short stream is latency-bound
  // on uncached PCIe reads -- both copy the records to HBM first (one DMA per array)
  src.stage = params && (params->B >= kMappedCopyMinB || n <= mapped_copy_max_n());
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  rc = check_cfg_n(n, cfg, err, errlen);
  if (rc != THMM_OK) return rc;
  std::lock_guard<std::mutex> lk(obs->mu);
  try {
    DeviceGuard dg(obs->device);
    cudaStream_t s = pick_stream(obs, cfg);
    const bool prof = g_profile;
    const bool graphable = graphs_enabled() && s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread;
    const void* host[3] = {present, lon, lat};
    thmm_obs_s::HostGraph* hit = nullptr;
    if (graphable) {
      const uintptr_t sig = workspace_signature(obs);
      for (auto& g : obs->host_graphs)
        if (g.valid && g.mapped && g.src[0] == host[0] && g.src[1] == host[1] && g.src[2] == host[2] && g.n == n &&
            g.K == params->K && g.B == params->B && g.precision == cfg->precision &&
            g.period == cfg->renorm_period && g.segments == cfg->segments && g.lo == cfg->lo && g.hi == cfg->hi &&
            g.prof == prof && g.signature == sig && g.cmode == collapse_env())
          hit = &g;
    }
    if (hit) {
      stage_params_host(obs->ws, params);
      hit->last_use = ++obs->uses;
      THMM_CUDA(cudaGraphLaunch(hit->exec, s));
      g_launches = hit->launches;
      g_prof_segments = hit->nseg;
      g_prof_runs = hit->runs;
      rc = read_results(obs->ws, params->B, s, out, status);
    } else {
      estimate_source(src);
      run_range(obs, params, cfg, s, true, nullptr, nullptr, 1, nullptr, nullptr, &src);
      rc = finish_results(obs->ws, params->B, s, out, status);
      if (graphable && rc != kStitchFailed) capture_mapped_graph(obs, host, src, params, cfg, s, prof);
    }
    if (rc == kStitchFailed) {
      estimate_source(src);
      rc = rerun_without_stitch(obs, params, cfg, s, &src, out, status);
    }
    prof_collect();
    if (rc == THMM_ECOLLAPSE)
      set_err(err, errlen, "running state vector collapsed to zero while combining segments");
    return rc;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

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
    MappedSource src;
    if (mapped_source(present, lon, lat, n, src)) {  // pinned: read in place, the handle keeps its records
      rc = check_cfg_n(n, cfg, err, errlen);
      if (rc != THMM_OK) return rc;
      cudaStream_t s = pick_stream(obs, cfg);
      estimate_source(src);
      run_range(obs, params, cfg, s, false, d_m, d_e, 1, nullptr, nullptr, &src);
      THMM_CUDA(cudaEventRecord(staged_event(obs->ws), s));
      return THMM_OK;
    }
    rc = check_cfg_n(n, cfg, err, errlen);  // before the handle's records are replaced
    if (rc != THMM_OK) return rc;
    ensure_obs_capacity(obs, n);
    obs->n = n;
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


int thmm_emissions(thmm_obs obs, const thmm_params* params, int64_t lo, int64_t hi, double* out, char* err,
                   size_t errlen) {
  return emissions_impl(obs, params, lo, hi, out, err, errlen, false);
}

int thmm_emissions_chain(thmm_obs obs, const thmm_params* params, int64_t lo, int64_t hi, double* out,
                         char* err, size_t errlen) {
  return emissions_impl(obs, params, lo, hi, out, err, errlen, true);
}

}  // extern "C"

namespace {

int emissions_impl(thmm_obs obs, const thmm_params* params, int64_t lo, int64_t hi, double* out, char* err,
                   size_t errlen, bool chain) {
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
    auto kern = chain ? thmm::emission_table_kernel<true> : thmm::emission_table_kernel<false>;
    kern<<<static_cast<unsigned>(blocks), threads, 0, s>>>(obs->present, obs->lon, obs->lat, lo, n, params->K,
                                                           sp.states, params->B, -std::log(2.0 * M_PI), d);
    ++g_launches;
    THMM_CUDA(cudaGetLastError());
    THMM_CUDA(cudaMemcpyAsync(out, d, total * sizeof(double), cudaMemcpyDeviceToHost, s));
    THMM_CUDA(cudaStreamSynchronize(s));
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

}  // namespace

extern "C" {

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

#include "thmm_capi_peer.cuh"
