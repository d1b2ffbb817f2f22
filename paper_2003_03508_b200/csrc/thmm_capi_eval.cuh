// thmm_capi_eval.cuh -- one evaluation: parameter staging, chain over a range, segment tree, CUDA graphs, the chunked host-array pipeline, range nodes and the node fold.
//
// Implementation part of thmm_capi.cu (one translation unit: included there
// once, after the previous parts; not a standalone header).
#pragma once

namespace {

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
  THMM_CUDA((thmm::tree_launch<NT, SKIP>(a, grid, thmm::tree_smem_bytes(NT), s)));
  ++g_launches;
}

// Ordered fold of n0 nodes per proposal (layout given by element strides)
// with the one-launch radix-8 (radix-4 for wide rows) tree (tree_fold_kernel).  finish: log(delta' M 1) + e ln 2
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
  ta.radix = thmm::tree_radix(NT);
  ta.count[0] = n0;
  int levels = 0;
  do {
    if (levels >= thmm::kTreeMaxLevels) throw CudaError{cudaErrorInvalidValue, "segment tree too deep"};
    ta.count[levels + 1] = (ta.count[levels] + ta.radix - 1) / ta.radix;
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

// Records read in place from pinned host memory (zero-copy) instead of the
// handle's device buffers: device-usable pointers, count, and the steps per
// record of the run-absorbing chain sampled from the host flags.
struct MappedSource {
  const uint8_t* present = nullptr;
  const double* lon = nullptr;
  const double* lat = nullptr;
  int64_t n = 0;
  const uint8_t* host_present = nullptr;  // the caller's pointer (sampling the step ratio on the host)
  double ratio[33];  // filled by estimate_runs_ratios (estimated == true)
  bool estimated = false;
  // Batches of proposals read every record once per proposal: for B >=
  // kMappedCopyMinB the records are first copied to a device staging buffer
  // (one DMA per array, inside the evaluation) and read from HBM.
  bool stage = false;
};
constexpr int kMappedCopyMinB = 2;
constexpr int64_t kMappedCopyMaxNDefault = 65536;  // records (1.1 MB): below this a DMA beats zero-copy latency
int64_t mapped_copy_max_n() {  // THMM_MAPPED_COPY_MAXN overrides (diagnostics)
  static const int64_t v = [] {
    const char* e = std::getenv("THMM_MAPPED_COPY_MAXN");
    return e ? static_cast<int64_t>(std::atoll(e)) : kMappedCopyMaxNDefault;
  }();
  return v;
}

// The stitched chain (thmm_vec.cuh) over the range of `ca` (lo, n, P, records
// set) cut into `total` segments: main pass, links, then either the finish
// (log L | status into res) or, with `block`, the shard summary of a
// multi-GPU chain; `first`: segment 0 starts from delta.  With `link_src`
// only the external link of segment 0 (p from another rank's final rows) is
// computed, into link_out [B][2].
// cuStreamWriteValue32 (driver API, through the runtime's entry-point query:
// no link-time libcuda dependency); nullptr if unavailable or
// THMM_STAGE_SINGLE=0 (then one launch per time chunk).
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value32() {
  static const WriteValue32Fn fn = []() -> WriteValue32Fn {
    const char* e = std::getenv("THMM_STAGE_SINGLE");
    if (e && e[0] == '0') return nullptr;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return reinterpret_cast<WriteValue32Fn>(p);
  }();
  return fn;
}

// Records of a host-array evaluation staged into HBM while the stitched main
// pass runs: the pinned host arrays and the device staging buffers.
struct StitchStage {
  const uint8_t* present;
  const double* lon;
  const double* lat;
  uint8_t* d_present;
  double* d_lon;
  double* d_lat;
};

// Time chunks of a staged stitched evaluation (fractions of every segment,
// f[0] = 0 < ... < f[C] = 1): geometric with ratio R = DMA rate / main-pass
// rate (records/s; DMA 55 GB/s = 3.2e9 records/s on B200, the main pass
// ~0.6 x 37.1 TF / 2 K K_p).  Chain-bound (R > 1): growing chunks, each copy
// hidden under the previous chunk's steps, the chain waits only for the
// small first one.  Copy-bound (R < 1): shrinking chunks, so only the small
// last chunk's steps run after the copy engine finishes.  Chunks >= 32
// records of a segment, at most max_chunks (<= 16).
int stitch_time_chunks(int64_t n, int64_t total, int K, int B, double* f, int max_chunks) {
  f[0] = 0.0;
  f[1] = 1.0;
  const int64_t per_seg = n / std::max<int64_t>(total, 1);
  if (n < (int64_t{1} << 18) || per_seg < 96) return 1;
  const double chain_rate = 0.6 * 37.1e12 / (2.0 * K * padded(K) * std::max(B, 1));
  // (x 0.75: a copy that lags its chunk stalls the chain at every boundary --
  // with the unscaled ratio K=80 N=1e8 lost 4.4 ms over 8 chunks)
  double R = 0.75 * (55e9 / 17.0) / chain_rate;
  R = R >= 1.0 ? std::min(4.0, std::max(1.15, R)) : std::max(0.4, std::min(0.8, R));
  static const double r_env = [] {  // diagnostics: THMM_STAGE_RATIO overrides R
    const char* e = std::getenv("THMM_STAGE_RATIO");
    return e ? std::atof(e) : 0.0;
  }();
  // (even chunks for copy-bound single launches measured slower: K=50 N=1e7
  // 4.27 -> 4.86 ms -- 16 narrow 2-D copies run below the DMA rate)
  if (r_env > 0.0) R = r_env;
  int C = 1;
  double sum = 1.0;
  while (C < max_chunks) {  // most chunks whose smallest stays >= 32 records per segment
    const double next = sum + std::pow(R, C);
    const double smallest = std::min(1.0, std::pow(R, C));
    if (static_cast<double>(per_seg) * smallest / next < 32.0) break;
    sum = next;
    ++C;
  }
  double acc = 0.0, t = 1.0;
  for (int c = 0; c < C; ++c) {
    f[c] = acc / sum;
    acc += t;
    t *= R;
  }
  f[C] = 1.0;
  return C;
}

// Copy time chunk c of every segment (records [begin(c), begin(c+1)) of a
// segment of length L, thmm::time_chunk_begin; the first `rem` segments are
// one record longer, so two 2-D copies per array) on the copy stream.
void enqueue_stage_chunk(const StitchStage& st, int64_t n, int64_t total, int c, int C, const double* f,
                         cudaStream_t cs) {
  if (C <= 1) {  // one chunk: three contiguous copies
    THMM_CUDA(cudaMemcpyAsync(st.d_present, st.present, n, cudaMemcpyDefault, cs));
    THMM_CUDA(cudaMemcpyAsync(st.d_lon, st.lon, n * sizeof(double), cudaMemcpyDefault, cs));
    THMM_CUDA(cudaMemcpyAsync(st.d_lat, st.lat, n * sizeof(double), cudaMemcpyDefault, cs));
    return;
  }
  // the flag bytes (1 B/record) go whole with the first chunk for streams up
  // to 16 Mi records (2-D copies of rows of a few dozen bytes cost ~25 ns a
  // row: K=25 N=1e6 staged 0.89 -> 0.61 ms); longer streams keep them in
  // their time chunks (K=80 N=1e8: 100 MB would hold up the first chunk ~2 ms)
  const bool flags_whole = n <= (int64_t{1} << 24);
  if (flags_whole && c == 0) THMM_CUDA(cudaMemcpyAsync(st.d_present, st.present, n, cudaMemcpyDefault, cs));
  const int64_t base = n / total, rem = n % total;
  for (int grp = 0; grp < 2; ++grp) {
    const int64_t L = base + (grp == 0 ? 1 : 0), rows = grp == 0 ? rem : total - rem;
    if (rows <= 0 || L <= 0) continue;
    const int64_t first = grp == 0 ? 0 : rem * (base + 1);  // first record of the group
    const int64_t off = first + thmm::time_chunk_begin(L, f, c);
    const int64_t w = thmm::time_chunk_begin(L, f, c + 1) - thmm::time_chunk_begin(L, f, c);
    if (w <= 0) continue;
    if (!flags_whole)
      THMM_CUDA(cudaMemcpy2DAsync(st.d_present + off, L, st.present + off, L, w, rows, cudaMemcpyDefault, cs));
    THMM_CUDA(cudaMemcpy2DAsync(st.d_lon + off, L * 8, st.lon + off, L * 8, w * 8, rows, cudaMemcpyDefault, cs));
    THMM_CUDA(cudaMemcpy2DAsync(st.d_lat + off, L * 8, st.lat + off, L * 8, w * 8, rows, cudaMemcpyDefault, cs));
  }
}

void enqueue_stitched(thmm_obs obs, thmm::ChainArgs ca, int64_t total, int first, cudaStream_t s, bool prof,
                      double* res, double* block, const double* link_src, int64_t link_src_stride,
                      double* link_out = nullptr, const StitchStage* stage = nullptr) {
  Workspace& ws = obs->ws;
  const int K = ca.K, B = ca.B, KP = padded(K);
  const int64_t nodes = static_cast<int64_t>(B) * total;
  const size_t fin_bytes = sizeof(double) * nodes * (KP + 2);
  const ChainPlan& vp = vec_plan(obs->device, K);
  const size_t gent_off = (fin_bytes + sizeof(int) * B + 15) / 16 * 16;
  const size_t arrive_off = gent_off + static_cast<size_t>(B) * thmm::runs_entry_pairs(vp.nt, vp.tail) * 16;
  const size_t bytes = arrive_off + 16;
  void* prev = ws.stitch.ptr;
  char* base = static_cast<char*>(ws.stitch.ensure(bytes));
  if (base != prev || ws.stitch_fail_off != fin_bytes) {
    THMM_CUDA(cudaMemsetAsync(base + fin_bytes, 0, sizeof(int) * B, s));  // link_fail starts clear
    ws.stitch_fail_off = fin_bytes;
  }
  double* fin = reinterpret_cast<double*>(base);
  ca.fin = fin;
  ca.fin_e = fin + nodes * KP;
  ca.link = fin + nodes * (KP + 1);
  ca.link_fail = reinterpret_cast<int*>(base + fin_bytes);
  ca.collapse_tol = collapse_tol();
  ca.stitch_delta = first;
  ca.nseg = total;
  ca.node_offset = 0;
  ca.node_stride_b = total;
  g_prof_collapse = false;
  g_prof_stitch = true;
  g_prof_runs = false;
  g_prof_segments = total;
  const StitchOps& ops = stitch_ops_for(vp);
  // Gamma in the B-fragment layout once per proposal; every CTA of the
  // main pass and the links bulk-copies it into shared memory
  double2* gent = reinterpret_cast<double2*>(base + gent_off);
  THMM_CUDA(ops.prep(ca, gent, s));
  ++g_launches;
  ca.gent = gent;
  if (link_src) {
    ca.link_src = link_src;
    ca.link_src_stride = link_src_stride;
    ca.link_out = link_out;
    THMM_CUDA(cudaMemsetAsync(link_out, 0, sizeof(double) * 2 * B, s));
    const VecSpread sp = vec_spread(vp, 1, 1);
    ca.ebatch = sp.batch ? 1 : 0;
    THMM_CUDA(ops.link(ca, dim3(1, static_cast<unsigned>(B)), 32 * sp.W, sp.smem, s));
    ++g_launches;
    return;
  }
  const VecSpread fw = vec_spread(vp, B, (total + 7) / 8);  // 8 rows (segments) per warp
  // (16 chunks for the single launch, whose chunks cost nothing; 8 launches otherwise)
  int C = stage ? stitch_time_chunks(ca.n, total, K, B, ca.t_frac, write_value32() ? 16 : 8) : 1;
  if (!stage) {  // diagnostics: THMM_TIME_CHUNKS=C splits a device-resident main pass evenly
    static const int forced = [] {
      const char* e = std::getenv("THMM_TIME_CHUNKS");
      return e ? std::max(1, std::min(8, std::atoi(e))) : 1;
    }();
    C = forced;
    for (int c = 0; c <= C; ++c) ca.t_frac[c] = static_cast<double>(c) / C;
  }
  // single launch: the copy stream signals each landed chunk with a stream
  // memory operation and the main pass waits per record window (no launch
  // boundary per chunk: each one cost ~5 % of its chunk in warp-tail time)
  const WriteValue32Fn wv = stage && C > 1 ? write_value32() : nullptr;
  unsigned* arrive = wv ? reinterpret_cast<unsigned*>(base + arrive_off) : nullptr;
  if (stage) {
    // copies on the copy stream (behind every earlier read of the staging
    // buffer on s), time chunk c of the main pass behind copy c
    if (!obs->copy_stream) THMM_CUDA(cudaStreamCreateWithFlags(&obs->copy_stream, cudaStreamNonBlocking));
    for (auto& e : obs->chunk_ready)
      if (!e) THMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!obs->reads_done) THMM_CUDA(cudaEventCreateWithFlags(&obs->reads_done, cudaEventDisableTiming));
    if (arrive) THMM_CUDA(cudaMemsetAsync(arrive, 0, sizeof(unsigned), s));
    THMM_CUDA(cudaEventRecord(obs->reads_done, s));
    THMM_CUDA(cudaStreamWaitEvent(obs->copy_stream, obs->reads_done, 0));
    for (int c = 0; c < C; ++c) {
      enqueue_stage_chunk(*stage, ca.n, total, c, C, ca.t_frac, obs->copy_stream);
      if (arrive) {
        if (wv(reinterpret_cast<CUstream>(obs->copy_stream), reinterpret_cast<CUdeviceptr>(arrive),
               static_cast<cuuint32_t>(c + 1), 0) != CUDA_SUCCESS)
          throw CudaError{cudaErrorUnknown, "cuStreamWriteValue32"};
      } else {
        THMM_CUDA(cudaEventRecord(obs->chunk_ready[c], obs->copy_stream));  // (C <= 8 launches)
      }
    }
    if (arrive) THMM_CUDA(cudaEventRecord(obs->chunk_ready[0], obs->copy_stream));  // the join below
  }
  if (prof) THMM_CUDA(record_prof(g_prof_ev[0], s));
  ca.t_chunks = C;
  ca.ebatch = fw.batch ? 1 : 0;
  if (arrive) {
    ca.arrive = arrive;
    ca.t_chunk = 0;
    THMM_CUDA(ops.fwd(ca, dim3(static_cast<unsigned>(fw.ctas), static_cast<unsigned>(B)), 32 * fw.W, fw.smem, s));
    ++g_launches;
    THMM_CUDA(cudaStreamWaitEvent(s, obs->chunk_ready[0], 0));  // (joins the copy stream; already passed)
    ca.arrive = nullptr;
  } else {
    for (int c = 0; c < C; ++c) {
      if (stage) THMM_CUDA(cudaStreamWaitEvent(s, obs->chunk_ready[c], 0));
      ca.t_chunk = c;
      THMM_CUDA(ops.fwd(ca, dim3(static_cast<unsigned>(fw.ctas), static_cast<unsigned>(B)), 32 * fw.W, fw.smem, s));
      ++g_launches;
    }
  }
  ca.t_chunks = 1;
  ca.t_chunk = 0;
  if (prof) THMM_CUDA(record_prof(g_prof_ev[3], s));
  if (total > 1) {
    const VecSpread lk = vec_spread(vp, B, (total - 1 + 3) / 4);  // 4 (p, h) pairs per warp
    ca.ebatch = lk.batch ? 1 : 0;
    THMM_CUDA(ops.link(ca, dim3(static_cast<unsigned>(lk.ctas), static_cast<unsigned>(B)), 32 * lk.W, lk.smem, s));
    ++g_launches;
  }
  if (prof) THMM_CUDA(record_prof(g_prof_ev[1], s));
  THMM_CUDA(ops.finish(ca, res, res ? reinterpret_cast<int32_t*>(res + B) : nullptr, block, s));
  ++g_launches;
  if (prof) THMM_CUDA(record_prof(g_prof_ev[2], s));
}

// Runs the chain over [lo, hi) for all proposals and folds the segments.
// finish: write loglik/status to ws.result; else write one node per
// proposal to (out_m, out_e).
// chunks > 1 (host-array pipeline): the range is cut into `chunks`
// contiguous sub-ranges, each reduced by its own chain launch once ready[c]
// (the host->device copy of its records) has fired, so the copy of chunk
// c+1 overlaps the tensor work of chunk c; all segment nodes feed one tree.
// src: read the records from pinned host memory (zero-copy) instead.
void run_range(thmm_obs obs, const thmm_params* P, const thmm_config* cfg, cudaStream_t s, bool finish,
               double* out_m, double* out_e, int chunks = 1, const cudaEvent_t* ready = nullptr,
               const int64_t* chunk_bounds = nullptr, const MappedSource* src = nullptr) {
  const int K = P->K, B = P->B, KP = padded(K);
  const int64_t n_range = (cfg->hi > 0 ? cfg->hi : (src ? src->n : obs->n)) - cfg->lo;
  const bool runs = src ? use_runs(K, cfg->precision, src->ratio[thmm::runs_r_for_k(K)], n_range)
                        : runs_for(obs, K, cfg->precision, n_range);
  const int64_t lo = cfg->lo, hi = cfg->hi > 0 ? cfg->hi : (src ? src->n : obs->n);
  const int64_t n = hi - lo;
  chunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(chunks, n)));
  // rank-one collapse (thmm_vec.cuh): burn-in on the run-absorbing chain, then
  // the row-stacked vector continuation; segment count sized for the latter
  const double rr = src ? src->ratio[thmm::runs_r_for_k(K)] : obs_runs_ratio(obs, K);
  const int64_t st_segs =
      (finish && chunks == 1 && !g_no_stitch)
          ? stitch_segments(obs->device, K, cfg, n, B, runs ? rr : 1.0, src && !src->stage ? src->ratio[0] : -1.0,
                            src ? src->ratio[0] : obs->runs_ratio[0])
          : 0;
  const int64_t col_segs = st_segs > 0 ? st_segs : (chunks == 1 ? collapse_segments(obs->device, K, cfg, n, B) : 0);
  const bool collapse = col_segs > 0;
  const bool use_runs_kernel = runs || collapse;
  const ChainPlan& plan = use_runs_kernel ? runs_plan(obs->device, K) : plan_for(obs->device, K, cfg->precision);
  ensure_fold(obs->device, K);
  int64_t c_nseg[8], c_lo[8], c_n[8], total = 0;
  for (int c = 0; c < chunks; ++c) {
    const int64_t base = n / chunks, rem = n % chunks;
    c_lo[c] = chunk_bounds ? chunk_bounds[c] : c * base + std::min<int64_t>(c, rem);
    c_n[c] = chunk_bounds ? chunk_bounds[c + 1] - chunk_bounds[c] : base + (c < rem ? 1 : 0);
    c_nseg[c] = collapse ? col_segs
                         : (cfg->segments > 0 ? std::min<int64_t>(cfg->segments, c_n[c]) : auto_segments(plan, c_n[c], B));
    total += c_nseg[c];
  }
  Workspace& ws = obs->ws;
  thmm::StateParams sp = upload_params(ws, P, s);

  const size_t node_bytes = static_cast<size_t>(KP) * KP * sizeof(double);
  double* seg_m = static_cast<double*>(ws.nodes_a.ensure(node_bytes * B * total));
  double* seg_e = static_cast<double*>(ws.exps_a.ensure(sizeof(double) * B * total));

  thmm::ChainArgs ca{};
  ca.present = src ? src->present : obs->present;
  ca.lon = src ? src->lon : obs->lon;
  ca.lat = src ? src->lat : obs->lat;
  ca.sysmem = src ? 1 : 0;
  if (src && src->stage) {
    // pinned host records -> device staging buffer (DMA), then read from HBM
    const int64_t m = src->n;
    char* rec = static_cast<char*>(ws.recs.ensure(static_cast<size_t>(m) * 17 + 64));
    double* dlon = reinterpret_cast<double*>(rec);
    double* dlat = dlon + m;
    uint8_t* dpr = reinterpret_cast<uint8_t*>(dlat + m);
    THMM_CUDA(cudaMemcpyAsync(dpr, src->present, m, cudaMemcpyDefault, s));
    THMM_CUDA(cudaMemcpyAsync(dlon, src->lon, m * sizeof(double), cudaMemcpyDefault, s));
    THMM_CUDA(cudaMemcpyAsync(dlat, src->lat, m * sizeof(double), cudaMemcpyDefault, s));
    ca.present = dpr;
    ca.lon = dlon;
    ca.lat = dlat;
    ca.sysmem = 0;
  }
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
  if (collapse) {
    const int64_t nodes = static_cast<int64_t>(B) * total;
    double* col = static_cast<double*>(ws.col.ensure(sizeof(double) * nodes * (3 * KP + 2)));
    ca.collapse_tol = collapse_tol();
    ca.collapse_win = collapse_win();
    ca.col_r = col;
    ca.col_d = col + nodes * KP;
    ca.col_c = col + 2 * nodes * KP;
    ca.col_meta = col + 3 * nodes * KP;
    ws.col_nodes = nodes;
    ws.col_kp = KP;
  }
  g_prof_segments = total;
  g_prof_runs = use_runs_kernel;
  g_prof_collapse = collapse;
  g_prof_stitch = false;
  const bool prof = g_profile && prof_events(obs->device);
  if (st_segs > 0) {
    // Stitched chain (thmm_vec.cuh): main pass + links + finish, no K x K products.
    double* res = static_cast<double*>(ws.result.ensure(2 * sizeof(double) * B));
    ca.lo = lo;
    ca.n = n;
    StitchStage stage{};
    const int hmode = src && !src->stage ? stitch_host_mode(src->ratio[0]) : 0;
    const bool staged = hmode == 1 && lo == 0 && hi == src->n;
    if (hmode == 2) ca.sysmem = 2;
    if (staged) {
      // pinned host records -> HBM by DMA (55 GB/s on B200, vs ~28 GB/s of
      // uncached zero-copy reads), in time chunks the main pass follows
      const int64_t m = src->n;
      char* rec = static_cast<char*>(ws.recs.ensure(static_cast<size_t>(m) * 17 + 64));
      stage = StitchStage{src->present, src->lon, src->lat, reinterpret_cast<uint8_t*>(rec + 16 * m),
                          reinterpret_cast<double*>(rec), reinterpret_cast<double*>(rec) + m};
      ca.present = stage.d_present;
      ca.lon = stage.d_lon;
      ca.lat = stage.d_lat;
      ca.sysmem = 0;
    }
    enqueue_stitched(obs, ca, total, 1, s, prof, res, nullptr, nullptr, 0, nullptr, staged ? &stage : nullptr);
    return;
  }
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
      if (runs)
        launch_chain_runs(ca, plan, (c_nseg[c] + plan.G - 1) / plan.G, cs);
      else
        launch_chain(ca, plan, cfg->precision, (c_nseg[c] + plan.G - 1) / plan.G, cs);
      THMM_CUDA(cudaEventRecord(obs->chunk_done[c], cs));
    } else {
      if (ready) THMM_CUDA(cudaStreamWaitEvent(s, ready[c], 0));
      if (use_runs_kernel)
        launch_chain_runs(ca, plan, (c_nseg[c] + plan.G - 1) / plan.G, s);
      else
        launch_chain(ca, plan, cfg->precision, (c_nseg[c] + plan.G - 1) / plan.G, s);
      if (collapse) {
        if (prof) THMM_CUDA(record_prof(g_prof_ev[3], s));
        const ChainPlan& vp = vec_plan(obs->device, K);
        launch_chain_vec(ca, vp, vec_spread(vp, B, (c_nseg[c] + 7) / 8), s);
      }
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
  float c = 0.f;
  if ((g_prof_collapse || g_prof_stitch) && cudaEventElapsedTime(&c, g_prof_ev[0], g_prof_ev[3]) == cudaSuccess) {
    g_prof_burn_ms = c;  // collapse: burn-in | stitch: main pass
    g_prof_vec_ms = g_prof_chain_ms - c;  // collapse: vector continuation | stitch: links
  } else {
    cudaGetLastError();
    g_prof_burn_ms = g_prof_vec_ms = -1.0;
  }
}

// Results (loglik[B] | status[B]) land in the head of the pinned staging
// buffer (the parameter upload that used it is stream-ordered before).
void enqueue_results(Workspace& ws, int B, cudaStream_t s) {
  double* res = static_cast<double*>(ws.result.ptr);
  double* host = static_cast<double*>(ws.staging.ensure(2 * sizeof(double) * B));
  // loglik[B] doubles then status[B] int32 (the tail of the status half is padding)
  THMM_CUDA(cudaMemcpyAsync(host, res, (sizeof(double) + sizeof(int32_t)) * B, cudaMemcpyDeviceToHost, s));
}

// Internal return code: a stitched evaluation's link did not converge; the
// caller repeats the evaluation without the stitch (rerun_without_stitch).
constexpr int kStitchFailed = 77;

int read_results(Workspace& ws, int B, cudaStream_t s, double* out, int32_t* status) {
  THMM_CUDA(cudaStreamSynchronize(s));
  const double* host = static_cast<const double*>(ws.staging.ptr);
  const int32_t* st = reinterpret_cast<const int32_t*>(host + B);
  int rc = THMM_OK;
  for (int b = 0; b < B; ++b)
    if (st[b] == 3) return kStitchFailed;  // (the tree reports collapse as 2, the stitched finish as 1)
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
                        w.exps_a.ptr, w.exps_b.ptr, w.result.ptr, w.counters.ptr, w.staging.ptr, w.col.ptr,
                        w.stitch.ptr, w.recs.ptr};
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
  g_launches = 0;
  try {
    run_range(obs, P, cfg, cs, true, nullptr, nullptr);
    enqueue_results(obs->ws, P->B, cs);
  } catch (const CudaError&) {
    ok = false;
  }
  g_capturing = false;
  const int launches = g_launches;
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
  slot->runs = g_prof_runs;
  slot->runs_key = runs_for(obs, P->K, cfg->precision, hi - cfg->lo);
  slot->cmode = collapse_env();
  slot->launches = launches;
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

// After a stitched evaluation reported a link that did not converge: once
// more stitched with segments twice as long (links get twice the records),
// then, if a link still fails, on the rank-one collapse / matrix path (exact
// in every case).
int rerun_without_stitch(thmm_obs obs, const thmm_params* P, const thmm_config* cfg, cudaStream_t s,
                         const MappedSource* src, double* out, int32_t* status) {
  ++g_stitch_reruns;
  g_stitch_len_scale = 2;
  int rc = kStitchFailed;
  try {
    run_range(obs, P, cfg, s, true, nullptr, nullptr, 1, nullptr, nullptr, src);
    rc = finish_results(obs->ws, P->B, s, out, status);
  } catch (...) {
    g_stitch_len_scale = 1;
    throw;
  }
  g_stitch_len_scale = 1;
  if (rc != kStitchFailed) return rc;
  g_no_stitch = true;
  try {
    run_range(obs, P, cfg, s, true, nullptr, nullptr, 1, nullptr, nullptr, src);
  } catch (...) {
    g_no_stitch = false;
    throw;
  }
  g_no_stitch = false;
  return finish_results(obs->ws, P->B, s, out, status);
}

int translate(const CudaError& e, char* err, size_t errlen) {
  set_err(err, errlen, "CUDA error %s (%s) in %s", cudaGetErrorName(e.code), cudaGetErrorString(e.code), e.what);
  return THMM_ECUDA;
}

int check_cfg_n(int64_t n, const thmm_config* cfg, char* err, size_t errlen);

int check_cfg(thmm_obs obs, const thmm_config* cfg, char* err, size_t errlen) { return check_cfg_n(obs->n, cfg, err, errlen); }

int check_cfg_n(int64_t n, const thmm_config* cfg, char* err, size_t errlen) {
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
  const int64_t hi = cfg->hi > 0 ? cfg->hi : n;
  if (cfg->lo < 0 || hi > n || cfg->lo >= hi) {
    set_err(err, errlen, "observation range [%lld, %lld) is empty or outside the stream of %lld records",
            (long long)cfg->lo, (long long)hi, (long long)n);
    return THMM_EINVAL;
  }
  return THMM_OK;
}

// Step-count estimates of the run-absorbing chain from host flags (overlaps
// the asynchronous upload); unknown (never chosen automatically) without them.
void set_runs_ratios(thmm_obs obs, const uint8_t* host_present, int64_t n) {
  for (auto& r : obs->runs_ratio) r = -1.0;
  if (host_present) estimate_runs_ratios(host_present, n, obs->runs_ratio);
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
  set_runs_ratios(obs, kind == cudaMemcpyHostToDevice ? present : nullptr, n);
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
    // Geometric chunks: chunk c+1 is R times chunk c, R ~ copy rate / chain
    // rate.  Chain-bound (R > 1): growing chunks, so each chunk's copy hides
    // under the previous chunk's chain and the GPU waits only for the small
    // first chunk.  Copy-bound (R < 1, e.g. the run-absorbing chain on sparse
    // streams): shrinking chunks, so the chain of the last (small) chunk is all
    // that runs after the copy engine finishes.  The smallest chunk stays >=
    // kMinFirstChunk records; few chunks keep the per-launch tails few.  Whole-
    // stream evaluations only (ranges and explicit segment counts keep the
    // single-launch schedule).
    set_runs_ratios(obs, present, n);
    const bool whole = cfg->lo == 0 && (cfg->hi == 0 || cfg->hi == n) && cfg->segments == 0;
    std::fill(bounds, bounds + 9, int64_t{0});
    int chunks = 1;
    bounds[1] = n;
    if (whole && n >= 2 * kMinFirstChunk) {
      const int K = params->K, KP = padded(K);
      // records/s of the chain (B200 measurements at K=25: 26 TF record by
      // record, 23 TF per step of the run-absorbing chain) and of the copy
      // engine (42-48 GB/s for multi-MB pinned copies, measured in round 1)
      double chain_rate = 26e12 / (2.0 * K * K * K * params->B);
      if (runs_for(obs, K, cfg->precision))
        chain_rate = 23e12 / (2.0 * K * K * K * params->B) * K / (KP * obs_runs_ratio(obs, K));
      const double copy_rate = 42e9 / 17.0;
      double R = copy_rate / chain_rate;
      R = R >= 1.0 ? std::min(8.0, std::max(1.2, R)) : std::max(0.5, std::min(1.0 / 1.2, R));
      int C = 1;
      double sum = 1.0;
      while (C < 8) {  // largest chunk count whose smallest chunk stays >= kMinFirstChunk
        const double next_sum = sum + std::pow(R, C);
        const double smallest = std::min(1.0, std::pow(R, C));
        if (static_cast<double>(n) * smallest / next_sum < kMinFirstChunk) break;
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
    if (!whole) {  // one copy of the whole stream; the evaluation covers [lo, hi) (bounds relative to lo)
      bounds[0] = 0;
      bounds[1] = (cfg->hi > 0 ? cfg->hi : n) - cfg->lo;
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
  slot->mapped = false;
  slot->runs = g_prof_runs;
  slot->cmode = collapse_env();
  slot->precision = cfg->precision;
  slot->period = cfg->renorm_period;
  slot->segments = cfg->segments;
  slot->lo = cfg->lo;
  slot->hi = cfg->hi;
  slot->prof = prof;
  slot->signature = sig;
  slot->nseg = g_prof_segments;
  slot->launches = launches;
  slot->exec = exec;
  slot->last_use = ++obs->uses;
  slot->valid = true;
}

// Zero-copy source: all three arrays pinned and device-mapped (UVA), and
// not disabled with THMM_ZEROCOPY=0.  Fills the device-usable pointers.
bool mapped_source(const uint8_t* present, const double* lon, const double* lat, int64_t n, MappedSource& src) {
  static const bool enabled = [] {
    const char* v = std::getenv("THMM_ZEROCOPY");
    return !(v && v[0] == '0');
  }();
  if (!enabled) return false;
  const void* in[3] = {present, lon, lat};
  void* dev[3] = {};
  for (int i = 0; i < 3; ++i) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, in[i]) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (a.type != cudaMemoryTypeHost || a.devicePointer == nullptr) return false;
    dev[i] = a.devicePointer;
  }
  src.present = static_cast<const uint8_t*>(dev[0]);
  src.lon = static_cast<const double*>(dev[1]);
  src.lat = static_cast<const double*>(dev[2]);
  src.n = n;
  src.host_present = present;
  return true;
}

// Step-count estimates of the run-absorbing chain for a zero-copy source
// (sampled host flags); only needed when an evaluation is enqueued, not when
// a recorded graph is replayed.
void estimate_source(MappedSource& src) {
  if (!src.estimated && src.host_present) {
    estimate_runs_ratios(src.host_present, src.n, src.ratio);
    src.estimated = true;
  }
}

// Record a zero-copy evaluation (params H2D, chain reading host memory, tree,
// result D2H) as a CUDA graph keyed by the host buffers.
void capture_mapped_graph(thmm_obs obs, const void* const* host, const MappedSource& src, const thmm_params* P,
                          const thmm_config* cfg, cudaStream_t s, bool prof) {
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
    run_range(obs, P, cfg, s, true, nullptr, nullptr, 1, nullptr, nullptr, &src);
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
  for (int i = 0; i < 3; ++i) slot->src[i] = host[i];
  slot->n = src.n;
  slot->K = P->K;
  slot->B = P->B;
  slot->runs = g_prof_runs;
  slot->cmode = collapse_env();
  slot->mapped = true;
  slot->precision = cfg->precision;
  slot->period = cfg->renorm_period;
  slot->segments = cfg->segments;
  slot->lo = cfg->lo;
  slot->hi = cfg->hi;
  slot->prof = prof;
  slot->signature = sig;
  slot->nseg = g_prof_segments;
  slot->launches = launches;
  slot->exec = exec;
  slot->last_use = ++obs->uses;
  slot->valid = true;
}

}  // namespace

namespace {

// Multi-GPU stitched chain, one rank's part (thmm_stitch_shard / thmm_stitch_link).
// host: the shard's records from host memory (n records; page-locked for
// an overlapped copy) -- they replace the handle's records, staged by DMA in
// time chunks the main pass follows (thmm_stitch_shard_host).
struct HostShard {
  const uint8_t* present;
  const double* lon;
  const double* lat;
  int64_t n;
};

int stitch_shard_impl(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, int first, double* d_block,
                      const double* d_prev, int64_t prev_stride, double* d_link, char* err, size_t errlen,
                      const HostShard* host = nullptr) {
  g_launches = 0;
  if (!obs || (!d_block && !d_link)) {
    set_err(err, errlen, "null observation handle or output");
    return THMM_EINVAL;
  }
  int rc = validate_params(params, err, errlen);
  if (rc != THMM_OK) return rc;
  std::lock_guard<std::mutex> lk(obs->mu);
  rc = host ? check_cfg_n(host->n, cfg, err, errlen) : check_cfg(obs, cfg, err, errlen);
  if (rc != THMM_OK) return rc;
  if (cfg->lo != 0 || cfg->hi != 0) {
    set_err(err, errlen, "a stitched shard covers the handle's whole stream");
    return THMM_EINVAL;
  }
  try {
    DeviceGuard dg(obs->device);
    const int K = params->K, B = params->B;
    StitchStage stage{};
    if (host) {
      // the records are replaced below, asynchronously; wait for earlier readers
      if (obs->ws.staged_pending && obs->ws.staged) THMM_CUDA(cudaStreamWaitEvent(obs->stream, obs->ws.staged, 0));
      ensure_obs_capacity(obs, host->n);
      obs->n = host->n;
      set_runs_ratios(obs, host->present, host->n);
      stage = StitchStage{host->present, host->lon, host->lat, obs->present, obs->lon, obs->lat};
    }
    const int64_t total =
        stitch_segments(obs->device, K, cfg, obs->n, B, runs_for(obs, K, cfg->precision) ? obs_runs_ratio(obs, K) : 1.0,
                        -1.0, obs->runs_ratio[0]);
    if (total < 1) {
      if (host) {  // the handle still holds the new records (for the caller's fallback)
        rc = upload_obs(obs, host->present, host->lon, host->lat, host->n, cudaMemcpyHostToDevice, err, errlen);
        if (rc == THMM_OK) THMM_CUDA(cudaStreamSynchronize(obs->stream));
      }
      set_err(err, errlen, "shard too short for the stitched chain");
      return THMM_EINVAL;
    }
    cudaStream_t s = pick_stream(obs, cfg);
    Workspace& ws = obs->ws;
    thmm::StateParams sp = upload_params(ws, params, s);
    thmm::ChainArgs ca{};
    ca.present = obs->present;
    ca.lon = obs->lon;
    ca.lat = obs->lat;
    ca.K = K;
    ca.B = B;
    ca.period = cfg->renorm_period;
    ca.neg_log_2pi = -std::log(2.0 * M_PI);
    ca.P = sp;
    ca.lo = 0;
    ca.n = obs->n;
    const bool prof = g_profile && prof_events(obs->device) && !d_prev;
    if (host && s != obs->stream) {  // the copies follow s: order s after the handle's own stream too
      cudaEvent_t ev;
      THMM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      THMM_CUDA(cudaEventRecord(ev, obs->stream));
      THMM_CUDA(cudaStreamWaitEvent(s, ev, 0));
      THMM_CUDA(cudaEventDestroy(ev));  // (released once the wait has been satisfied)
    }
    enqueue_stitched(obs, ca, total, first, s, prof, nullptr, d_block, d_prev, prev_stride, d_link,
                     host ? &stage : nullptr);
    THMM_CUDA(cudaEventRecord(staged_event(obs->ws), s));
    return THMM_OK;
  } catch (const CudaError& e) {
    return translate(e, err, errlen);
  }
}

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
