/*
 * thmm.h -- C-ABI of the B200-native HMM forward log-likelihood.
 *
 * This is the drop-in boundary for the reference's parallel likelihood engine
 * (tremorhmm, /root/reference/pkg/src/tremorhmm).  Every entry point takes
 * plain pointers and sizes; no torch or numpy types cross it.  The Python
 * mirror of the reference API (paper_2003_03508_b200/engine.py) binds these
 * with ctypes; INTEGRATION.md shows the binding a tremorhmm maintainer would
 * add.
 *
 * Chain convention (reference core.py:7, 281-289; engine.py:3-11):
 *     L = delta' (Gamma P(x_0)) (Gamma P(x_1)) ... (Gamma P(x_{N-1})) 1
 * with P(x) = diag(p_k phi_k(x)) for a located event, diag(1 - p_k) for a
 * quiet hour.
 *
 * Return codes: THMM_OK, THMM_EINVAL (-> ValueError), THMM_ECOLLAPSE
 * (-> RuntimeError, reference engine.py:313-315), THMM_ECUDA (-> RuntimeError).
 * On error a message is written to err[0..errlen) when err is non-NULL.
 *
 * Threading: calls on distinct observation handles are independent; calls on
 * one handle are serialised by the handle's mutex.  All results are
 * deterministic (fixed reduction order, no floating-point atomics), matching
 * the reference's run-to-run bitwise determinism (engine.py:15-16).
 */
#ifndef THMM_H
#define THMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define THMM_OK 0
#define THMM_EINVAL 1
#define THMM_ECOLLAPSE 2
#define THMM_ECUDA 3

/* Largest supported state count; reference engine.py:39 (MAX_PARALLEL_STATES). */
#define THMM_MAX_STATES 80

/* Precision codes for thmm_config.precision; reference EngineConfig.precision
 * ("float64" | "float32"), engine.py:64, 73-74. */
#define THMM_F64 0
#define THMM_F32 1
/* Precision-study extensions (BASELINE.json configs[3]): the float32
 * semantics of THMM_F32 with the chain products on the tcgen05 tensor cores,
 * TF32 operands (THMM_TF32), hi+lo split 3xTF32 operands (THMM_TF32X3), or
 * split Gamma only, rows rounded to tf32 (THMM_TF32X2). */
#define THMM_TF32 2
#define THMM_TF32X3 3
#define THMM_TF32X2 4

/* Opaque device-resident observation stream (present u8, lon f64, lat f64).
 * Replaces the per-call `observation_arrays` + `_emission_columns` inputs of
 * reference engine.py:321-329 / core.py:209-260: the stream is uploaded once
 * and reused by every likelihood evaluation (the MCMC loop of bayes.py:712-715
 * builds its arrays once as well). */
typedef struct thmm_obs_s* thmm_obs;

/* B parameter sets sharing K, structure-of-arrays, host memory, float64.
 *   gamma  [B][K][K] row-major          (HmmParams.gamma, core.py:131)
 *   delta  [B][K]                       (HmmParams.delta, core.py:132)
 *   states [8][B][K] in the order p, q=1-p, mu0, mu1, l00, l10, l11, log_det
 *          (HmmParams._p ... _log_det, core.py:162-169; the 2x2 Cholesky of
 *          core.py:33-53 and log_det of core.py:119 are done by the host). */
typedef struct {
  int32_t K;
  int32_t B;
  const double* gamma;
  const double* delta;
  const double* states;
} thmm_params;

/* Engine knobs; reference EngineConfig (engine.py:49-81).
 *   renorm_period  steps between renormalisations (>= 1; default 8)
 *   precision      THMM_F64, THMM_F32, THMM_TF32, THMM_TF32X3 or THMM_TF32X2
 *   segments       chain segments per proposal; 0 = fill the GPU
 *   lo, hi         sub-range [lo, hi) of the stream (hi == 0: whole stream);
 *                  used by the multi-GPU shard of reference segment_bounds
 *                  (engine.py:97-111)
 *   stream         cudaStream_t to launch on; NULL = the handle's stream */
typedef struct {
  int32_t renorm_period;
  int32_t precision;
  int64_t segments;
  int64_t lo;
  int64_t hi;
  void* stream;
} thmm_config;

/* Library version (major*10000 + minor*100 + patch). */
int thmm_version(void);

/* Number of visible CUDA devices (0 when none). */
int thmm_device_count(void);

/* Padded state count the device kernels use for K (multiple of 8). */
int thmm_padded_states(int32_t K);

/* Upload an observation stream to `device`.  The host arrays stay owned by
 * the caller.  n must be >= 1 (reference engine.py:324-325 rejects empty). */
int thmm_obs_create(const uint8_t* present, const double* lon, const double* lat,
                    int64_t n, int device, thmm_obs* out, char* err, size_t errlen);

/* Re-upload into an existing handle (capacity grows as needed). */
int thmm_obs_assign(thmm_obs obs, const uint8_t* present, const double* lon,
                    const double* lat, int64_t n, char* err, size_t errlen);

/* Upload from device memory already on the handle's device (no host copy). */
int thmm_obs_assign_device(thmm_obs obs, const uint8_t* d_present, const double* d_lon,
                           const double* d_lat, int64_t n, char* err, size_t errlen);

int thmm_obs_destroy(thmm_obs obs);
int64_t thmm_obs_length(thmm_obs obs);
int thmm_obs_device(thmm_obs obs);

/* Page-lock and device-map a caller-owned host range (cudaHostRegister,
 * mapped + portable) so the host-array entries read it in place over PCIe
 * (zero-copy) instead of staging a copy.  The reference's MCMC driver passes
 * the same observation arrays on every likelihood call (bayes.py:709-715):
 * the Python mirror registers them on first use and unregisters them when
 * the array is released.  Returns 0, or THMM_EINVAL when the range is
 * already (partly) registered or cannot be locked (the caller then takes
 * the copy path).  thmm_host_unregister: 0 or THMM_EINVAL. */
int thmm_host_register(const void* ptr, size_t bytes, char* err, size_t errlen);
int thmm_host_unregister(const void* ptr);

/* Log-likelihood of each of the B parameter sets over the stream range.
 * Replaces reference engine._parallel_loglik_arrays (engine.py:321-345) for
 * B == 1 and adds the batched-proposal entry point for B > 1.
 *   out     [B] host doubles; collapsed proposals get -inf
 *   status  [B] host int32 (THMM_OK / THMM_ECOLLAPSE), may be NULL
 * Returns THMM_ECOLLAPSE when any proposal collapsed. */
int thmm_loglik(thmm_obs obs, const thmm_params* params, const thmm_config* cfg,
                double* out, int32_t* status, char* err, size_t errlen);

/* Host-array entry (reference engine._parallel_loglik_arrays with numpy
 * arrays, engine.py:321-345): copies `n` records from HOST memory into the
 * handle (capacity grows) and evaluates them, pipelined -- the stream is cut
 * into up to 8 chunks whose host->device copies run on a copy stream while
 * the chain kernel of the previous chunk runs (pinned host memory gives full
 * copy bandwidth).  The handle keeps the records afterwards. */
int thmm_loglik_host(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                     const thmm_params* params, const thmm_config* cfg, double* out, int32_t* status,
                     char* err, size_t errlen);

/* Zero-copy host-array entry: when present/lon/lat are pinned (page-locked,
 * device-mapped) host memory the chain kernels read the records in place
 * over PCIe -- uncached loads, coordinates only for present records, no
 * staging copy and no chunk pipeline -- so the transfer overlaps the whole
 * chain.  The handle's own record buffers are neither used nor changed (its
 * workspace and graphs are).  Pageable arrays (or THMM_ZEROCOPY=0) fall back
 * to thmm_loglik_host.  The arrays must stay valid and unmodified for the
 * call.  cfg->lo/hi index the host arrays. */
int thmm_loglik_mapped(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                       const thmm_params* params, const thmm_config* cfg, double* out, int32_t* status,
                       char* err, size_t errlen);

/* Reduce the stream range [cfg->lo, cfg->hi) of every proposal to one scaled
 * product node: value = 2^e * m, m [KP][KP] (KP = thmm_padded_states(K)) with
 * max entry in [1, 2) (or all zero).  Outputs are DEVICE pointers on the
 * handle's device:  d_m [B][KP][KP], d_e [B].  This is one GPU's share of the
 * segment chain (reference engine.py:336-344); the shares are exchanged with
 * NCCL all-gather and folded by thmm_fold_nodes. */
int thmm_range_nodes(thmm_obs obs, const thmm_params* params, const thmm_config* cfg,
                     double* d_m, double* d_e, char* err, size_t errlen);

/* thmm_range_nodes without the host synchronisation: the nodes are valid once
 * the launch stream (cfg->stream, else the handle's) reaches this point, so a
 * collective and thmm_fold_nodes_strided can be queued behind it. */
int thmm_range_nodes_async(thmm_obs obs, const thmm_params* params, const thmm_config* cfg,
                           double* d_m, double* d_e, char* err, size_t errlen);

/* thmm_range_nodes_async over HOST arrays: the n records replace the stream
 * (as thmm_obs_assign) with the host->device copy pipelined against the
 * chain kernels (geometric chunks on the handle's copy stream, as
 * thmm_loglik_host), nothing synchronised.  Pinned (device-mapped) arrays
 * are instead read in place by the kernels (zero-copy, as
 * thmm_loglik_mapped) and the handle keeps its own records.  The host arrays must stay valid
 * (and unmodified) until the launch stream has passed this call, e.g. until
 * the thmm_fold_nodes_strided that consumes the nodes returns.  cfg->lo/hi
 * must be 0.  One GPU's share of a sharded evaluation from host memory. */
int thmm_range_nodes_host(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat,
                          int64_t n, const thmm_params* params, const thmm_config* cfg,
                          double* d_m, double* d_e, char* err, size_t errlen);

/* Ordered fold of G nodes per proposal into the log-likelihood; the device
 * analogue of reference combine_segments (engine.py:292-318).
 *   d_m [G][B][KP][KP], d_e [G][B] device pointers on `device`
 *   out [B] host, status [B] host (may be NULL). */
int thmm_fold_nodes(const thmm_params* params, int32_t G, const double* d_m, const double* d_e,
                    int device, void* stream, double* out, int32_t* status,
                    char* err, size_t errlen);

/* thmm_fold_nodes over an arbitrary [G][B] node layout: node (g, b) at
 * d_m + g*m_stride_g + b*KP*KP doubles, its exponent at d_e[g*e_stride_g + b]
 * (e.g. the packed per-rank blocks of one all-gather, see distributed.py).
 * Node rows are read as 16-byte vectors: d_m must be 16-byte aligned and
 * m_stride_g even (THMM_EINVAL otherwise). */
int thmm_fold_nodes_strided(const thmm_params* params, int32_t G, const double* d_m, int64_t m_stride_g,
                            const double* d_e, int64_t e_stride_g, int device, void* stream,
                            double* out, int32_t* status, char* err, size_t errlen);

/* Peer-memory combine for one process per GPU over NVLink / NVSwitch (the
 * B200-native replacement of the NCCL all-gather + fold of the sharded
 * path).  Each rank creates a mailbox of 2 x world x slot_doubles doubles
 * (slot_doubles >= B*KP*KP + B) and exports its CUDA IPC handle (64 bytes);
 * the handles are exchanged out of band (torch.distributed) and opened with
 * thmm_peer_open (world x 64 bytes, rank order).  thmm_peer_loglik reduces
 * this rank's stream to root nodes written into its own mailbox slot, stores
 * them into every peer's mailbox with P2P stores and a release-ordered epoch
 * flag, acquires every peer's flag, and folds the world's nodes in rank order
 * -- every rank returns the identical values.  present/lon/lat/n, when
 * non-NULL, are this rank's records from host memory (as
 * thmm_range_nodes_host: pinned arrays read in place, pageable ones
 * replace the stream).  A peer that never publishes makes the call fail
 * with THMM_ECUDA after ~4 s instead of hanging. */
typedef struct thmm_peer_s* thmm_peer;
int thmm_peer_create(int device, int rank, int world, int64_t slot_doubles, thmm_peer* out, void* ipc_handle,
                     char* err, size_t errlen);
int thmm_peer_open(thmm_peer peer, const void* handles, char* err, size_t errlen);
int thmm_peer_loglik(thmm_peer peer, thmm_obs obs, const uint8_t* present, const double* lon, const double* lat,
                     int64_t n, const thmm_params* params, const thmm_config* cfg, double* out, int32_t* status,
                     char* err, size_t errlen);
int thmm_peer_destroy(thmm_peer peer);

/* Filtered distribution of the state one step past the stream range, per
 * proposal: normalise(delta' Gamma P(x_lo) ... Gamma P(x_{hi-1})) Gamma,
 * normalised (reference simforecast._filtered_next_state_dist,
 * simforecast.py:97-118, which conditions forecasts on a history).
 *   out [B][K] host; status [B] (THMM_ECOLLAPSE: zero-likelihood history). */
int thmm_filtered_state(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, double* out,
                        int32_t* status, char* err, size_t errlen);

/* Emission diagonals for records [lo, hi) of the stream, parameter set 0:
 * out [(hi-lo)][K] host.  Reference batch_emissions / _emission_columns
 * (engine.py:234-243, core.py:235-260). */
int thmm_emissions(thmm_obs obs, const thmm_params* params, int64_t lo, int64_t hi,
                   double* out, char* err, size_t errlen);

/* Diagnostic: the same table computed with the chain kernels' emission
 * arithmetic (Cholesky divisions refined from correctly rounded reciprocals,
 * csrc/thmm_kernels.cuh emission_rc -- the values the likelihood actually
 * multiplies by), so tests can hold the hot path's emissions against the
 * reference's _emission_columns (core.py:235-260) directly. */
int thmm_emissions_chain(thmm_obs obs, const thmm_params* params, int64_t lo, int64_t hi,
                         double* out, char* err, size_t errlen);

/* Segment products over an explicit factor stack (reference
 * segment_chain_product, engine.py:259-289): factors [n][K][K] host,
 * nonnegative; out_m [S][K][K] host normalised (max == 1 or zero),
 * out_log_scale [S] host, with S = segments and segment_bounds(n, S). */
int thmm_factor_segments(const double* factors, int64_t n, int32_t K, int64_t segments,
                         int32_t renorm_period, int device, double* out_m,
                         double* out_log_scale, char* err, size_t errlen);

/* Stationary distributions of B row-stochastic K x K matrices in one launch
 * (reference core.stationary_distribution, core.py:350-388: power iteration
 * from the uniform vector, stop when the max-norm change < tol, at most
 * max_iter sweeps; the reference uses tol = 1e-12, max_iter = 1e5).
 *   gammas [B][K][K] host, out [B][K] host, status [B] (THMM_ECOLLAPSE =
 *   not converged; the call then returns THMM_ECOLLAPSE -> RuntimeError). */
int thmm_stationary(const double* gammas, int32_t K, int32_t B, double tol, int32_t max_iter, int device,
                    double* out, int32_t* status, char* err, size_t errlen);

/* Observation CSV ingestion (reference dataio.load_dataset, dataio.py:46-87):
 * header `timestamp,lon,lat`, one row per hour, both coordinates empty for a
 * quiet hour, ISO-8601 timestamps strictly increasing.  Malformed input gives
 * THMM_EINVAL with the reference's "line N: ..." message.  Two passes:
 * thmm_csv_count for the record count, thmm_csv_read to fill caller arrays
 * (t_us = timestamps in microseconds since the epoch, may be NULL).  No GPU
 * needed; the arrays feed thmm_obs_create. */
int thmm_csv_count(const char* path, int64_t* n, char* err, size_t errlen);
int thmm_csv_read(const char* path, int64_t n, uint8_t* present, double* lon, double* lat, int64_t* t_us,
                  char* err, size_t errlen);

/* Number of kernels the calling thread launched in its last thmm_* call. */
int thmm_last_launch_count(void);

/* Kernel timing for the benchmark: when enabled (per calling thread), the
 * likelihood calls bracket the chain kernel and the fold kernels with CUDA
 * events on the launch stream; thmm_profile_last reports the device times of
 * the calling thread's last call and the segment count it used. */
int thmm_profile_enable(int on);
int thmm_profile_last(double* chain_ms, double* fold_ms, int64_t* segments);

/* Launch plan the engine uses for K states at `precision` on `device`:
 * DMMA head tiles (nt), SIMT tail states (tail), segments stacked per CTA (G),
 * warps per CTA (W), registers per thread, resident CTAs per SM.
 * Diagnostic; no kernel runs. */
int thmm_plan_info(int32_t K, int32_t precision, int device, int32_t* nt, int32_t* tail, int32_t* G,
                   int32_t* W, int32_t* regs, int32_t* ctas_per_sm);

/* Run-absorbing chain (FP64): a run of r absent records multiplies the
 * product by the fixed matrix (Gamma diag(1-p))^r, so one MMA step with a
 * precomputed power replaces up to R records (R = 16, 8, 4 or 3 by K: the
 * table of powers must fit in shared memory).  The engine picks it per
 * evaluation from the handle's estimated steps per record (sampled from the
 * host flags at upload) and a cost model; THMM_RUNS=0/1 in the environment
 * (or thmm_set_runs_mode) forces it off/on.  Reports whether `obs` would use
 * it for (K, precision), the estimated steps per record (< 0 unknown), its
 * launch plan and R.  Diagnostic; no kernel runs. */
int thmm_runs_info(thmm_obs obs, int32_t K, int32_t precision, int32_t* active, double* steps_per_record,
                   int32_t* G, int32_t* W, int32_t* regs, int32_t* ctas_per_sm, int32_t* R);

/* 1 if the calling thread's last likelihood call ran the run-absorbing chain. */
int thmm_profile_runs(void);

/* Process-wide run-absorbing chain mode: -1 automatic (default), 0 never,
 * 1 always (whenever eligible: FP64).  Overrides THMM_RUNS. */
int thmm_set_runs_mode(int mode);

/* Rank-one collapse of converged segment products (csrc/thmm_vec.cuh): 1 on
 * (default; THMM_COLLAPSE=0 in the environment starts it off), 0 off.  The
 * FP64 likelihood is the same to within 1e-12 relative per segment either
 * way; tests run both. */
int thmm_set_collapse_mode(int mode);

/* Phase times of the last profiled evaluation, in ms: rank-one collapse
 * (returns 1): burn-in (run-absorbing chain up to the rank-one test) and
 * vector continuation; stitched chain (returns 2): main pass and links;
 * else returns 0 (both -1). */
int thmm_profile_phases(double* burn_ms, double* vec_ms);

/* Stitched chain (csrc/thmm_vec.cuh) for whole-chain evaluations in collapse
 * mode: 1 on (default; THMM_STITCH=0 starts it off), 0 off.  Evaluations
 * whose links do not converge are repeated on the collapse path; the counter
 * reports how many were. */
int thmm_set_stitch_mode(int mode);
long long thmm_stitch_reruns(void);

/* Multi-GPU stitched chain (one shard of the records per rank; reference
 * segment_bounds / combine_segments, engine.py:97-111, 292-318, restated on
 * forward rows instead of K x K nodes).  Asynchronous on cfg's stream.
 *   thmm_stitch_shard: the rank's records (cfg->lo = cfg->hi = 0) reduced to
 *     d_block [B][KP + 2] (device): the final normalised forward row, the
 *     log-scale of the shard relative to its start vector (delta when `first`,
 *     else all-ones), and a fail flag (an internal link did not converge).
 *   thmm_stitch_link: the link into this shard from the previous rank's final
 *     rows (d_prev + b*prev_stride, KP doubles each, device): d_link [B][2] =
 *     log-scale term, fail flag.
 * log L = sum_r A_r + sum_{r>=1} link_r + log(final row of the last rank . 1).
 * THMM_EINVAL when the shard is too short for the stitched path (the caller
 * exchanges thmm_range_nodes nodes instead). */
int thmm_stitch_shard(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, int32_t first,
                      double* d_block, char* err, size_t errlen);
int thmm_stitch_link(thmm_obs obs, const thmm_params* params, const thmm_config* cfg, const double* d_prev,
                     int64_t prev_stride, double* d_link, char* err, size_t errlen);
/* thmm_stitch_shard with this rank's records from host memory (present[n],
 * lon[n], lat[n]; page-locked for an overlapped copy): they replace the
 * handle's records, copied by DMA in time chunks that the main pass follows
 * (end-to-end evaluation of a sharded chain; reference engine.py:321-345 per
 * rank).  The host arrays must stay unchanged until cfg's stream has passed
 * the call.  On THMM_EINVAL "shard too short" the records are in the handle
 * (synchronously copied) for the caller's node-exchange fallback. */
int thmm_stitch_shard_host(thmm_obs obs, const uint8_t* present, const double* lon, const double* lat, int64_t n,
                           const thmm_params* params, const thmm_config* cfg, int32_t first, double* d_block,
                           char* err, size_t errlen);
/* Read the profiling events of this thread's last asynchronous evaluation
 * (thmm_stitch_shard) once its stream has passed them. */
int thmm_profile_collect(void);

/* Segments the stitched path would cut the handle's stream into for (K, B);
 * 0 = not eligible (too short, or stitch mode off). */
int64_t thmm_stitch_segments(thmm_obs obs, int32_t K, int32_t B);

/* Collapse parameters: per-entry relative tolerance of the rank-one test
 * (default 2^-40), the shortest segment of a collapse-mode split (default
 * 1024 records), and the gate B n >= min_fill x 1024 x (vector rows of one
 * wave), K > 8 (default 0.25; negative: no gate); 0 keeps the current value.
 * Diagnostics: segments of the handle's last collapse-mode evaluation, how
 * many collapsed, and the records they spent in the matrix burn-in. */
int thmm_set_collapse_params(double tol, int64_t min_len, double min_fill);
int thmm_collapse_stats(thmm_obs obs, int64_t* nodes, int64_t* collapsed, double* records_burned);

#ifdef __cplusplus
}
#endif

#endif /* THMM_H */
