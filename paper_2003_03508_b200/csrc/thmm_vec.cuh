// thmm_vec.cuh -- rank-one collapse of a segment product and the row-stacked
// vector continuation.
//
// The rows of a segment product M = Gamma P(x_lo) ... Gamma P(x_t) are the
// forward recursions started from every state (reference core.py:7-11,
// engine.py:133-179).  The forward filter forgets its start: after a few
// dozen records every row is a multiple of one common row, M = c r' (the
// product of positive-ish stochastic factors contracts to rank one).  Once
// that holds to working precision the rest of the segment needs ONE row:
//     c r' Gamma P(x_{t+1}) ... = c (r' Gamma P(x_{t+1}) ...),
// i.e. 2K^2 flops per record instead of 2K^3.
//
// Test (chain_runs_kernel, every 32-record window, collapse_tol > 0): rows are
// renormalised to max in [1, 2) by exact powers of two; the pivot p is the row
// with the largest exponent; the product is rank one when every entry of every
// nonzero row satisfies |m_ij - rho_i m_pj| <= tol rho_i m_pj + 2^-1022 (elementwise
// RELATIVE to the pivot: all later factors are nonnegative, so replacing M by
// c r' changes the likelihood by at most a factor (1 +- tol); the absolute
// slack is the FP64 normal floor relative to the row max, below which the
// reference's own renormalised arithmetic underflows too).  Then
// c_i = rho_i 2^(e_i - e_p) with rho_i = m_ij*/m_pj* at the pivot's largest
// entry j* (zero rows: c_i = 0) and r = 2^e_p m_p.  The group stores (r,
// d_i = e_i - e_p, rho_i, records consumed, e_p) and exits.
//
// chain_vec_kernel continues every collapsed segment from its row r over the
// rest of its records.  Rows of DIFFERENT segments now share the B operand
// (Gamma), so a warp stacks 8 segments into one m8n8k4 tile (the DMMA head +
// SIMT tail machinery of thmm_runs.cuh), each row scaled by the emission row
// of its own record.  Emissions are computed lane-per-state (the 8 rows'
// records broadcast from shared memory, no divergence) with the chain
// kernels' arithmetic (emission_rc).  The node of segment s is written as
// c r_final' (a K_p x K_p node in the tree's format), so the segment tree is
// unchanged.  Segments that never pass the test keep their full node from the
// matrix kernel (col_meta records -1) and are skipped here.
#pragma once

#include "thmm_runs.cuh"

namespace thmm {

// Time chunks of a staged main pass (ChainArgs::t_chunks): chunk c covers
// records [begin(c), begin(c+1)) of a segment of length L, begin(c) =
// floor(L t_frac[c]) -- the same expression on the host (copies) and here.
__host__ __device__ inline int64_t time_chunk_begin(int64_t L, const double* t_frac, int c) {
  return static_cast<int64_t>(static_cast<double>(L) * t_frac[c]);
}

// Records staged per window and row.
__host__ __device__ constexpr int vec_win(int) { return 32; }

__host__ __device__ constexpr int vec_slots(int kpe) { return (kpe + 31) / 32; }

// Emission rows per warp: one step's 8 (per-step mode) or the events of 8
// steps, at most 64 (batched mode, ChainArgs::ebatch).
constexpr int kVecBatchSteps = 8;
__host__ __device__ constexpr int vec_erows(bool batch) { return batch ? 8 * kVecBatchSteps : 8; }

// Shared memory: Gamma (runs entry layout) + the state constants, then per
// warp: the emission rows and the 8 rows' records of one window.
__host__ __device__ constexpr size_t vec_warp_bytes(int kpe, bool batch = false) {
  return static_cast<size_t>(8) * vec_win(kpe / 8) * 17 + static_cast<size_t>(vec_erows(batch)) * kpe * 8 +
         (batch ? 8 * kVecBatchSteps : 0);
}
__host__ __device__ constexpr size_t vec_smem_bytes(int nt, int tail, int warps, bool batch = false) {
  return static_cast<size_t>(runs_entry_pairs(nt, tail)) * 16 + static_cast<size_t>(10) * 8 * (nt + (tail > 0)) * 8 +
         64 * 8 + static_cast<size_t>(warps) * vec_warp_bytes(8 * (nt + (tail > 0)), batch);
}
// Warps per CTA (one CTA per SM): 20 for rows of <= 4 tiles (<= 96
// registers: no spills; two 16-warp CTAs at 64 registers spilled in the step
// loop and ran 4 % slower), 12 for wider rows (<= 168 registers: the
// accumulators plus the emission constants of SLOTS states stay in registers).
#ifndef THMM_VEC_WIDE_WARPS
#define THMM_VEC_WIDE_WARPS 12
#endif
__host__ __device__ constexpr int vec_warps(int rt) { return rt <= 4 ? 20 : THMM_VEC_WIDE_WARPS; }
__host__ __device__ constexpr int vec_min_blocks(int nt, int tail) { return nt + (tail > 0) <= 4 ? 1 : 1; }

__device__ __forceinline__ uint32_t vec_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Gamma of every proposal in the entry layout (one CTA per proposal), for the
// bulk copies of the row-stacked kernels' prologues.
template <int NT, int TAIL>
__global__ void __launch_bounds__(256) entry_prep_kernel(const ChainArgs args, double2* gent) {
  const int b = blockIdx.x, K = args.K;
  const double* gam = args.P.gamma + static_cast<size_t>(b) * K * K;
  runs_stage_entry<NT, TAIL>(gent + static_cast<size_t>(b) * runs_entry_pairs(NT, TAIL), K,
                             [&](int i, int j) { return gam[i * K + j]; });
}

// Stage Gamma (runs entry layout: one bulk copy of the prepared entry when
// args.gent, else permuted here) and the 10 per-state emission constants of
// proposal b (reciprocals of the Cholesky divisors included); CTA barrier.
// Row 1 of the constants (q = 1 - p, 0 for padding states) doubles as the
// emission row of a quiet record.
template <int NT, int TAIL>
__device__ __forceinline__ void vec_prologue(const ChainArgs& args, int b, double2* ent, double* csm) {
  constexpr int KPE = 8 * (NT + (TAIL > 0 ? 1 : 0));
  constexpr uint32_t kEntBytes = static_cast<uint32_t>(runs_entry_pairs(NT, TAIL)) * 16;
  const int K = args.K;
  __shared__ __align__(8) uint64_t ent_bar;
  if (args.gent) {
    // one bulk copy (TMA engine) of the prepared entry, completion counted on an mbarrier
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(vec_smem_u32(&ent_bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile(
          "{\n.reg .b64 st;\n"
          "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(vec_smem_u32(&ent_bar)),
          "r"(kEntBytes)
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              vec_smem_u32(ent)),
          "l"(args.gent + static_cast<size_t>(b) * runs_entry_pairs(NT, TAIL)), "r"(kEntBytes),
          "r"(vec_smem_u32(&ent_bar))
          : "memory");
    }
  } else {
    const double* gam = args.P.gamma + static_cast<size_t>(b) * K * K;
    runs_stage_entry<NT, TAIL>(ent, K, [&](int i, int j) { return gam[i * K + j]; });
  }
  for (int j = threadIdx.x; j < KPE; j += blockDim.x) {
    const double* st = args.P.states;
    double v[10] = {0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0, 0.0, 1.0, 1.0};  // padding states: harmless
    if (j < K) {
#pragma unroll
      for (int f = 0; f < 7; ++f) v[f] = st[(static_cast<size_t>(f) * args.B + b) * K + j];
      v[7] = __dsub_rn(args.neg_log_2pi, __dmul_rn(0.5, st[(static_cast<size_t>(7) * args.B + b) * K + j]));
      v[8] = __drcp_rn(v[4]);
      v[9] = __drcp_rn(v[6]);
    }
#pragma unroll
    for (int f = 0; f < 10; ++f) csm[f * KPE + j] = v[f];
  }
  for (int j = threadIdx.x; j < 64; j += blockDim.x) csm[10 * KPE + j] = kExp2Tab64[j];  // exp table
  __syncthreads();  // (also orders the barrier's initialisation before the waits below)
  if (args.gent) {
    const uint32_t bar = vec_smem_u32(&ent_bar);
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
          "selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar)
          : "memory");
    }
  }
}

// Per-warp shared memory of the row-stacked kernels.
struct VecWarpSmem {
  double* rx;           // [8][win]
  double* ry;           // [8][win]
  double* ebuf;         // [8][KPE]: emission rows of the step's events
  unsigned char* rf;    // [win][8]: 0 quiet, 1 event, 2 none (step-major: one 8-byte load per step)
  unsigned char* elist;  // batched mode: (step, row) index of each event slot of the 8-step batch
};
template <int KPE>
__device__ __forceinline__ VecWarpSmem vec_warp_smem(double* csm, int warp, bool batch) {
  constexpr int WIN = vec_win(KPE / 8);
  unsigned char* wsm =
      reinterpret_cast<unsigned char*>(csm + 10 * KPE + 64) + static_cast<size_t>(warp) * vec_warp_bytes(KPE, batch);
  VecWarpSmem w;
  w.ebuf = reinterpret_cast<double*>(wsm);
  w.rx = w.ebuf + vec_erows(batch) * KPE;
  w.ry = w.rx + 8 * WIN;
  w.rf = reinterpret_cast<unsigned char*>(w.ry + 8 * WIN);
  w.elist = w.rf + 8 * WIN;
  return w;
}

// Debug only (tools/vec_trace.cu defines THMM_VEC_TRACE): cycles per phase of
// the step loop, accumulated by every warp and written to args.trace by lane 0.
#ifdef THMM_VEC_TRACE
#define VEC_TR_DECL long long tr_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long tr_t = clock64();
#define VEC_TR(i) { const long long tr_n = clock64(); tr_acc[i] += tr_n - tr_t; tr_t = tr_n; }
#else
#define VEC_TR_DECL
#define VEC_TR(i)
#endif

// The forward recursion of the warp's 8 stacked rows, row g (= lane / 4)
// over records [start, start + len) of its own segment:
//     a <- (a Gamma) o e(record)       (renormalised every `period` steps)
// `hook(t, since)` runs after every step t (warp-uniform call); it may
// shorten `len` and returns true when the whole warp is finished.
// PAIRED (link pass): rows 2k and 2k+1 read the same records, so only the
// even rows' emissions are evaluated and both rows scale by them.
//
// Step schedule: the DMMAs of step i are issued, then the emission rows of
// the step's events are evaluated (they do not depend on the chain) while the
// tensor pipe works, then the products are scaled.  Quiet records need no
// evaluation: their emission row is the constant q row.  With one state per
// lane (K_p <= 32) event rows are evaluated two at a time (independent
// dependency chains).
template <int NT, bool SKIP, int TAIL, bool PAIRED, bool BATCH, typename Hook>
__device__ __forceinline__ void vec_run_impl(const ChainArgs& args, const double2* ent, const double* csm,
                                        const VecWarpSmem& w, double (&a)[NT][2],
                                        double (&at)[TAIL > 0 ? TAIL : 1], double& rexp, int64_t start,
                                        int64_t& len, int lane, Hook hook) {
  constexpr int RT = NT + (TAIL > 0 ? 1 : 0);
  constexpr int KPE = 8 * RT;
  constexpr int H = 8 * NT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  constexpr int SLOTS = vec_slots(KPE);
  constexpr int WIN = vec_win(RT);
  const int g = lane >> 2, q = lane & 3;
  const int K = args.K;
  const double* tab = csm + 10 * KPE;
  const double* qrow = csm + KPE;
  const unsigned ent_s = static_cast<unsigned>(__cvta_generic_to_shared(ent));  // once, not per step
  int64_t maxlen = len;
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) maxlen = max(maxlen, __shfl_xor_sync(kFull, maxlen, o));
  int since = 0;
  const int period = args.period;

  // batched emissions: LPE lanes per event (one state each), EPP events side by side
  constexpr int LPE = KPE <= 8 ? 8 : (KPE <= 16 ? 16 : 32);
  constexpr int EPP = 32 / LPE;
  auto consts = [&](StateConsts (&kc)[SLOTS]) {
#pragma unroll
    for (int sl = 0; sl < SLOTS; ++sl) {
      // (lanes >= KPE of the per-step pass compute discarded values; lane % LPE
      // gives the batched pass its state, and is the lane itself below KPE)
      const int j = min((SLOTS == 1 ? lane % LPE : lane) + 32 * sl, KPE - 1);
      kc[sl].p = csm[j];
      kc[sl].q = csm[KPE + j];
      kc[sl].mu0 = csm[2 * KPE + j];
      kc[sl].mu1 = csm[3 * KPE + j];
      kc[sl].l00 = csm[4 * KPE + j];
      kc[sl].l10 = csm[5 * KPE + j];
      kc[sl].l11 = csm[6 * KPE + j];
      kc[sl].c = csm[7 * KPE + j];
      kc[sl].r00 = csm[8 * KPE + j];
      kc[sl].r11 = csm[9 * KPE + j];
    }
  };
  StateConsts kc1[SLOTS];  // one state per lane: kept in registers for the whole run
  if (SLOTS == 1) consts(kc1);

  // emission rows of the present rows at window step i into eb; returns the step's 8 flags
  auto emit = [&](int i, double* eb) -> unsigned long long {
    const unsigned long long f8 = *reinterpret_cast<const unsigned long long*>(w.rf + 8 * i);
    unsigned pm = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) pm |= (((f8 >> (8 * r)) & 0xff) == 1 ? 1u : 0u) << r;
    if (PAIRED) pm &= 0x55u;
    if (SLOTS == 1) {
      const int j = lane;
      for (unsigned m = pm; m;) {
        const int r0 = __ffs(m) - 1;
        m &= m - 1;
        if (m) {  // two rows: independent chains interleave
          const int r1 = __ffs(m) - 1;
          m &= m - 1;
          const double e0 = emission_rc(true, w.rx[r0 * WIN + i], w.ry[r0 * WIN + i], kc1[0], tab);
          const double e1 = emission_rc(true, w.rx[r1 * WIN + i], w.ry[r1 * WIN + i], kc1[0], tab);
          if (j < KPE) {
            eb[r0 * KPE + j] = j < K ? e0 : 0.0;
            eb[r1 * KPE + j] = j < K ? e1 : 0.0;
          }
        } else {
          const double e0 = emission_rc(true, w.rx[r0 * WIN + i], w.ry[r0 * WIN + i], kc1[0], tab);
          if (j < KPE) eb[r0 * KPE + j] = j < K ? e0 : 0.0;
        }
      }
    } else if (pm) {
      StateConsts kc[SLOTS];
      consts(kc);
      for (unsigned m = pm; m; m &= m - 1) {
        const int r = __ffs(m) - 1;
        const double x = w.rx[r * WIN + i], y = w.ry[r * WIN + i];
#pragma unroll
        for (int sl = 0; sl < SLOTS; ++sl) {
          const int j = lane + 32 * sl;
          const double e = emission_rc(true, x, y, kc[sl], tab);
          if (j < KPE) eb[r * KPE + j] = j < K ? e : 0.0;
        }
      }
    }
    return f8;
  };

  // batched mode: emission rows of every event of window steps [i0, i0 + 8)
  // into w.ebuf in (step, row) order, four independent chains per lane; returns
  // the events as a 64-bit mask over (step - i0) * 8 + row
  constexpr bool batch = BATCH;
  auto emit_batch = [&](int i0) -> unsigned long long {
    unsigned m0 = __ballot_sync(kFull, w.rf[8 * i0 + lane] == 1);
    unsigned m1 = __ballot_sync(kFull, w.rf[8 * i0 + 32 + lane] == 1);
    if (PAIRED) {
      m0 &= 0x55555555u;
      m1 &= 0x55555555u;
    }
    // event list: slot -> (step - i0) * 8 + row, in that order
    const unsigned lt = (1u << lane) - 1u;
    if ((m0 >> lane) & 1u) w.elist[__popc(m0 & lt)] = static_cast<unsigned char>(lane);
    if ((m1 >> lane) & 1u) w.elist[__popc(m0) + __popc(m1 & lt)] = static_cast<unsigned char>(32 + lane);
    __syncwarp();
    const int nev = __popc(m0) + __popc(m1);
    const int sub = SLOTS == 1 ? lane / LPE : 0;
    for (int s0 = 0; s0 < nev; s0 += 4 * EPP) {
      int sl_[4];
      double xs[4], ys[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sl_[u] = s0 + u * EPP + sub;
        const int pp = w.elist[sl_[u] < nev ? sl_[u] : 0];
        const int r = pp & 7, t = i0 + (pp >> 3);
        xs[u] = w.rx[r * WIN + t];
        ys[u] = w.ry[r * WIN + t];
      }
#pragma unroll
      for (int sl = 0; sl < SLOTS; ++sl) {
        StateConsts kcs[1];
        if (SLOTS == 1) {
          kcs[0] = kc1[0];
        } else {
          const int j = min(lane + 32 * sl, KPE - 1);
          kcs[0] = StateConsts{csm[j], csm[KPE + j], csm[2 * KPE + j], csm[3 * KPE + j], csm[4 * KPE + j],
                               csm[5 * KPE + j], csm[6 * KPE + j], csm[7 * KPE + j], csm[8 * KPE + j],
                               csm[9 * KPE + j]};
        }
        double e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) e[u] = emission_rc(true, xs[u], ys[u], kcs[0], tab);
        const int j = (SLOTS == 1 ? lane % LPE : lane) + 32 * sl;
        if (j < KPE) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (sl_[u] < nev) w.ebuf[sl_[u] * KPE + j] = j < K ? e[u] : 0.0;
        }
      }
    }
    return static_cast<unsigned long long>(m0) | (static_cast<unsigned long long>(m1) << 32);
  };
  unsigned long long bmask = 0;
  int arrived = 0;  // staged single launch: time chunks known to have landed

  VEC_TR_DECL
  for (int64_t t0 = 0; t0 < maxlen; t0 += WIN) {
    // records [t0, t0 + WIN) of the 8 rows (consecutive lanes: consecutive
    // records of one row); device-resident streams load the coordinates
    // unconditionally (one memory latency, not two) and prefetch the next
    // window into L2; zero-copy streams read coordinates of present records only
    if (args.sysmem) {
#pragma unroll
      for (int k = 0; k < 8 * WIN / 32; ++k) {
        const int idx = lane + 32 * k, r = idx / WIN, t = idx - r * WIN;
        const int64_t st_r = __shfl_sync(kFull, start, 4 * r), len_r = __shfl_sync(kFull, len, 4 * r);
        unsigned char f = 2;
        double x = 0.0, y = 0.0;
        if (t0 + t < len_r) {
          const int64_t rec = st_r + t0 + t;
          if (args.sysmem == 2) {  // dense events: every line is needed anyway -- one PCIe round trip
            f = __ldcv(args.present + rec) != 0 ? 1 : 0;
            x = __ldcv(args.lon + rec);
            y = __ldcv(args.lat + rec);
          } else {
            f = load_record(args, rec, x, y) ? 1 : 0;
          }
        }
        w.rf[8 * t + r] = f;
        w.rx[r * WIN + t] = x;
        w.ry[r * WIN + t] = y;
      }
    } else {
      if (args.arrive && arrived < args.t_chunks) {
        // the time chunk holding this window's last record (per row; the warp's max)
        int need = 0;
        {
          const int64_t last = min(t0 + WIN, len) - 1;  // this lane's row
#pragma unroll 1
          for (int c = 1; c < args.t_chunks; ++c)
            if (last >= 0 && static_cast<int64_t>(static_cast<double>(len) * args.t_frac[c]) <= last) need = c;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) need = max(need, __shfl_xor_sync(kFull, need, o));
        if (need + 1 > arrived) {
          if (lane == 0) {
            unsigned v = 0;
            long long spins = 0;
            for (;;) {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(args.arrive) : "memory");
              if (static_cast<int>(v) >= need + 1 || ++spins > (1ll << 22)) break;  // (~1 s: never, unless a copy failed)
              __nanosleep(256);
            }
            if (static_cast<int>(v) < need + 1) {  // a copy never landed: flag (repeated unstaged), stop waiting
              atomicOr(args.link_fail + blockIdx.y, 4);
              v = static_cast<unsigned>(args.t_chunks);
            }
            arrived = static_cast<int>(v);
          }
          arrived = __shfl_sync(kFull, arrived, 0);
        }
      }
      // all loads of the window first (independent, in flight together), then the stores
      constexpr int KW = 8 * WIN / 32;
      unsigned char fr[KW];
      double xr[KW], yr[KW];
#pragma unroll
      for (int k = 0; k < KW; ++k) {
        const int idx = lane + 32 * k, r = idx / WIN, t = idx - r * WIN;
        const int64_t st_r = __shfl_sync(kFull, start, 4 * r), len_r = __shfl_sync(kFull, len, 4 * r);
        const bool ok = t0 + t < len_r;
        const int64_t rec = ok ? st_r + t0 + t : 0;
        fr[k] = ok ? (args.present[rec] != 0 ? 1 : 0) : 2;
        xr[k] = ok ? args.lon[rec] : 0.0;
        yr[k] = ok ? args.lat[rec] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < KW; ++k) {
        const int idx = lane + 32 * k, r = idx / WIN, t = idx - r * WIN;
        w.rf[8 * t + r] = fr[k];
        w.rx[r * WIN + t] = xr[k];
        w.ry[r * WIN + t] = yr[k];
      }
      // next window of every row into L2 (lanes 0..7: one row each; addresses inside the row's records)
      const int64_t st_r = __shfl_sync(kFull, start, 4 * (lane & 7)), len_r = __shfl_sync(kFull, len, 4 * (lane & 7));
      if (lane < 8) {
        if (t0 + WIN < len_r) {
          const int64_t rec = st_r + t0;
          const int64_t last = min(static_cast<int64_t>(2 * WIN - 1), len_r - 1 - t0);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(args.present + rec + WIN));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(args.lon + rec + WIN));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(args.lat + rec + WIN));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(args.lon + rec + last));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(args.lat + rec + last));
        }
      }
    }
    __syncwarp();
    VEC_TR(0)
    const int cnt = static_cast<int>(maxlen - t0 < WIN ? maxlen - t0 : WIN);
    for (int i = 0; i < cnt; ++i) {
      double c[NT][2], ct[TA];
      if (batch && (i & (kVecBatchSteps - 1)) == 0) {
        bmask = emit_batch(i);
        __syncwarp();
      }
      runs_mul_issue<NT, SKIP, TAIL>(c, ct, a, at, ent, ent_s, lane);
      VEC_TR(1)
      const double* e_cur = w.ebuf;
      unsigned long long f_cur = 0;
      if (batch)
        f_cur = *reinterpret_cast<const unsigned long long*>(w.rf + 8 * i);
      else
        f_cur = emit(i, w.ebuf);  // while the DMMAs run
      runs_mul_couple<NT, TAIL>(c, at, ent_s, lane);
#ifdef THMM_VEC_TRACE
      if (c[0][0] == -1.2345) tr_acc[7] += 1;  // wait for the products here (timing only)
#endif
      VEC_TR(4)
      __syncwarp();
      if (t0 + i < len) {
        const int gr = PAIRED ? (g & ~1) : g;
        const bool ev = ((f_cur >> (8 * gr)) & 0xff) == 1;
        const int pb = 8 * (i & (kVecBatchSteps - 1)) + gr;  // batched: slot = events before (step, row)
        const int erow_i = batch ? __popcll(bmask & ((1ull << pb) - 1ull)) : gr;
        const double* erow = ev ? e_cur + erow_i * KPE : qrow;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 ev = *reinterpret_cast<const double2*>(erow + 8 * nt + 2 * q);
          a[nt][0] = c[nt][0] * ev.x;
          a[nt][1] = c[nt][1] * ev.y;
        }
#pragma unroll
        for (int j = 0; j < TAIL; ++j) at[j] = ct[j] * erow[H + j];
      }
      __syncwarp();
      if (++since == period) {
        since = 0;
        renorm_row_tail<NT, TAIL>(a, at, rexp);
      }
      VEC_TR(5)
      if (hook(t0 + i, since)) {
        t0 = maxlen;  // every row of the warp is finished
        break;
      }
    }
    __syncwarp();
  }
  renorm_row_tail<NT, TAIL>(a, at, rexp);
#ifdef THMM_VEC_TRACE
  if (args.trace && lane == 0) {
    const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int k = 0; k < 8; ++k) args.trace[wid * 8 + k] = tr_acc[k];
  }
#endif
}

// One inlined copy per emission mode (args.ebatch, warp-uniform for the
// launch): each gets its own register allocation.
template <int NT, bool SKIP, int TAIL, bool PAIRED = false, typename Hook>
__device__ __forceinline__ void vec_run(const ChainArgs& args, const double2* ent, const double* csm,
                                        const VecWarpSmem& w, double (&a)[NT][2],
                                        double (&at)[TAIL > 0 ? TAIL : 1], double& rexp, int64_t start,
                                        int64_t& len, int lane, Hook hook) {
  if (args.ebatch)
    vec_run_impl<NT, SKIP, TAIL, PAIRED, true>(args, ent, csm, w, a, at, rexp, start, len, lane, hook);
  else
    vec_run_impl<NT, SKIP, TAIL, PAIRED, false>(args, ent, csm, w, a, at, rexp, start, len, lane, hook);
}

// Load a row (KPE doubles) into the accumulator layout of row g of the warp.
template <int NT, int TAIL>
__device__ __forceinline__ void vec_load_row(const double* r0, double (&a)[NT][2], double (&at)[TAIL > 0 ? TAIL : 1],
                                             int q) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const double2 v = *reinterpret_cast<const double2*>(r0 + 8 * nt + 2 * q);
    a[nt][0] = v.x;
    a[nt][1] = v.y;
  }
#pragma unroll
  for (int j = 0; j < TAIL; ++j) at[j] = r0[8 * NT + j];
}

// Store row g of the warp (accumulator layout) as KPE doubles (tail padded with zeros).
template <int NT, int TAIL>
__device__ __forceinline__ void vec_store_row(double* r0, const double (&a)[NT][2],
                                              const double (&at)[TAIL > 0 ? TAIL : 1], int q) {
  constexpr int H = 8 * NT;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) *reinterpret_cast<double2*>(r0 + 8 * nt + 2 * q) = make_double2(a[nt][0], a[nt][1]);
  if (TAIL > 0 && q == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r0[H + j] = j < TAIL ? at[j < TAIL ? j : 0] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Collapse continuation: every collapsed segment from its pivot row r over the
// rest of its records; node c r_final' in the tree's format.
// ---------------------------------------------------------------------------
template <int NT, bool SKIP, int TAIL>
__global__ void __launch_bounds__(32 * vec_warps(NT + (TAIL > 0)), vec_min_blocks(NT, TAIL))
    chain_vec_kernel(const ChainArgs args) {
  constexpr int RT = NT + (TAIL > 0 ? 1 : 0);
  constexpr int KPE = 8 * RT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ent = reinterpret_cast<double2*>(smem_raw);                       // Gamma
  double* csm = reinterpret_cast<double*>(ent + runs_entry_pairs(NT, TAIL));  // [10][KPE] state constants
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int K = args.K;
  const VecWarpSmem w = vec_warp_smem<KPE>(csm, warp, args.ebatch != 0);
  vec_prologue<NT, TAIL>(args, b, ent, csm);

  // my row: segment seg of proposal b
  const int64_t seg = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * 8 + g;
  const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg;
  int64_t start = 0, len = 0;
  double rexp = 0.0;
  bool active = false;
  double a[NT][2], at[TA];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) a[nt][0] = a[nt][1] = 0.0;
#pragma unroll
  for (int j = 0; j < TA; ++j) at[j] = 0.0;
  if (seg < args.nseg) {
    const double t_s = args.col_meta[2 * node];
    if (t_s >= 0.0) {
      int64_t s_lo, s_hi;
      segment_range(args.n, args.nseg, seg, s_lo, s_hi);
      active = true;
      start = args.lo + s_lo + static_cast<int64_t>(t_s);
      len = (s_hi - s_lo) - static_cast<int64_t>(t_s);
      rexp = args.col_meta[2 * node + 1];
      vec_load_row<NT, TAIL>(args.col_r + node * KPE, a, at, q);
    }
  }
  vec_run<NT, SKIP, TAIL>(args, ent, csm, w, a, at, rexp, start, len, lane, [](int64_t, int) { return false; });

  // nodes: m_ij = 2^d_i rho_i r_j (r normalised, node exponent = the row's), rows >= K zero
  vec_store_row<NT, TAIL>(w.ebuf + g * KPE, a, at, q);
  __syncwarp();
#pragma unroll 1
  for (int r = 0; r < 8; ++r) {
    const bool act = __shfl_sync(kFull, active, 4 * r);
    if (!act) continue;
    const double E = __shfl_sync(kFull, rexp, 4 * r);
    const size_t nd = node - g + r;  // node of row r (same proposal, consecutive segments)
    const double* d = args.col_d + nd * KPE;
    const double* rc = args.col_c + nd * KPE;
    const double* rr = w.ebuf + r * KPE;
    double* out = args.seg_m + nd * KPE * KPE;
    for (int idx = lane; idx < KPE * KPE / 2; idx += 32) {
      const int i = idx / (KPE / 2), j = 2 * (idx - i * (KPE / 2));
      double v0 = 0.0, v1 = 0.0;
      if (i < K) {
        const double di = d[i];
        if (di >= -2044.0) {
          const int sh = static_cast<int>(di);
          const double ci = rc[i];
          v0 = scale_pow2(__dmul_rn(ci, rr[j]), sh);
          v1 = scale_pow2(__dmul_rn(ci, rr[j + 1]), sh);
        }
      }
      *reinterpret_cast<double2*>(out + static_cast<size_t>(i) * KPE + j) = make_double2(v0, v1);
    }
    if (lane == 0) args.seg_e[nd] = E;
  }
}

// ---------------------------------------------------------------------------
// Stitched chain (finish evaluations).  The forward filter forgets its start
// vector: two forward rows started anywhere become proportional after a few
// dozen records.  So every segment s >= 1 runs ONE row from the all-ones
// vector (segment 0 from delta) over its records -- u M_s = 2^E_s w_s -- and
// a second pass links consecutive segments: the previous segment's final row
// w_{s-1} and the all-ones row are both propagated from the start of segment s
// until they are proportional (every entry within tol relative, tested every
// 8 records: p = 2^G p^, h = 2^F h^, p^ = rho h^).  By linearity and
// nonnegativity the true forward vector at the end of s is then
//     alpha_s w_s,  alpha_s = alpha_{s-1} rho_s 2^(G_s + E_s - F_s)
// within a factor 1 +- tol, and
//     log L = E_0 ln 2 + sum_{s>=1} [log rho_s + (G_s + E_s - F_s) ln 2] + log(w_{S-1} . 1).
// No K x K product is formed anywhere: 2K^2 flop per record, plus ~2 x 8-48
// records per segment for the links.  A link that does not converge within
// its segment flags the evaluation, which the host then repeats on the
// rank-one collapse path (exact in every case).
// ---------------------------------------------------------------------------

// Main pass: row g = segment seg; start delta (segment 0 when args.stitch_delta)
// or all-ones; writes the final normalised row and its exponent.
template <int NT, bool SKIP, int TAIL>
__global__ void __launch_bounds__(32 * vec_warps(NT + (TAIL > 0)), vec_min_blocks(NT, TAIL))
    chain_fwd_kernel(const ChainArgs args) {
  constexpr int RT = NT + (TAIL > 0 ? 1 : 0);
  constexpr int KPE = 8 * RT;
  constexpr int H = 8 * NT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ent = reinterpret_cast<double2*>(smem_raw);
  double* csm = reinterpret_cast<double*>(ent + runs_entry_pairs(NT, TAIL));
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int K = args.K;
  const VecWarpSmem w = vec_warp_smem<KPE>(csm, warp, args.ebatch != 0);
  vec_prologue<NT, TAIL>(args, b, ent, csm);

  const int64_t seg = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * 8 + g;
  const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg;
  int64_t start = 0, len = 0;
  double rexp = 0.0;
  double a[NT][2], at[TA];
  const bool active = seg < args.nseg;
  const int C = (args.t_chunks > 1 && !args.arrive) ? args.t_chunks : 1, ci = C > 1 ? args.t_chunk : 0;
  const bool from_delta = active && seg == 0 && args.stitch_delta;
  const double* delta = args.P.delta + static_cast<size_t>(b) * K;
  if (ci == 0) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 8 * nt + 2 * q + h;
        a[nt][h] = (active && j < K) ? (from_delta ? delta[j] : 1.0) : 0.0;
      }
#pragma unroll
    for (int j = 0; j < TA; ++j) at[j] = (TAIL > 0 && active) ? (from_delta ? delta[H + j] : 1.0) : 0.0;
  } else {  // continue the row the previous time chunk left (normalised, exponent in fin_e)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) a[nt][0] = a[nt][1] = 0.0;
#pragma unroll
    for (int j = 0; j < TA; ++j) at[j] = 0.0;
    if (active) {
      vec_load_row<NT, TAIL>(args.fin + node * KPE, a, at, q);
      rexp = args.fin_e[node];
    }
  }
  if (active) {
    int64_t s_lo, s_hi;
    segment_range(args.n, args.nseg, seg, s_lo, s_hi);
    const int64_t L = s_hi - s_lo;
    const int64_t tb = C > 1 ? time_chunk_begin(L, args.t_frac, ci) : 0;
    start = args.lo + s_lo + tb;
    len = (C > 1 ? time_chunk_begin(L, args.t_frac, ci + 1) : L) - tb;
  }
  vec_run<NT, SKIP, TAIL>(args, ent, csm, w, a, at, rexp, start, len, lane, [](int64_t, int) { return false; });
  if (active) {
    vec_store_row<NT, TAIL>(args.fin + node * KPE, a, at, q);
    if (q == 0) args.fin_e[node] = rexp;
  }
}

// Link pass: rows (2k, 2k+1) of a warp = (p, h) of segment s = 4 warp + k + 1
// (segments 1 .. nseg-1): p from w_{s-1} (exponent 0), h from all-ones, both
// over the records of segment s until proportional.  Writes the link term
// log rho_s + (G_s - F_s) ln 2, or flags the proposal (link_fail).
template <int NT, bool SKIP, int TAIL>
__global__ void __launch_bounds__(32 * vec_warps(NT + (TAIL > 0)), vec_min_blocks(NT, TAIL))
    chain_link_kernel(const ChainArgs args) {
  constexpr int RT = NT + (TAIL > 0 ? 1 : 0);
  constexpr int KPE = 8 * RT;
  constexpr int H = 8 * NT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ent = reinterpret_cast<double2*>(smem_raw);
  double* csm = reinterpret_cast<double*>(ent + runs_entry_pairs(NT, TAIL));
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int K = args.K;
  const VecWarpSmem w = vec_warp_smem<KPE>(csm, warp, args.ebatch != 0);
  vec_prologue<NT, TAIL>(args, b, ent, csm);

  // external mode (args.link_src): segment 0 of this range, p from another rank's final row
  const bool ext = args.link_src != nullptr;
  const int64_t seg = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * 4 + (g >> 1) + (ext ? 0 : 1);
  const bool is_p = (g & 1) == 0;
  const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg;
  int64_t start = 0, len = 0;
  double rexp = 0.0;
  double a[NT][2], at[TA];
  const bool active = seg < (ext ? 1 : args.nseg);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) a[nt][0] = a[nt][1] = 0.0;
#pragma unroll
  for (int j = 0; j < TA; ++j) at[j] = 0.0;
  if (active) {
    int64_t s_lo, s_hi;
    segment_range(args.n, args.nseg, seg, s_lo, s_hi);
    start = args.lo + s_lo;
    len = s_hi - s_lo;
    if (is_p) {
      vec_load_row<NT, TAIL>(ext ? args.link_src + static_cast<size_t>(b) * args.link_src_stride
                                 : args.fin + (node - 1) * KPE,
                             a, at, q);
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) a[nt][h] = (8 * nt + 2 * q + h < K) ? 1.0 : 0.0;
#pragma unroll
      for (int j = 0; j < TAIL; ++j) at[j] = 1.0;
    }
  }
  const int64_t seg_len = len;
  bool done = !active;  // this pair's link found (or no pair)
  const double tol = args.collapse_tol, slack = 0x1p-1022;
  auto hook = [&](int64_t t, int) -> bool {
    const bool at_end = active && t == seg_len - 1;
    if ((t & 7) != 7 && !__any_sync(kFull, at_end)) return false;  // test every 8 records and at segment ends
    renorm_row_tail<NT, TAIL>(a, at, rexp);  // exact: both rows of every pair to max in [1, 2)
    // p lanes read their h partner (lane + 4: row g + 1, same columns)
    double pa[NT][2], pt[TA];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      pa[nt][0] = __shfl_down_sync(kFull, a[nt][0], 4);
      pa[nt][1] = __shfl_down_sync(kFull, a[nt][1], 4);
    }
#pragma unroll
    for (int j = 0; j < TA; ++j) pt[j] = __shfl_down_sync(kFull, at[j], 4);
    const double hexp = __shfl_down_sync(kFull, rexp, 4);
    // j*: first largest entry of h (quad reduction on (value, column))
    double hv = -1.0;
    int hj = 0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (pa[nt][h] > hv) {
          hv = pa[nt][h];
          hj = 8 * nt + 2 * q + h;
        }
#pragma unroll
    for (int j = 0; j < TAIL; ++j)
      if (pt[j] > hv) {
        hv = pt[j];
        hj = H + j;
      }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const double ov = __shfl_xor_sync(kFull, hv, o);
      const int oj = __shfl_xor_sync(kFull, hj, o);
      if (ov > hv || (ov == hv && oj < hj)) {
        hv = ov;
        hj = oj;
      }
    }
    double pv = 0.0;  // p at j*
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (8 * nt + 2 * q + h == hj) pv = a[nt][h];
    pv += __shfl_xor_sync(kFull, pv, 1);
    pv += __shfl_xor_sync(kFull, pv, 2);
#pragma unroll
    for (int j = 0; j < TAIL; ++j)
      if (H + j == hj) pv = at[j];
    const double rho = hv > 0.0 ? __ddiv_rn(pv, hv) : 0.0;
    bool bad = !(rho > 0.0);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double e0 = __dmul_rn(rho, pa[nt][h]);
        bad |= !(fabs(a[nt][h] - e0) <= fma(tol, e0, slack));
      }
#pragma unroll
    for (int j = 0; j < TAIL; ++j) {
      const double e0 = __dmul_rn(rho, pt[j]);
      bad |= !(fabs(at[j] - e0) <= fma(tol, e0, slack));
    }
    bad |= __shfl_xor_sync(kFull, bad, 1);
    bad |= __shfl_xor_sync(kFull, bad, 2);
    bool linked = is_p && !done && !bad;
    if (linked && q == 0) {
      const double term = log(rho) + (rexp - hexp) * 0.6931471805599453;
      if (ext)
        args.link_out[2 * b] = term;
      else
        args.link[node] = term;
    }
    // the h row of the pair (lane + 4) learns the outcome from its p row
    const bool linked_pair = __shfl_sync(kFull, linked, is_p ? lane : lane - 4);
    if (linked_pair) {
      done = true;
      len = t + 1;  // both rows of the pair stop here
    }
    if (is_p && !done && at_end && q == 0) {  // no link within the segment
      if (ext)
        args.link_out[2 * b + 1] = 1.0;
      else
        args.link_fail[b] = 1;
    }
    if (at_end) done = true;
    return __all_sync(kFull, done);
  };
  vec_run<NT, SKIP, TAIL, true>(args, ent, csm, w, a, at, rexp, start, len, lane, hook);
}

// log L per proposal from the main pass and the links (fixed summation
// order: deterministic).  status: 1 collapse (zero / non-finite), 3 a link
// failed (the host repeats the evaluation on the collapse path).
// With `block` (a shard of a multi-GPU chain): [B][KPE + 2] = the final
// normalised row, the shard's log-scale A = E_0 ln 2 + sum_{s>=1} (link_s + E_s ln 2)
// relative to its start vector, and the fail flag -- instead of log L.
template <int KPE>
__global__ void __launch_bounds__(256) stitch_finish_kernel(const ChainArgs args, double* loglik, int32_t* status,
                                                             double* block) {
  __shared__ double red[8];
  const int b = blockIdx.x;
  const size_t base = static_cast<size_t>(b) * args.node_stride_b + args.node_offset;
  const int64_t S = args.nseg;
  constexpr double kLn2 = 0.6931471805599453;
  double acc = 0.0;
  for (int64_t s = threadIdx.x; s < S; s += blockDim.x)
    acc += (s == 0 ? 0.0 : args.link[base + s]) + args.fin_e[base + s] * kLn2;
  acc = block_sum(acc, red, blockDim.x / 32);
  double tail = 0.0;
  for (int j = threadIdx.x; j < KPE; j += blockDim.x) tail += args.fin[(base + S - 1) * KPE + j];
  tail = block_sum(tail, red, blockDim.x / 32);
  if (block) {
    double* out = block + static_cast<size_t>(b) * (KPE + 2);
    for (int j = threadIdx.x; j < KPE; j += blockDim.x) out[j] = args.fin[(base + S - 1) * KPE + j];
    __syncthreads();
    if (threadIdx.x == 0) {
      out[KPE] = acc;
      out[KPE + 1] = args.link_fail[b] ? 1.0 : 0.0;
      args.link_fail[b] = 0;
    }
    return;
  }
  if (threadIdx.x == 0) {
    const double ll = acc + log(tail);
    const int fail = args.link_fail[b];
    args.link_fail[b] = 0;  // reset for the next evaluation (graph replays)
    loglik[b] = (tail > 0.0 && isfinite(ll)) ? ll : -INFINITY;
    status[b] = fail ? 3 : ((tail > 0.0 && isfinite(ll)) ? 0 : 1);
  }
}

}  // namespace thmm
