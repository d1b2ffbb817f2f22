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

constexpr int kVecWin = 32;  // records staged per window (per row)

__host__ __device__ constexpr int vec_slots(int kpe) { return (kpe + 31) / 32; }

// Shared memory: Gamma (runs entry layout) + the state constants, then per
// warp: the 8 rows' records of one window and one step's emission rows.
__host__ __device__ constexpr size_t vec_warp_bytes(int kpe) {
  return static_cast<size_t>(8) * kVecWin * 16 + static_cast<size_t>(8) * kVecWin + static_cast<size_t>(8) * kpe * 8;
}
__host__ __device__ constexpr size_t vec_smem_bytes(int nt, int tail, int warps) {
  return static_cast<size_t>(runs_entry_pairs(nt, tail)) * 16 + static_cast<size_t>(10) * 8 * (nt + (tail > 0)) * 8 +
         static_cast<size_t>(warps) * vec_warp_bytes(8 * (nt + (tail > 0)));
}
// Warps per CTA: 16 for rows of <= 4 tiles (two CTAs per SM, <= 64
// registers), 12 for wider rows (one CTA per SM, <= 168 registers: the
// accumulators plus the emission constants of SLOTS states stay in registers).
__host__ __device__ constexpr int vec_warps(int rt) { return rt <= 4 ? 16 : 12; }
__host__ __device__ constexpr int vec_min_blocks(int nt, int tail) { return nt + (tail > 0) <= 4 ? 2 : 1; }

template <int NT, bool SKIP, int TAIL>
__global__ void __launch_bounds__(32 * vec_warps(NT + (TAIL > 0)), vec_min_blocks(NT, TAIL))
    chain_vec_kernel(const ChainArgs args) {
  constexpr int RT = NT + (TAIL > 0 ? 1 : 0);
  constexpr int KPE = 8 * RT;
  constexpr int H = 8 * NT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  constexpr int SLOTS = vec_slots(KPE);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ent = reinterpret_cast<double2*>(smem_raw);                       // Gamma
  double* csm = reinterpret_cast<double*>(ent + runs_entry_pairs(NT, TAIL));  // [10][KPE] state constants
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int K = args.K;
  unsigned char* wsm = reinterpret_cast<unsigned char*>(csm + 10 * KPE) + static_cast<size_t>(warp) * vec_warp_bytes(KPE);
  double* rx = reinterpret_cast<double*>(wsm);  // [8][kVecWin]
  double* ry = rx + 8 * kVecWin;                // [8][kVecWin]
  double* ebuf = ry + 8 * kVecWin;              // [8][KPE]
  unsigned char* rf = reinterpret_cast<unsigned char*>(ebuf + 8 * KPE);  // [8][kVecWin]: 0 quiet, 1 event, 2 none

  const double* gam = args.P.gamma + static_cast<size_t>(b) * K * K;
  runs_stage_entry<NT, TAIL>(ent, K, [&](int i, int j) { return gam[i * K + j]; });
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
  __syncthreads();

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
      const double* r0 = args.col_r + node * KPE;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double2 v = *reinterpret_cast<const double2*>(r0 + 8 * nt + 2 * q);
        a[nt][0] = v.x;
        a[nt][1] = v.y;
      }
#pragma unroll
      for (int j = 0; j < TAIL; ++j) at[j] = r0[H + j];
    }
  }
  int64_t maxlen = len;
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) maxlen = max(maxlen, __shfl_xor_sync(kFull, maxlen, o));

  int since = 0;
  const int period = args.period;
  for (int64_t t0 = 0; t0 < maxlen; t0 += kVecWin) {
    // records [t0, t0 + 32) of the 8 rows: lane l loads step t0 + l of every row
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int64_t st_r = __shfl_sync(kFull, start, 4 * r), len_r = __shfl_sync(kFull, len, 4 * r);
      const int64_t t = t0 + lane;
      unsigned char f = 2;
      double x = 0.0, y = 0.0;
      if (t < len_r) f = load_record(args, st_r + t, x, y) ? 1 : 0;
      rf[r * kVecWin + lane] = f;
      rx[r * kVecWin + lane] = x;
      ry[r * kVecWin + lane] = y;
    }
    __syncwarp();
    const int cnt = static_cast<int>(maxlen - t0 < kVecWin ? maxlen - t0 : kVecWin);
    for (int i = 0; i < cnt; ++i) {
      double c[NT][2], ct[TA];
      runs_mul<NT, SKIP, TAIL>(c, ct, a, at, ent, lane);
      // emission rows of the 8 rows' records at this step, one state per lane
      // (SLOTS states per lane: independent chains); loops over the present /
      // quiet rows of the step (warp-uniform masks) keep the code small
      {
        StateConsts kc[SLOTS];
#pragma unroll
        for (int sl = 0; sl < SLOTS; ++sl) {
          const int j = min(lane + 32 * sl, KPE - 1);
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
        unsigned pm = 0, qm = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const unsigned char f = rf[r * kVecWin + i];
          pm |= (f == 1 ? 1u : 0u) << r;
          qm |= (f == 0 ? 1u : 0u) << r;
        }
        for (unsigned m = qm; m; m &= m - 1) {
          const int r = __ffs(m) - 1;
#pragma unroll
          for (int sl = 0; sl < SLOTS; ++sl) {
            const int j = lane + 32 * sl;
            if (j < KPE) ebuf[r * KPE + j] = j < K ? kc[sl].q : 0.0;
          }
        }
        for (unsigned m = pm; m; m &= m - 1) {
          const int r = __ffs(m) - 1;
          const double x = rx[r * kVecWin + i], y = ry[r * kVecWin + i];
#pragma unroll
          for (int sl = 0; sl < SLOTS; ++sl) {
            const int j = lane + 32 * sl;
            const double e = emission_rc(true, x, y, kc[sl]);
            if (j < KPE) ebuf[r * KPE + j] = j < K ? e : 0.0;
          }
        }
      }
      __syncwarp();
      if (t0 + i < len) {
        const double* erow = ebuf + g * KPE;
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
    }
    __syncwarp();
  }
  renorm_row_tail<NT, TAIL>(a, at, rexp);

  // nodes: m_ij = 2^d_i rho_i r_j (r normalised, node exponent = the row's), rows >= K zero
  {
    double* erow = ebuf + g * KPE;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) *reinterpret_cast<double2*>(erow + 8 * nt + 2 * q) = make_double2(a[nt][0], a[nt][1]);
    if (TAIL > 0 && q == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) erow[H + j] = 0.0;
#pragma unroll
      for (int j = 0; j < TAIL; ++j) erow[H + j] = at[j];
    }
  }
  __syncwarp();
#pragma unroll 1
  for (int r = 0; r < 8; ++r) {
    const bool act = __shfl_sync(kFull, active, 4 * r);
    if (!act) continue;
    const double E = __shfl_sync(kFull, rexp, 4 * r);
    const size_t nd = node - g + r;  // node of row r (same proposal, consecutive segments)
    const double* d = args.col_d + nd * KPE;
    const double* rc = args.col_c + nd * KPE;
    const double* rr = ebuf + r * KPE;
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

}  // namespace thmm
